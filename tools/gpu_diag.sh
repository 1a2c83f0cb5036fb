for L in libdkv.so libdkv_old.so libdkv.so libdkv_old.so; do echo -n "$L "; DKV_LIB=$L REPS=250 timeout 200 python tools/power_probe.py fwd; done
