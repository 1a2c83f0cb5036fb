for L in libdkv.so libdkv_old.so libdkv.so libdkv_old.so libdkv.so libdkv_old.so; do echo -n "$L "; DKV_LIB=$L REPS=80 timeout 200 python tools/power_probe.py bwd; done
