timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_twocall.py -x -q -p no:cacheprovider 2>&1 | tail -2
for L in libdkv.so libdkv_old.so libdkv.so libdkv_old.so libdkv.so libdkv_old.so; do echo -n "$L "; DKV_LIB=$L REPS=250 timeout 200 python tools/power_probe.py fwd; done
for i in 1 2; do for L in libdkv.so libdkv_old.so; do DKV_LIB=$L timeout 100 python tools/time_fwd.py; done; done
