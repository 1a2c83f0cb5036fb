DKV_FWD_PAIR=1 DKV_LIB=libdkv_trace.so timeout 120 python tools/trace_fwd.py 0 6 2>&1 | grep -v -i "warn\|mean\|ret =\|nan" | head -9
DKV_FWD_PAIR=1 timeout 300 python -m pytest tests/test_gpu_variants.py -x -q -p no:cacheprovider 2>&1 | tail -1
for pr in 0 1 0 1; do echo -n "pair=$pr "; DKV_FWD_PAIR=$pr REPS=250 timeout 200 python tools/power_probe.py fwd; done
