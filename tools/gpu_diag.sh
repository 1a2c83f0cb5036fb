DKV_BWD_PAIR=1 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider 2>&1 | tail -2
DKV_BWD_PAIR=1 DKV_LIB=libdkv_trace.so timeout 120 python tools/trace_bwd.py 0 4 2>&1 | tail -11
for i in 1 2; do for pr in 0 1; do echo -n "pair=$pr "; DKV_BWD_PAIR=$pr timeout 200 python tools/ablate_bwd.py 0; done; done
for pr in 0 1 0 1; do echo -n "pair=$pr "; DKV_BWD_PAIR=$pr timeout 200 python tools/power_probe.py bwd; done
