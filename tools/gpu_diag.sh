for L in libdkv.so libdkv_old.so libdkv.so libdkv_old.so; do echo -n "$L "; DKV_LIB=$L timeout 600 python bench.py --no-cpu --no-e2e --no-replicated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], 'fwd', d['fwd_ms_group0'], 'bwd', d['bwd_ms_group0'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"; done
