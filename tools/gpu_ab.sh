# A/B: GPU tests on the default build, then the bench (kernel split) for default vs DKV_BWD_V1=1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 2>&1 | tail -15
for v in 0 1; do
  DKV_BWD_V2=$v timeout 300 python bench.py --no-cpu --no-e2e --no-replicated 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('V2=$v', d['value'], 'fwd', d['fwd_ms_group0'], 'bwd', d['bwd_ms_group0'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done
