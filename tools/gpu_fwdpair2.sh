mkdir -p gpurun_out
DKV_FWD_PAIR=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/fwdpair_suite.log
for r in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-replicated > gpurun_out/fwdpair_bench_def_$r.json 2>/dev/null
  DKV_FWD_PAIR=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-replicated > gpurun_out/fwdpair_bench_pair_$r.json 2>/dev/null
done
