mkdir -p gpurun_out/pb
for r in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-replicated > gpurun_out/pb/def_$r.json 2>/dev/null
  DKV_BWD_PAIR=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-replicated > gpurun_out/pb/pair_$r.json 2>/dev/null
done
