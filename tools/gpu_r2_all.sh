#!/bin/bash
# Round-2 GPU pass: GPU tests, bench lines for every BASELINE config, full-C3 CPU calibration.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | grep -v "^  \|warn" | tail -40 > gpurun_out/pytest.log
for c in C3 C5 C2 C1 C4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 1500 python tools/cpu_full_c3.py --out gpurun_out/r2_cpu_full_c3.json > gpurun_out/cpu_full.log 2>&1
tail -3 gpurun_out/pytest.log
