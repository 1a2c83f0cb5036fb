#!/bin/bash
# Round-2 final evidence pass (one B200): GPU tests + smoke, the driver's bench command, every other
# BASELINE config, the 2-rank paths on one GPU, the reference arm, ncu launch list + full captures of
# both main kernels + L2 reduction counts, sanitizer-free.
mkdir -p gpurun_out/ev
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | grep -v "^  \|warn" | tail -40 > gpurun_out/ev/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev/bench_C3.json 2> gpurun_out/ev/bench_C3.err
for c in C5 C2 C1 C4 Q14; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err
done
DKV_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --config C2 --no-e2e --no-replicated > gpurun_out/ev/bench_2rank.json 2> gpurun_out/ev/bench_2rank.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-replicated > gpurun_out/ev/bench_under_ncu.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 -f \
    -o gpurun_out/ev/prof_bwd python tools/profile_step.py > gpurun_out/ev/prof_bwd.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:dualkv_fwd -c 1 -f \
    -o gpurun_out/ev/prof_fwd python tools/profile_step.py > gpurun_out/ev/prof_fwd.txt 2>&1
tail -3 gpurun_out/ev/pytest.log
