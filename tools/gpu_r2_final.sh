#!/bin/bash
# Round-2 evidence pass on one B200: GPU tests + smoke, the driver's bench command, every other
# BASELINE config, the 2-rank bench path on one GPU, ncu launch list + full captures, traces.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | grep -v "^  \|warn" | tail -40 > gpurun_out/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
for c in C5 C2 C1 C4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
DKV_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --config C2 --no-e2e --no-replicated > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
DKV_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --gpus 2 --steps 2 --warmup 3 --config C4 > gpurun_out/bench_2rank_C4.json 2> gpurun_out/bench_2rank_C4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/gpu_prof_r2.sh
make -C paper_2605_15422_b200/csrc trace -j8 > /dev/null 2>&1
DKV_LIB=libdkv_trace.so python tools/trace_bwd.py 0 40 > gpurun_out/trace_bwd0.txt 2>&1
DKV_LIB=libdkv_trace.so python tools/trace_fwd.py > gpurun_out/trace_fwd.txt 2>&1
tail -3 gpurun_out/pytest.log
