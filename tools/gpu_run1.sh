set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
bash tools/hang_probe.sh
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 200 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/bench.txt
