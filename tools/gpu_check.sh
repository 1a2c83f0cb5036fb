mkdir -p gpurun_out
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm --format=csv > gpurun_out/gpu1_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x 2>&1 | tail -15 > gpurun_out/gpu1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/gpu1_smoke.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/gpu1_bench_C3.json 2> gpurun_out/gpu1_bench_C3.err
