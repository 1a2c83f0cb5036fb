mkdir -p gpurun_out/c1
timeout 600 python -m pytest tests/test_gpu_twocall.py tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_structure.py -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/c1/tests.log
DKV_FORCE_SIMT=1 timeout 600 python -m pytest tests/test_gpu_twocall.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "not tensor" 2>&1 | tail -2 >> gpurun_out/c1/tests.log
for r in 1 2; do timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu > gpurun_out/c1/bench_$r.json 2>/dev/null; done
