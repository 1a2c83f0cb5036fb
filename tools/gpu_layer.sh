mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_qkv_prep.py tests/test_gpu_layer.py tests/test_gpu_groups.py -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/layer_tests.log
python tools/profile_layer.py > gpurun_out/layer_prof2.txt 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu > gpurun_out/bench_C4_new.json 2>/dev/null
