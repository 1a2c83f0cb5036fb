timeout 300 python -m pytest tests/test_gpu_rope.py tests/test_gpu_pipeline.py tests/test_gpu_layer.py -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do for L in libdkv.so libdkv_old.so; do DKV_LIB=$L timeout 100 python tools/time_repack.py; done; done
