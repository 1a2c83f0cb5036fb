timeout 600 python -m pytest tests/test_gpu_rescale.py -q -p no:cacheprovider 2>&1 | tail -8
