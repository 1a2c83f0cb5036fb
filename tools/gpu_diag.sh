# scratch script for one-off gpurun experiments (its content changes per experiment)
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 200 2>&1 | tail -2
