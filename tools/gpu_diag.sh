timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 200 2>&1 | tail -2
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
