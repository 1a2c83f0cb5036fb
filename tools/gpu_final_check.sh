mkdir -p gpurun_out/fin
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/fin/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin/bench_C3.json 2> gpurun_out/fin/bench_C3.err
