# Full evidence pass: GPU tests, smoke, default bench, ncu launch list of the bench command,
# ncu --set full of the two main kernels.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 200 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.txt 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.txt
if [ "${SKIP_NCU:-0}" != "1" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
    python bench.py --no-cpu > gpurun_out/bench_under_ncu.txt 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 -f \
    -o gpurun_out/prof_bwd python tools/profile_step.py > gpurun_out/prof_bwd.txt 2>&1; echo "bwd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dualkv_fwd -c 1 -f \
    -o gpurun_out/prof_fwd python tools/profile_step.py > gpurun_out/prof_fwd.txt 2>&1; echo "fwd rc=$?"
fi
