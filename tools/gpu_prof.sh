# ncu evidence for the current build: launch list of the default bench command + full captures
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --no-cpu > gpurun_out/bench_under_ncu.txt 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 -f \
    -o gpurun_out/prof_bwd python tools/profile_step.py > gpurun_out/prof_bwd.txt 2>&1; echo "bwd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dualkv_fwd -c 1 -f \
    -o gpurun_out/prof_fwd python tools/profile_step.py > gpurun_out/prof_fwd.txt 2>&1; echo "fwd rc=$?"
