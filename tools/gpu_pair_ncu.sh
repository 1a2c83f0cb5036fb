mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 -f \
    -o gpurun_out/prof_bwd_pair python tools/profile_step.py > gpurun_out/prof_bwd_pair.txt 2>&1; echo "pair rc=$?"
DKV_BWD_PAIR=0 ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 -f \
    -o gpurun_out/prof_bwd_single python tools/profile_step.py > gpurun_out/prof_bwd_single.txt 2>&1; echo "single rc=$?"
