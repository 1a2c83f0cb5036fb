mkdir -p gpurun_out
DKV_BWD_PAIR=1 ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 -f \
    -o gpurun_out/prof_bwd_pair2 python tools/profile_step.py > gpurun_out/prof_bwd_pair2.txt 2>&1; echo "pair rc=$?"
