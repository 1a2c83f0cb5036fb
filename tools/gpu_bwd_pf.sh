# Backward: L2 prefetch of Q / dO BWD_L2PF tiles ahead of the stage loads (C3, interleaved)
mkdir -p gpurun_out/pf
AB_REP=0 bash tools/ab.sh pf/ab.jsonl libdkv.so libdkv_pf3.so libdkv_pf6.so
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_active.avg
for lib in libdkv.so libdkv_pf6.so; do
  DKV_LIB=$lib ncu --metrics $M --clock-control none -k regex:dualkv_bwd -c 1 --csv --log-file gpurun_out/pf/ncu_$lib.csv python tools/profile_step.py > /dev/null 2>&1
done
