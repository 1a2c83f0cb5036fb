# Shared-prompt chunk size (sequences per backward work item) vs DRAM traffic and time, C3
mkdir -p gpurun_out/chunk
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_red.sum
for c in 0 32 16 8 4; do
  DKV_CTX_CHUNK=$c ncu --metrics $M --clock-control none -k regex:dualkv_bwd -c 1 --csv \
      --log-file gpurun_out/chunk/ncu_$c.csv python tools/profile_step.py > /dev/null 2>&1; echo "chunk $c rc=$?" >> gpurun_out/chunk/rc.txt
done
AB_REP=0 bash tools/ab_env.sh chunk/ab.jsonl "c0:DKV_CTX_CHUNK=0" "c16:DKV_CTX_CHUNK=16" "c8:DKV_CTX_CHUNK=8" "c4:DKV_CTX_CHUNK=4"
