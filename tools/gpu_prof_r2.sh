#!/bin/bash
# Round-2 ncu evidence: launch list of a short default bench, full captures of both main kernels,
# and the L2 reduction / atomic counts of the backward with the atomic merge vs the ordered fold.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-replicated > gpurun_out/bench_under_ncu.txt 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 -f \
    -o gpurun_out/prof_bwd python tools/profile_step.py > gpurun_out/prof_bwd.txt 2>&1; echo "bwd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dualkv_fwd -c 1 -f \
    -o gpurun_out/prof_fwd python tools/profile_step.py > gpurun_out/prof_fwd.txt 2>&1; echo "fwd rc=$?"
M=lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed_op_global_red.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_bytes.sum
for det in 0 1; do
  DET=$det ncu --metrics $M --clock-control none -k regex:dualkv_bwd -c 1 --csv \
      --log-file gpurun_out/red_det$det.csv python tools/profile_step.py > /dev/null 2>&1; echo "red det=$det rc=$?"
done
