mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc
for v in 1 2; do make variant NAME=fpw$v DEFS=-DFWD_PAIR_WAIT=$v > /dev/null 2>&1 & done; wait; cd ../..
for r in 1 2 3; do
  DKV_FWD_PAIR=0 AB_LABEL=single AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpair_ab.jsonl 2>>gpurun_out/pair_ab.err
  AB_LABEL=pair_spin AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpair_ab.jsonl 2>>gpurun_out/pair_ab.err
  for v in 1 2; do
    DKV_LIB=libdkv_fpw$v.so AB_LABEL=pair_w$v AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpair_ab.jsonl 2>>gpurun_out/pair_ab.err
  done
done
