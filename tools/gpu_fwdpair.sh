mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc
for h in 100 400 1500; do make variant NAME=fh$h DEFS=-DFWD_PAIR_HINT=$h > /dev/null 2>&1 & done; wait; cd ../..
for r in 1 2 3; do
  AB_LABEL=default AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpair_ab.jsonl 2>>gpurun_out/pair_ab.err
  DKV_FWD_PAIR=1 AB_LABEL=fwdpair AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpair_ab.jsonl 2>>gpurun_out/pair_ab.err
  for h in 100 400 1500; do
    DKV_LIB=libdkv_fh$h.so DKV_FWD_PAIR=1 AB_LABEL=fwdpair_h$h AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpair_ab.jsonl 2>>gpurun_out/pair_ab.err
  done
done
