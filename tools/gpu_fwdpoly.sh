mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc
for v in 0 3 7; do make variant NAME=fp$v DEFS="-DFWD_POLY=$v" > /dev/null 2>&1 & done; wait; cd ../..
for r in 1 2 3; do
  AB_LABEL=poly5 AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpoly.jsonl 2>>gpurun_out/pair_ab.err
  for v in 0 3 7; do DKV_LIB=libdkv_fp$v.so AB_LABEL=poly$v AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/fwdpoly.jsonl 2>>gpurun_out/pair_ab.err; done
done
