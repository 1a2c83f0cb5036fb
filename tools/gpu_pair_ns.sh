# pair backward: per-role wait policy (C: compute warps, I: issuers + forwarder), -1 = suspend
mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc
make variant NAME=w_i0 DEFS="-DPAIR_NS_I=0" > /dev/null 2>&1 &
make variant NAME=w_i0_c64 DEFS="-DPAIR_NS_I=0 -DPAIR_NS_C=64" > /dev/null 2>&1 &
make variant NAME=w_c64 DEFS="-DPAIR_NS_C=64" > /dev/null 2>&1 &
make variant NAME=w_i32 DEFS="-DPAIR_NS_I=32" > /dev/null 2>&1 &
wait; cd ../..
for r in 1 2; do
  AB_LABEL=single AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/pair_ns2.jsonl 2>>gpurun_out/pair_ab.err
  DKV_BWD_PAIR=1 AB_LABEL=pair_default AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/pair_ns2.jsonl 2>>gpurun_out/pair_ab.err
  for v in w_i0 w_i0_c64 w_c64 w_i32; do
    DKV_BWD_PAIR=1 DKV_LIB=libdkv_$v.so AB_LABEL=$v AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/pair_ns2.jsonl 2>>gpurun_out/pair_ab.err
  done
done
