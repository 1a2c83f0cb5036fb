mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc
for v in 4 8; do make variant NAME=poly$v DEFS=-DPAIR_POLY=$v > /dev/null 2>&1 & done; make variant NAME=ns0 DEFS=-DPAIR_NS=0 > /dev/null 2>&1 & wait
cd ../..
for r in 1 2; do
  for lib in libdkv.so libdkv_poly4.so libdkv_poly8.so libdkv_ns0.so; do
    DKV_LIB=$lib AB_REP=0 AB_LABEL=$lib timeout 300 python tools/ab.py >> gpurun_out/pair_ns.jsonl 2>>gpurun_out/pair_ab.err
  done
  DKV_BWD_PAIR=0 AB_LABEL=single AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/pair_ns.jsonl 2>>gpurun_out/pair_ab.err
done
