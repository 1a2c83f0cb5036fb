mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc; make variant NAME=cw16 DEFS="-DPAIR_CW=16" > /dev/null 2>&1; cd ../..
DKV_BWD_PAIR=1 DKV_LIB=libdkv_cw16.so timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twocall.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/cw_parity.log
for r in 1 2 3; do
  AB_LABEL=single AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/cw_ab.jsonl 2>>gpurun_out/pair_ab.err
  DKV_BWD_PAIR=1 AB_LABEL=pair8 AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/cw_ab.jsonl 2>>gpurun_out/pair_ab.err
  DKV_BWD_PAIR=1 DKV_LIB=libdkv_cw16.so AB_LABEL=pair16 AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/cw_ab.jsonl 2>>gpurun_out/pair_ab.err
done
