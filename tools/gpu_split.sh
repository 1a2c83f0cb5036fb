mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc; make variant NAME=nosplit DEFS=-DBWD_SPLIT=0 > /dev/null 2>&1; cd ../..
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twocall.py tests/test_gpu_headline.py tests/test_gpu_gqa.py tests/test_gpu_variants.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/split_tests.log
for r in 1 2 3; do
  AB_LABEL=split AB_REP=1 timeout 300 python tools/ab.py >> gpurun_out/split_ab.jsonl 2>>gpurun_out/pair_ab.err
  DKV_LIB=libdkv_nosplit.so AB_LABEL=nosplit AB_REP=1 timeout 300 python tools/ab.py >> gpurun_out/split_ab.jsonl 2>>gpurun_out/pair_ab.err
done
