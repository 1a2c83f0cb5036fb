# CTA-pair backward (opt-in, DKV_BWD_PAIR=1) vs the single-CTA default: parity subset, interleaved
# C3 A/B, trace of both CTAs of the first cluster
mkdir -p gpurun_out
DKV_BWD_PAIR=1 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twocall.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/pair_parity.log
for r in 1 2; do
  AB_LABEL=single AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/pair_ab.jsonl 2>>gpurun_out/pair_ab.err
  DKV_BWD_PAIR=1 AB_LABEL=pair AB_REP=0 timeout 300 python tools/ab.py >> gpurun_out/pair_ab.jsonl 2>>gpurun_out/pair_ab.err
done
make -C paper_2605_15422_b200/csrc trace -j8 > /dev/null 2>&1
for c in 0 1; do
  DKV_BWD_PAIR=1 TRACE_FN=dkv_trace_read_pair DKV_LIB=libdkv_trace.so timeout 120 python tools/trace_bwd.py $c 24 > gpurun_out/trace_pair_$c.txt 2>&1
done
