mkdir -p gpurun_out
make -C paper_2605_15422_b200/csrc trace -j8 > /dev/null 2>&1
for c in 0 1; do
  DKV_BWD_PAIR=1 TRACE_FN=dkv_trace_read_pair DKV_LIB=libdkv_trace.so timeout 120 python tools/trace_bwd.py $c 24 > gpurun_out/trace_pair_$c.txt 2>&1
done
