mkdir -p gpurun_out
make -C paper_2605_15422_b200/csrc trace -j8 > /dev/null 2>&1
for c in 0 1; do DKV_LIB=libdkv_trace.so timeout 120 python tools/trace_fwd.py $c 12 > gpurun_out/trace_fwdpair_$c.txt 2>&1; done
DKV_FWD_PAIR=0 DKV_LIB=libdkv_trace.so timeout 120 python tools/trace_fwd.py 0 12 > gpurun_out/trace_fwdsingle_0.txt 2>&1
