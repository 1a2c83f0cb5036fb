mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc
make trace -j8 > /dev/null 2>&1
cp ../libdkv_trace.so ../libdkv_tr_base.so
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I. -I../../include -DDKV_TRACE -DDKV_ABLATION -DPAIR_TRACE_NLOAD -c bwd_pair_sm100.cu -o build_trace/bwd_pair_nored.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../libdkv_tr_nored.so $(ls build_trace/*.o | grep -v "bwd_pair_sm100.o")
cd ../..
for lib in tr_base tr_nored; do
  for c in 0 1; do
    TRACE_FN=dkv_trace_read_pair DKV_LIB=libdkv_$lib.so timeout 120 python tools/trace_bwd.py $c 24 > gpurun_out/trace_${lib}_$c.txt 2>&1
  done
done
