mkdir -p gpurun_out/kt
for lib in libdkv_trace.so libdkv_kttr.so; do
  for cta in 0 300; do
    echo "== $lib cta $cta" >> gpurun_out/kt/trace.txt
    DKV_LIB=$lib TRACE_FN=dkv_trace_read_v1 timeout 300 python tools/trace_bwd.py $cta 16 >> gpurun_out/kt/trace.txt 2>&1
  done
done
