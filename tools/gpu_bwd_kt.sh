# K-in-TMEM backward variants (BWD_KT=1; issuer waits: kt suspend, kt1 spin, kt2 try_wait no hint)
mkdir -p gpurun_out/kt
AB_REP=0 bash tools/ab.sh kt/ab2.jsonl libdkv.so libdkv_kt.so libdkv_kt1.so libdkv_kt2.so
for lib in libdkv.so libdkv_kt1.so libdkv_kt2.so; do DKV_LIB=$lib timeout 300 python tools/power_probe.py bwd >> gpurun_out/kt/probe2.txt 2>&1; done
