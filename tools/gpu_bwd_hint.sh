# Backward MMA-issuer waits with short suspend-time hints (BWD_SPIN=ns), default and BWD_KT=1
mkdir -p gpurun_out/hint
AB_REP=0 bash tools/ab.sh hint/ab.jsonl libdkv.so libdkv_h32.so libdkv_h200.so libdkv_h1000.so libdkv_kth200.so
