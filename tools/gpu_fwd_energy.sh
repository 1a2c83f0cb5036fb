# Forward energy experiment: the pair forward's S MMA with A from TMEM (DKV_FWD_ABLATE=8, garbage
# operand, no Q shared-memory reads) vs the real SS MMA, trace build, 60-launch power probe x3.
mkdir -p gpurun_out/fe
for i in 1 2 3; do
  for a in 0 8; do
    DKV_LIB=libdkv_trace.so DKV_FWD_ABLATE=$a timeout 300 python tools/power_probe.py fwd >> gpurun_out/fe/probe.txt 2>&1
  done
done
