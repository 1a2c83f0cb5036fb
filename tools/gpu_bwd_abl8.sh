# Backward: cost of the two K=16 additive-constant MMAs per tile (DKV_BWD_ABLATE=8, timing only)
mkdir -p gpurun_out/be
for i in 1 2 3; do
  for a in 0 8; do
    DKV_LIB=libdkv_abl.so DKV_BWD_ABLATE=$a timeout 300 python tools/power_probe.py bwd >> gpurun_out/be/probe_abl8.txt 2>&1
  done
done
