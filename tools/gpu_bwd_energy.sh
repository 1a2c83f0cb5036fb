# Backward energy ceiling: S^T / dP^T MMAs with A from TMEM (DKV_BWD_ABLATE=16, garbage operand,
# no K / V shared-memory reads) vs the real SS MMAs; ablation build without tracing
# (`make variant NAME=abl DEFS=-DDKV_ABLATION`), 60-launch power probe x3.
mkdir -p gpurun_out/be
for i in 1 2 3; do
  for a in 0 16; do
    DKV_LIB=libdkv_abl.so DKV_BWD_ABLATE=$a timeout 300 python tools/power_probe.py bwd >> gpurun_out/be/probe_abl.txt 2>&1
  done
done
