mkdir -p gpurun_out
cd paper_2605_15422_b200/csrc; make variant NAME=ns-1 DEFS=-DPAIR_NS=-1 > /dev/null 2>&1; cd ../..
for r in 1 2; do
DKV_BWD_PAIR=0 timeout 300 python tools/power_probe.py bwd >> gpurun_out/pair_pw.txt 2>&1
DKV_LIB=libdkv_ns-1.so timeout 300 python tools/power_probe.py bwd >> gpurun_out/pair_pw.txt 2>&1
timeout 300 python tools/power_probe.py bwd >> gpurun_out/pair_pw.txt 2>&1
done
