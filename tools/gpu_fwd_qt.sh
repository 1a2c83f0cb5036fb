# Q-in-TMEM pair forward (DKV_FWD_QT=1; libdkv_qt1.so: one softmax warp per row): forward-path
# parity tests, then interleaved C3 timing and a power probe.
mkdir -p gpurun_out/qt
K="fwd or forward or twocall or parity or headline or group or causal"
DKV_LIB=libdkv_qt1.so DKV_FWD_QT=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/qt/pytest_qt1.log 2>&1
tail -1 gpurun_out/qt/pytest_qt1.log
AB_REP=0 bash tools/ab_env.sh qt/ab2.jsonl "base:DKV_FWD_QT=0" "qt2w:DKV_FWD_QT=1" "qt1w:DKV_FWD_QT=1 DKV_LIB=libdkv_qt1.so"
for spec in "DKV_FWD_QT=0" "DKV_FWD_QT=1" "DKV_FWD_QT=1 DKV_LIB=libdkv_qt1.so"; do
  env $spec timeout 300 python tools/power_probe.py fwd >> gpurun_out/qt/probe2.txt 2>&1
done
