# compute-sanitizer memcheck + synccheck over the small cases with the opt-in Q-in-TMEM forward
mkdir -p gpurun_out/sanqt
for tool in memcheck synccheck; do
  DKV_FWD_QT=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanqt/$tool.txt 2>&1
  echo "$tool qt rc=$?" >> gpurun_out/sanqt/rc.txt
done
