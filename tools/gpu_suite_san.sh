# full GPU suite (pair forward default) + compute-sanitizer over the small cases with the pair
# forward (default) and, separately, the opt-in pair backward
mkdir -p gpurun_out/san2
python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -4 > gpurun_out/san2/pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san2/$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/san2/rc.txt
  DKV_BWD_PAIR=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san2/${tool}_bwdpair.txt 2>&1
  echo "$tool bwdpair rc=$?" >> gpurun_out/san2/rc.txt
done
