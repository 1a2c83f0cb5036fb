# compute-sanitizer passes over small two-call fwd+bwd cases (memcheck, racecheck, synccheck)
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_case.py \
    > gpurun_out/sanitize/$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize/$tool.txt
done
