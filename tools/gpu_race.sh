mkdir -p gpurun_out/san2
SAN_SMALL=1 timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san2/racecheck_small.txt 2>&1; echo "rc=$?" >> gpurun_out/san2/racecheck_small.txt
SAN_SMALL=1 DKV_BWD_PAIR=1 timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/san2/racecheck_small_bwdpair.txt 2>&1; echo "rc=$?" >> gpurun_out/san2/racecheck_small_bwdpair.txt
