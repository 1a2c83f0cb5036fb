timeout 900 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/c5.txt 2>&1; echo rc=$?; tail -1 gpurun_out/c5.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['value'], d['repack_rope'])"
