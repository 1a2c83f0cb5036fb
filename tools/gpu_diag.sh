timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bt.txt 2>&1; echo rc=$?; tail -1 gpurun_out/bt.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['replicated_ncopy']))"
