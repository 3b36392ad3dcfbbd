timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pipelined" 2>&1 | tail -2
timeout 900 python bench.py --skip-cpu --steps 3 > gpurun_out/bench_e2e2.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_e2e2.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
bash scratch/r01_ncu_step.sh
