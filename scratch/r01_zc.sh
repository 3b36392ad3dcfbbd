timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python scratch/e2e_prof.py 2>&1 | head -2
timeout 300 python bench.py --workload 13b-decode --skip-cpu --steps 20 --warmup 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode', round(d['value']), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"
