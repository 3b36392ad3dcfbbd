timeout 600 python -m pytest tests -q -m gpu -x -k "host or rejected or in_place or decode" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --workload 13b-decode --skip-cpu --steps 10 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1))"; done
