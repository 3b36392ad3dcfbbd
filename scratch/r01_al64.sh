timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('decode', round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3))"; done
