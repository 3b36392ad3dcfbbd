timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('decode', round(d['value']), round(d['ms_per_step'],3), 'shrink', round(r['shrink_ms_per_step'],3), 'launches', d['gpu_launches'])"
timeout 300 python bench.py --skip-cpu --skip-e2e --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('13b', round(d['value']), round(d['ms_per_step'],1), 'shrink', round(r['shrink_ms_per_step'],2), d['clocks']['sm_mhz'])"
