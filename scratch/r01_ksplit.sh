timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 300 python scratch/grads_bench.py 2>&1 | tail -2
timeout 600 python bench.py --workload 13b-decode --skip-cpu --skip-e2e --steps 20 --warmup 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('decode', round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'share', round(r['gemm_share_of_step'],3), 'shrink', round(r['shrink_ms_per_step'],3))"
timeout 600 python bench.py --skip-e2e --skip-cpu --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=d['adapter_grads']; print('13b', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), 'shrink', round(r['shrink_ms_per_step'],2), 'grads', round(g['ms_per_step'],1), round(g['achieved_gbs']))"
