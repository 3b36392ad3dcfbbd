timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for w in 13b 7b; do
timeout 300 python bench.py --workload $w --skip-cpu --skip-e2e --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; c=r['cublas_same_shapes']; print('$w', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), 'cublas', round(c['ms_per_step'],1), round(c['gemm_time_ratio'],3), d['clocks']['sm_mhz'])"
done
