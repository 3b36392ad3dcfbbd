timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/g_pytest.log
timeout 600 python bench.py --workload 13b-decode --skip-cpu --steps 20 --warmup 5 > gpurun_out/g_dec.log 2>&1
timeout 900 python bench.py > gpurun_out/g_13b.log 2>&1
timeout 600 python bench.py --workload 7b --skip-cpu > gpurun_out/g_7b.log 2>&1
cat gpurun_out/g_pytest.log
for f in g_dec g_13b g_7b; do tail -1 gpurun_out/$f.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', round(d['value']), round(d['ms_per_step'],2), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1), d['clocks']['sm_mhz'])"; done
