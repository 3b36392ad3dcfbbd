timeout 600 python -m pytest tests/test_gpu_grads.py tests/test_gpu_plans.py -q 2>&1 | tail -3
timeout 300 python scratch/grads_bench.py 2>&1 | tail -3
timeout 600 python bench.py --skip-e2e --skip-cpu --steps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=d['adapter_grads']; print(round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), 'grads', round(g['ms_per_step'],1), round(g['kernel_ms_per_step'],1), round(g['achieved_gbs']), round(g['frac'],3))"
