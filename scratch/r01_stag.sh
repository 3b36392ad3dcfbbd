timeout 120 python scratch/cublas_vs_ours.py 2>&1 | tail -6; echo rc=$?
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "every_kernel or tma_store or batched or large_layer" 2>&1 | tail -2
for o in "" "--opt pair_n=256" ""; do
timeout 300 python bench.py --skip-cpu --skip-e2e --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; c=r['cublas_same_shapes']; print('[$o]', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), 'cublas', round(c['ms_per_step'],1), round(c['gemm_time_ratio'],3), d['clocks']['sm_mhz'])"
done
