timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -4 > gpurun_out/p_pytest.log
for o in "--opt pdl=0" "" "--opt pdl=0" ""; do
  timeout 600 python bench.py --workload 13b-decode --skip-e2e --skip-cpu --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('decode [$o]', round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'launches', d['gpu_launches'])" >> gpurun_out/p_time.log 2>&1
done
for o in "--opt pdl=0" ""; do
  timeout 600 python bench.py --skip-e2e --skip-cpu --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('13b [$o]', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/p_time.log 2>&1
done
cat gpurun_out/p_pytest.log gpurun_out/p_time.log
