timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_dec2.log
for o in "--opt a_rows64=0 --opt prefetch_mb=0 --opt l2_hints=0" "--opt prefetch_mb=0" "" "--opt prefetch_hint=0" "--opt prefetch_mb=128" "--opt prefetch_mb=32"; do
  echo "== $o" >> gpurun_out/dec2_bench.log
  timeout 600 python bench.py --workload 13b-decode --skip-e2e --skip-cpu --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'share', round(r['gemm_share_of_step'],3), 'shrink', round(r['shrink_ms_per_step'],3), 'gather', round(r['gather_ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/dec2_bench.log 2>&1
done
cat gpurun_out/pytest_dec2.log gpurun_out/dec2_bench.log
