timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_hints.log
for rep in 1 2; do
for o in "--opt l2_hints=0" "" "--opt raster=-1" "--opt raster=-1 --opt l2_budget_mb=96"; do
  echo "== $o" >> gpurun_out/hints_bench.log
  timeout 600 python bench.py --skip-e2e --skip-cpu --steps 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/hints_bench.log 2>&1
done; done
cat gpurun_out/pytest_hints.log gpurun_out/hints_bench.log
