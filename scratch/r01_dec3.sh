timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -4 > gpurun_out/d3_pytest.log
for i in 1 2; do
  timeout 600 python bench.py --workload 13b-decode --skip-e2e --skip-cpu --steps 20 --warmup 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('decode', round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'shrink', round(r['shrink_ms_per_step'],3), 'gather', round(r['gather_ms_per_step'],3))" >> gpurun_out/d3_time.log 2>&1
done
timeout 600 python bench.py --skip-e2e --skip-cpu --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('13b', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), 'shrink', round(r['shrink_ms_per_step'],2), 'gather', round(r['gather_ms_per_step'],2), d['clocks']['sm_mhz'])" >> gpurun_out/d3_time.log 2>&1
B="python bench.py --workload 13b-decode --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gather_rows|seg_gemm|lora_shrink|zero_kernel" -c 3300 --csv --log-file gpurun_out/d3_launches.csv $B > gpurun_out/d3_run.log 2>&1
cat gpurun_out/d3_pytest.log gpurun_out/d3_time.log
