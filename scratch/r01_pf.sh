python scratch/raster_sweep.py --shapes Q_dec,FFUP_dec,FFDOWN_dec,HEAD_dec --iters 20 --warm 3 --configs "a_rows64=0;pf_depth=0;pf_depth=4;pf_depth=8;pf_depth=16;pf_depth=32;pf_depth=16,l2_hints=0" > gpurun_out/pf_time.log 2>&1
for o in "" "--opt pf_depth=8" "--opt pf_depth=16" "--opt pf_depth=32"; do
  echo "== $o" >> gpurun_out/pf_bench.log
  timeout 600 python bench.py --workload 13b-decode --skip-e2e --skip-cpu --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'share', round(r['gemm_share_of_step'],3), 'shrink', round(r['shrink_ms_per_step'],3), 'gather', round(r['gather_ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/pf_bench.log 2>&1
done
cat gpurun_out/pf_time.log gpurun_out/pf_bench.log
