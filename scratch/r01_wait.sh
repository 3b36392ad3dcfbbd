for v in "" scratch/variants/wait1.so scratch/variants/wait2.so; do
  echo "== lib $v" >> gpurun_out/wait_time.log
  SS_B200_LIB=$v python scratch/raster_sweep.py --shapes Q_dec,FFDOWN_dec,HEAD_dec,Q_fwd,FFDOWN_fwd --iters 10 --warm 3 --configs "pf_depth=0" >> gpurun_out/wait_time.log 2>&1
  SS_B200_LIB=$v timeout 600 python bench.py --workload 13b-decode --skip-e2e --skip-cpu --steps 20 --warmup 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('decode bench', round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'shrink', round(r['shrink_ms_per_step'],3), 'gather', round(r['gather_ms_per_step'],3))" >> gpurun_out/wait_time.log 2>&1
  SS_B200_LIB=$v timeout 600 python bench.py --skip-e2e --skip-cpu --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('13b bench', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), round(r['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/wait_time.log 2>&1
done
cat gpurun_out/wait_time.log
