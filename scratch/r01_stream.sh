timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -4 > gpurun_out/s_pytest.log
python scratch/raster_sweep.py --shapes Q_dec,FFUP_dec,FFDOWN_dec,HEAD_dec --iters 20 --warm 3 --configs "stream_gemm=0;stream_gemm=1" > gpurun_out/s_time.log 2>&1
for o in "--opt stream_gemm=0" ""; do
  timeout 600 python bench.py --workload 13b-decode --skip-e2e --skip-cpu --steps 20 --warmup 5 $o 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$o]', round(d['value']), round(d['ms_per_step'],3), 'gemm', round(r['achieved']), r['unit'], round(r['frac'],3), 'share', round(r['gemm_share_of_step'],3), 'shrink', round(r['shrink_ms_per_step'],3), 'gather', round(r['gather_ms_per_step'],3))" >> gpurun_out/s_time.log 2>&1
done
cat gpurun_out/s_pytest.log gpurun_out/s_time.log
