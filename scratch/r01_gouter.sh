for v in "" scratch/variants/gouter.so; do
SS_B200_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpc__cycles_elapsed.avg.per_second --clock-control none --kernel-name-base demangled -k regex:"seg_gemm2_kernel<\(bool\)0, \(int\)512>" -c 2 python scratch/cublas_vs_ours.py 2>&1 | grep -E "gpu__time|tensor_cycles"
done
for v in "" scratch/variants/gouter.so "" scratch/variants/gouter.so; do
SS_B200_LIB=$v timeout 300 python bench.py --skip-cpu --skip-e2e --steps 5 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; c=r['cublas_same_shapes']; print('[$v]', round(d['value']), round(d['ms_per_step'],1), 'gemm', round(r['achieved']), 'cublas', round(c['gemm_time_ratio'],3), d['clocks']['sm_mhz'])"
done
