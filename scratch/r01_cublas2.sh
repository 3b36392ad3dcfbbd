timeout 900 ncu --set full --clock-control none -k regex:"nvjet|Kernel|kernel" -c 40 --csv --metrics launch__grid_size python scratch/cublas_vs_ours.py 2>&1 | grep -v "^K=" | python -c "
import sys
for l in sys.stdin:
    if 'Kernel Name' in l or 'nvjet' in l or 'gemm' in l.lower(): print(l.strip()[:300])
" | head -20
timeout 900 ncu --set full --clock-control none -k regex:"nvjet" -c 2 -o gpurun_out/cb_nvjet python scratch/cublas_vs_ours.py > gpurun_out/cb_ncu2.log 2>&1
tail -3 gpurun_out/cb_ncu2.log
