python scratch/cublas_vs_ours.py > gpurun_out/cb_time.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm|xmma|cutlass|seg_gemm|sm100" -s 2 -c 4 -o gpurun_out/cb_q python scratch/cublas_vs_ours.py > gpurun_out/cb_ncu.log 2>&1
cat gpurun_out/cb_time.log; tail -5 gpurun_out/cb_ncu.log
