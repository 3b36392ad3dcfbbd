python scratch/cublas_vs_ours.py > gpurun_out/cb3_time.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_gemm2_kernel<0, 512>|seg_gemm2_kernel" -s 4 -c 1 -o gpurun_out/cb_512 python scratch/cublas_vs_ours.py > gpurun_out/cb_ncu3.log 2>&1
cat gpurun_out/cb3_time.log; tail -2 gpurun_out/cb_ncu3.log
