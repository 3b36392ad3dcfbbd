timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"seg_gemm2_kernel<\(bool\)0, \(int\)512>" -c 1 -o gpurun_out/cb_512b python scratch/cublas_vs_ours.py > gpurun_out/cb_ncu4.log 2>&1
tail -2 gpurun_out/cb_ncu4.log
