timeout 400 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"seg_gemm2_kernel<\(bool\)0, \(int\)256>" -c 1 -o /tmp/p256 python scratch/cublas_vs_ours.py > /dev/null 2>&1
ncu -i /tmp/p256.ncu-rep --page raw --csv > gpurun_out/p256_raw.csv 2>/dev/null
ls -la gpurun_out/p256_raw.csv
