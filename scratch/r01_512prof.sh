timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"seg_gemm2_kernel<\(bool\)0, \(int\)512>" -c 1 -o /tmp/p512 python scratch/cublas_vs_ours.py > /dev/null 2>&1
ncu -i /tmp/p512.ncu-rep --page source --csv --print-source sass > gpurun_out/p512_sass.csv 2>/dev/null
ncu -i /tmp/p512.ncu-rep --page raw --csv > gpurun_out/p512_raw.csv 2>/dev/null
ls -la gpurun_out/p512_*
