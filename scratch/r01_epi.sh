B="python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 1446 -c 1 -o /tmp/e_q $B > gpurun_out/e_ncu.log 2>&1
ncu -i /tmp/e_q.ncu-rep --page source --csv --print-source sass > gpurun_out/e_q_sass.csv 2>/dev/null
ncu -i /tmp/e_q.ncu-rep --page source --csv --print-source cuda > gpurun_out/e_q_cuda.csv 2>/dev/null
ls -la gpurun_out/e_q_*
