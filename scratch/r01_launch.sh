B="python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gather_rows|seg_gemm|lora_shrink|memset" -c 6000 --csv --log-file gpurun_out/l_launches.csv $B > gpurun_out/l_run.log 2>&1
ls -la gpurun_out; wc -l gpurun_out/l_launches.csv; tail -3 gpurun_out/l_run.log
