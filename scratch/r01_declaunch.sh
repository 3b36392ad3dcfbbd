B="python bench.py --workload 13b-decode --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gather_rows|seg_gemm|lora_shrink|zero_kernel" -c 3300 --csv --log-file gpurun_out/d_launches.csv $B > gpurun_out/d_run.log 2>&1
wc -l gpurun_out/d_launches.csv
