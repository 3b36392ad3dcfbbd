B="python bench.py --workload 13b-decode --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
# decode step: block 0's dispatches (gather, zero, shrink, streaming GEMM) after 3 warm-up steps (802 launches each)
timeout 900 ncu --set full --clock-control none -k regex:"gather_rows|zero_kernel|lora_shrink|seg_gemm" -s 2406 -c 14 -o /tmp/k_dec $B > gpurun_out/k_dec.log 2>&1
B2="python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 900 ncu --set full --clock-control none -k regex:"gather_rows|lora_shrink" -s 60 -c 6 -o /tmp/k_13b $B2 > gpurun_out/k_13b.log 2>&1
python scratch/ncu_summary.py /tmp/k_dec.ncu-rep /tmp/k_13b.ncu-rep > gpurun_out/k_tables.md 2>&1
cat gpurun_out/k_tables.md
