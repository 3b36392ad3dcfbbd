timeout 900 python bench.py > gpurun_out/h_13b.log 2>&1
timeout 600 python bench.py --workload 7b --skip-cpu > gpurun_out/h_7b.log 2>&1
timeout 600 python bench.py --workload 13b-decode --skip-cpu --steps 20 --warmup 5 > gpurun_out/h_dec.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/h_ref.log 2>&1
B="python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 1446 -c 6 -o /tmp/h_step_fwd $B > gpurun_out/h_ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 1686 -c 8 -o /tmp/h_step_head_bwd $B > gpurun_out/h_ncu_bwd.log 2>&1
python scratch/ncu_summary.py /tmp/h_step_fwd.ncu-rep /tmp/h_step_head_bwd.ncu-rep > gpurun_out/h_ncu_tables.md 2>&1
for f in h_13b h_7b h_dec; do tail -1 gpurun_out/$f.log | cut -c1-200; done
cat gpurun_out/h_ncu_tables.md
