timeout 900 python bench.py > gpurun_out/f_bench_13b.log 2>&1
timeout 600 python bench.py --workload 7b --skip-cpu > gpurun_out/f_bench_7b.log 2>&1
timeout 600 python bench.py --workload 13b-decode --skip-cpu > gpurun_out/f_bench_dec.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref.log 2>&1
B="python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu --graph 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv $B > gpurun_out/f_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 1446 -c 6 -o gpurun_out/f_step_fwd $B > gpurun_out/f_ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 1686 -c 8 -o gpurun_out/f_step_head_bwd $B > gpurun_out/f_ncu_bwd.log 2>&1
ls -la gpurun_out/
