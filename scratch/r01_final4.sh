timeout 900 python bench.py > gpurun_out/j_13b.log 2>&1
timeout 600 python bench.py --workload 7b --skip-cpu > gpurun_out/j_7b.log 2>&1
timeout 600 python bench.py --workload 13b-decode --skip-cpu --steps 20 --warmup 5 > gpurun_out/j_dec.log 2>&1
timeout 600 python bench.py --workload granite20b --clients 64 --skip-cpu --skip-e2e > gpurun_out/j_gr.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/j_ref.log 2>&1
for f in j_13b j_7b j_dec j_gr j_ref; do tail -1 gpurun_out/$f.log | cut -c1-150; done
