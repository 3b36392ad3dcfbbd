set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_13b.log 2>gpurun_out/bench_13b.err
timeout 600 python bench.py --workload 13b-decode --skip-cpu > gpurun_out/bench_13bdec.log 2>&1
timeout 600 python bench.py --workload 7b --skip-cpu > gpurun_out/bench_7b.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench_13b.log; echo; tail -c 800 gpurun_out/bench_13bdec.log; echo; tail -c 600 gpurun_out/bench_7b.log; tail -c 600 gpurun_out/bench_ref.log
