timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_13b.log 2>gpurun_out/bench_13b.err
timeout 900 python bench.py --workload 7b --skip-cpu > gpurun_out/bench_7b.log 2>&1
cat gpurun_out/pytest_full.log; tail -c 1200 gpurun_out/bench_13b.log; echo; tail -c 600 gpurun_out/bench_7b.log
