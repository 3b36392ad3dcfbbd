timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --skip-e2e --skip-cpu > gpurun_out/bench_graph.log 2>&1
timeout 600 python bench.py --skip-e2e --skip-cpu --graph 0 > gpurun_out/bench_eager.log 2>&1
cat gpurun_out/pytest_gpu3.log; tail -c 1500 gpurun_out/bench_graph.log; echo; tail -c 1500 gpurun_out/bench_eager.log
