timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pipelined or host or channel or lockstep" 2>&1 | tail -3 > gpurun_out/pytest_host.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>gpurun_out/bench_full.err
cat gpurun_out/pytest_host.log; tail -c 3000 gpurun_out/bench_full.log; tail -3 gpurun_out/bench_full.err
