timeout 900 python -m pytest tests/test_gpu_grads.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_grads2.log
timeout 300 python scratch/grads_bench.py > gpurun_out/grads_bench2.log 2>&1
timeout 120 python scratch/pcie.py > gpurun_out/pcie.log 2>&1
cat gpurun_out/pytest_grads2.log gpurun_out/grads_bench2.log gpurun_out/pcie.log
