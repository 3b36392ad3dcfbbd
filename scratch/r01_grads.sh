set -x
timeout 900 python -m pytest tests/test_gpu_grads.py -x -q 2>&1 | tail -25 > gpurun_out/pytest_grads.log
timeout 300 python scratch/grads_bench.py > gpurun_out/grads_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lora_grad|ia3_grad|lora_shrink" -s 6 -c 4 -o gpurun_out/grads_full python scratch/grads_bench.py > gpurun_out/ncu_grads.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_gemm2_kernel" -s 40 -c 2 -o gpurun_out/gemm2_full python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/ncu_gemm.log 2>&1
cat gpurun_out/pytest_grads.log gpurun_out/grads_bench.log; tail -5 gpurun_out/ncu_grads.log gpurun_out/ncu_gemm.log
