timeout 60 python scratch/cublas_vs_ours.py 2>&1 | tail -6
echo "rc=$?"
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "every_kernel or tma_store or batched" 2>&1 | tail -3
