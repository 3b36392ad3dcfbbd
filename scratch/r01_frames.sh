timeout 600 python -m pytest tests/test_gpu_frames.py tests/test_gpu_privacy.py -q 2>&1 | tail -15
timeout 300 python scratch/frames_bench.py 2>&1 | tail -6
