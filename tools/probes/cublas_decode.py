import torch
dev = torch.device("cuda:0")
for K, N in ((5120, 5120), (5120, 13824), (13824, 5120), (5120, 32000)):
    W = torch.randn(K, N, device=dev).to(torch.bfloat16)
    x = torch.randn(64, K, device=dev).to(torch.bfloat16)
    y = torch.empty(64, N, device=dev, dtype=torch.bfloat16)
    for _ in range(10):
        torch.matmul(x, W, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        torch.matmul(x, W, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"cuBLAS M=64 K={K} N={N}: {ms*1e3:.1f} us  {K*N*2/ms/1e6:.0f} GB/s of W")
