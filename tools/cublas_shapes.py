"""cuBLAS (torch.matmul) on the four per-chunk projection shapes (M=512, bf16),
CUDA-graph timed: the library reference point for the GEMM kernels."""
import os

import torch

shapes = {"qkv": (512, 6144, 4096), "o": (512, 4096, 4096), "gu": (512, 28672, 4096), "down": (512, 4096, 14336)}
for name, (M, N, K) in shapes.items():
    M = int(os.environ.get("M", M))
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    # weights larger than L2 in rotation so the weight stream comes from HBM as in the step
    nb = max(2, int(300e6 // (N * K * 2)) + 1)
    bs = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(nb)]
    for _ in range(3):
        torch.matmul(a, b.t())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.matmul(a, b.t())
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(20):
                torch.matmul(a, bs[i % nb].t())
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"cublas {name:5s} M={M} N={N} K={K}: {us:7.1f} us  {2*M*N*K/us/1e6:7.0f} TFLOP/s", flush=True)
