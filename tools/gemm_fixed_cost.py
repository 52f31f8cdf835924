"""Per-launch GEMM time vs K at a fixed tile grid (graph-captured: no host overhead)."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
for sched in (2, 8):
    lib.cake_gemm_set_schedule(sched)
    for (M, N, bn) in [(512, 4096, 128)]:
        for K in (64, 256, 1024, 2048, 4096, 8192):
            a = torch.randn(M, K, device="cuda").bfloat16()
            b = torch.randn(N, K, device="cuda").bfloat16()
            c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn, ctypes.c_void_p(s.cuda_stream))
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(20):
                        lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn,
                                      ctypes.c_void_p(s.cuda_stream))
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 20
            print(f"sched={sched} M={M} N={N} K={K:5d} bn={bn}: {us:7.1f} us/launch  {2*M*N*K/us/1e6:7.0f} TFLOP/s",
                  flush=True)
