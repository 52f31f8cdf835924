"""Per-k-block cost of the GEMM pipelines in isolation: a few CTAs (or pairs)
with a long K, CUDA-graph timed. (M, N) pick the tile count; slope over K
gives cycles per 64-deep k-block.
    python tools/gemm_single.py"""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
clk = torch.cuda.get_device_properties(0).clock_rate / 1e6 if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1.9


def t_us(M, N, K, bn, sched):
    lib.cake_gemm_set_schedule(sched)
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn, ctypes.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn, ctypes.c_void_p(s.cuda_stream))
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / 10


import sys
cases = [("2-SM 2x256 1 pair", 256, 512, 128, 0), ("2-SM 2x256 16 pairs", 512, 4096, 128, 0),
         ("2-SM 2x256 24 pairs", 512, 6144, 256, 0), ("2-SM 256 48 pairs", 512, 6144, 256, 64),
         ("1-SM 128x128 128 CTAs", 512, 4096, 128, 64 | 2)]
for name, M, N, bn, sched in cases:
    t1, t2 = t_us(M, N, 4096, bn, sched), t_us(M, N, 12288, bn, sched)
    per_kb = (t2 - t1) / (8192 / 64)
    print(f"{name:28s}: K=4096 {t1:6.1f} us, K=12288 {t2:6.1f} us, {per_kb*1e3:6.1f} ns/k-block "
          f"(= {per_kb*1.9e3:5.0f} cyc @1.9GHz; MMA floor {128*(bn if 'x256' in name or bn==256 else 128)*64/4096:.0f})",
          flush=True)
lib.cake_gemm_set_schedule(0)
