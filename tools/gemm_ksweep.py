"""Fixed vs per-k-block cost of the M = 512 pair GEMMs: time N x K shapes at
several K (CUDA graph of back-to-back launches, weights rotated beyond L2),
fit t = fixed + K/64 * per_kblock, next to torch (cuBLAS) on the same shapes.

    python tools/gemm_ksweep.py [N=4096] [bn=128] [epi=2] [schedules=0,256]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
bn = int(sys.argv[2]) if len(sys.argv) > 2 else 128
epi = int(sys.argv[3]) if len(sys.argv) > 3 else 2
scheds = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "0,256").split(",")]
M = 512
Ks = [1024, 2048, 4096, 8192, 14336]


def timed(fn, reps=24):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i, s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                fn(i, s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for sched in scheds + ["torch"]:
    ts = []
    for K in Ks:
        a = torch.randn(M, K, device="cuda").bfloat16()
        nb = max(2, int(400e6 // (N * K * 2)) + 1)
        bs = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(nb)]
        if sched == "torch":
            c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            us = timed(lambda i, s: torch.matmul(a, bs[i % nb].t(), out=c))
        else:
            lib.cake_gemm_set_schedule(sched)
            c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 0 else torch.float32)
            us = timed(lambda i, s: lib.cake_gemm(a.data_ptr(), bs[i % nb].data_ptr(), c.data_ptr(), M, N, K, epi, bn,
                                                  ctypes.c_void_p(s.cuda_stream)))
        ts.append(us)
        del bs
        torch.cuda.empty_cache()
    kb = np.array(Ks) / 64
    slope, fixed = np.polyfit(kb, ts, 1)
    print(f"sched={sched} N={N} bn={bn} epi={epi}: " + " ".join(f"K{K}={t:.1f}" for K, t in zip(Ks, ts)) +
          f" | fixed {fixed:.2f} us, per k-block {slope*1e3:.0f} ns", flush=True)
lib.cake_gemm_set_schedule(0)
