"""%globaltimer stamps inside back-to-back pair-cluster GEMMs (first and last
CTA of each launch): where the fixed per-launch cost goes.
    python tools/gemm_trace.py [N=4096] [K=4096] [bn=128] [epi=2] [launches=4]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
lib.cake_gemm_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
N, K, bn, epi, n = [int(x) for x in (sys.argv[1:] + ["4096", "4096", "128", "2", "4"][len(sys.argv) - 1:])[:5]]
M = 512
a = torch.randn(M, K, device="cuda").bfloat16()
nb = max(2, int(400e6 // (N * K * 2)) + 1)
bs = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(nb)]
c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 0 else torch.float32)
buf = torch.zeros(32 * n, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
for rep in range(3):
    lib.cake_gemm_debug_trace(ctypes.c_void_p(buf.data_ptr()) if rep == 2 else None, n)
    for i in range(n):
        lib.cake_gemm(a.data_ptr(), bs[i % nb].data_ptr(), c.data_ptr(), M, N, K, epi, bn, ctypes.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
lib.cake_gemm_debug_trace(None, 0)
t = buf.view(n, 32).cpu().numpy()
base = t[0, 0]
names = ["entry", "pdl_wait", "setup", "tma0", "full0", "mma_end", "epi_wait", "tfull", "epi_end", "sync", "exit"]
for i in range(n):
    for cta, off in (("first", 0), ("last", 16)):
        print(f"launch {i} {cta:5s} " + " ".join(f"{nm}={(t[i, off + j] - base) / 1e3:7.2f}" for j, nm in enumerate(names)))
