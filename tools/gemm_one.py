"""Launch one projection shape N times (for ncu --set full)."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
name, sched, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
lib.cake_gemm_set_schedule(sched)
M, N, K, bn = {"qkv": (512, 6144, 4096, 256), "o": (512, 4096, 4096, 128), "gu": (512, 28672, 4096, 256),
               "down": (512, 4096, 14336, 128)}[name]
a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
c = torch.zeros(M, N, device="cuda", dtype=torch.float32)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(n):
    lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 2, bn, st)
torch.cuda.synchronize()
