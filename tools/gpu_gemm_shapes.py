"""Time the four per-chunk projection shapes (M=512) under a GEMM schedule; for ncu."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
sched = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lib.cake_gemm_set_schedule(sched)
shapes = {"qkv": (512, 6144, 4096, 256), "o": (512, 4096, 4096, 128), "gu": (512, 28672, 4096, 256), "down": (512, 4096, 14336, 128)}
for name, (M, N, K, bn) in shapes.items():
    a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(3): lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn, st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"sched={sched} {name:5s} M={M} N={N} K={K} bn={bn}: {ms*1e3:7.1f} us  {2*M*N*K/ms/1e9:7.0f} TFLOP/s", flush=True)
