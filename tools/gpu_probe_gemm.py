"""Quick GPU probe: tcgen05 GEMM correctness + timing through the C ABI."""
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]


def err():
    buf = ctypes.create_string_buffer(1024)
    lib.cake_cuda_last_error(buf, 1024)
    return buf.value.decode()


def gemm(a, b, c, epi, bn):
    st = lib.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), a.shape[0], b.shape[0], a.shape[1], epi, bn,
                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if st != 0:
        raise RuntimeError(f"gemm status {st}: {err()}")


sched = int(os.environ.get("GEMM_SCHED", "1"))
lib.cake_gemm_set_schedule(sched)
print("schedule", sched)
torch.manual_seed(0)
ok = True
for (M, N, K) in [(128, 256, 64), (128, 128, 128), (200, 256, 512), (512, 6144, 4096), (300, 4096, 14336),
                  (1, 4096, 4096), (512, 28672, 4096)]:
    for bn in (128, 256):
        if N % bn:
            continue
        a = torch.randn(M, K, device="cuda").bfloat16()
        b = torch.randn(N, K, device="cuda").bfloat16() / K ** 0.5
        ref = a.float() @ b.float().t()
        for epi in (0, 1, 2):
            if epi == 0:
                c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            elif epi == 1:
                c = torch.empty(M, N, device="cuda", dtype=torch.float32)
            else:
                c = torch.ones(M, N, device="cuda", dtype=torch.float32)
            gemm(a, b, c, epi, bn)
            torch.cuda.synchronize()
            got = c.float() - (1.0 if epi == 2 else 0.0)
            e = (got - ref).abs().max().item()
            tol = 2e-2 * ref.abs().max().item() if epi == 0 else 1e-3 * ref.abs().max().item() + 1e-3
            flag = "OK" if e <= tol else "FAIL"
            ok &= e <= tol
            print(f"M={M} N={N} K={K} bn={bn} epi={epi}: maxerr={e:.4g} tol={tol:.3g} {flag}", flush=True)
        # timing (bf16 out)
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            gemm(a, b, c, 0, bn)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 20
        ev0.record()
        for _ in range(iters):
            gemm(a, b, c, 0, bn)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / iters
        tf = 2 * M * N * K / ms / 1e9
        # cuBLAS reference
        ev0.record()
        for _ in range(iters):
            torch.matmul(a, b.t())
        ev1.record()
        torch.cuda.synchronize()
        ms_cb = ev0.elapsed_time(ev1) / iters
        print(f"   time {ms*1e3:.1f} us  {tf:.0f} TFLOP/s   (cuBLAS {ms_cb*1e3:.1f} us {2*M*N*K/ms_cb/1e9:.0f} TFLOP/s)",
              flush=True)
print("ALL OK" if ok else "SOME FAILED")
sys.exit(0 if ok else 1)
