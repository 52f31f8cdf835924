"""Projection GEMMs at M = 512 under each dispatch variant, CUDA-graph timed,
weights rotated through > L2 worth of copies (as in the step, where every
layer's weights stream from HBM). Variants = cake_gemm_set_schedule bits:
1 stream-K, 2 no 2-SM (1-SM tiles), 4 1-SM weight-multicast clusters,
8 O/down on 1-SM N-128 tiles instead of CTA pairs.

    python tools/gemm_sweep.py [variants=0,2,6,1] [shapes=qkv,o,gu,down]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
lib.cake_gemm.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
variants = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,2,6,1").split(",")]
names = (sys.argv[2] if len(sys.argv) > 2 else "qkv,o,gu,down").split(",")
epi = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 0 bf16 store, 1 fp32 store, 2 fp32 residual add
shapes = {"qkv": (512, 6144, 4096, 256), "qkv192": (512, 6144, 4096, 192), "gu192": (512, 28416, 4096, 192), "o": (512, 4096, 4096, 128), "gu": (512, 28672, 4096, 256),
          "down": (512, 4096, 14336, 128), "o256": (512, 4096, 4096, 256), "down256": (512, 4096, 14336, 256), "o1k": (1024, 4096, 4096, 128), "qkv1k": (1024, 6144, 4096, 256)}
for name in names:
    M, N, K, bn = shapes[name]
    M = int(os.environ.get("M", M))  # e.g. M=1024: two chunks per forward
    a = torch.randn(M, K, device="cuda").bfloat16()
    nb = max(2, int(400e6 // (N * K * 2)) + 1)
    bs = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(nb)]
    c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 0 else torch.float32)
    for v in variants:
        if lib.cake_gemm_set_schedule(v) != 0:
            continue
        s = torch.cuda.Stream()
        reps = 24
        with torch.cuda.stream(s):
            for i in range(3):
                lib.cake_gemm(a.data_ptr(), bs[i % nb].data_ptr(), c.data_ptr(), M, N, K, epi, bn,
                              ctypes.c_void_p(s.cuda_stream))
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(reps):
                    lib.cake_gemm(a.data_ptr(), bs[i % nb].data_ptr(), c.data_ptr(), M, N, K, epi, bn,
                                  ctypes.c_void_p(s.cuda_stream))
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        print(f"variant={v} epi={epi} {name:5s} M={M} N={N} K={K} bn={bn}: {us:7.1f} us  {2*M*N*K/us/1e6:6.0f} TFLOP/s",
              flush=True)
    del bs
    torch.cuda.empty_cache()
lib.cake_gemm_set_schedule(0)
