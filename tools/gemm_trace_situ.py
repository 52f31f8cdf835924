"""%globaltimer stamps of the pair-cluster GEMMs (gemm2c: QKV and O of a layer)
INSIDE a real chunk (8B shape, chunk 20 of a 16K cache, layer 0 and 1 through
cake_prefill_layers): first and last CTA, in the PDL chain the bench runs.
    python tools/gemm_trace_situ.py"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200 import native  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = 16384
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
tier = rt.build_cache_tier(T, 512, 42)
lib = native.load()
lib.lib.cake_gpu_model.restype = ctypes.c_void_p
lib.lib.cake_gpu_model.argtypes = [ctypes.c_void_p]
model = lib.lib.cake_gpu_model(rt.h)
cl = native.load_cuda()
cl.cake_gemm_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
cl.cake_prefill_layers.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
tok = torch.randint(0, 32000, (512,), dtype=torch.int32, device="cuda")
bt = torch.arange(T // 64 + 8, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
n = 8
buf = torch.zeros(32 * n, dtype=torch.int64, device="cuda")
start = 20 * 512
for rep in range(3):
    if rep == 2:
        cl.cake_gemm_debug_trace(ctypes.c_void_p(buf.data_ptr()), n)
    assert cl.cake_prefill_layers(model, tok.data_ptr(), start, 512, 0, 3, bt.data_ptr(), None, 0, s.cuda_stream) == 0
    torch.cuda.synchronize()
cl.cake_gemm_debug_trace(None, 0)
t = buf.view(n, 32).cpu().numpy()
base = t[0, 0]
names = ["entry", "setup", "pdl", "tma0", "full0", "mma_end", "epi_pre", "tfull", "epi_end", "sync", "exit"]
for i in range(n):
    if t[i, 0] == 0:
        continue
    for cta, off in (("first", 0), ("last", 16)):
        print(f"gemm2c launch {i} {cta:5s} " + " ".join(f"{nm}={(t[i, off + j] - base) / 1e3:7.2f}" for j, nm in enumerate(names)))
