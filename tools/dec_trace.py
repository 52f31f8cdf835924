"""Phase timeline of one first-token chain launch (decode_chain.cuh): every
CTA's %globaltimer at entry, after the PDL wait, and per phase at its start
(after the grid barrier), after x is staged, after its rows are streamed.
Prints, per phase, the spread of starts, the staging time and the row-stream
time (median / max over CTAs) with the phase's weight bytes and rate.
    T=32768 LAYER=5 python tools/dec_trace.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200 import native  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(os.environ.get("T", "32768"))
LAYER = int(os.environ.get("LAYER", "5"))
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
tier = rt.build_cache_tier(T, 512, 42)
lib = native.load()
lib.lib.cake_gpu_model.restype = ctypes.c_void_p
lib.lib.cake_gpu_model.argtypes = [ctypes.c_void_p]
model = lib.lib.cake_gpu_model(rt.h)
cl = native.load_cuda()
cl.cake_final_logits.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
cl.cake_dec_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
rt.run(tier, T, 512, 42, mbps=256000, mode="io_only")
tok = torch.tensor([7], dtype=torch.int32, device="cuda")
bt = torch.arange((T + 63) // 64, dtype=torch.int32, device="cuda")
logits = torch.empty(rt.vocab, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    assert cl.cake_final_logits(model, T, tok.data_ptr(), 1, 0, bt.data_ptr(), logits.data_ptr(), s.cuda_stream) == 0
buf = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
cl.cake_dec_debug_trace(buf.data_ptr(), LAYER)
assert cl.cake_final_logits(model, T, tok.data_ptr(), 1, 0, bt.data_ptr(), logits.data_ptr(), s.cuda_stream) == 0
torch.cuda.synchronize()
cl.cake_dec_debug_trace(None, -2)
tr = buf.cpu().numpy().reshape(148, 16).astype(np.float64)
t0 = tr[:, 0].min()
tr = (tr - t0) / 1e3  # us
L, H, nh, nkv, hd, F, V = rt.dims
names = ["o", "gate/up", "down", "q"]
mb = [2 * H * nh * hd, 2 * 2 * F * H, 2 * H * F, 2 * nh * hd * H]
print(f"entry spread {tr[:, 0].max():.2f} us, PDL wait done median {np.median(tr[:, 1]):.2f} max {tr[:, 1].max():.2f}")
prev_end = tr[:, 1].max()
for p in range(4):
    st, sg, rw = tr[:, 2 + 3 * p], tr[:, 3 + 3 * p], tr[:, 4 + 3 * p]
    if not st.any():
        break
    end = rw.max()
    print(f"{names[p]:8s} start {st.min():7.2f}..{st.max():7.2f} (barrier {st.max() - prev_end:5.2f} after last rows) "
          f"staged +{np.median(sg - st):5.2f} rows +{np.median(rw - sg):6.2f} (max {np.max(rw - sg):6.2f}) "
          f"end {end:7.2f}  {mb[p] / 1e6:6.1f} MB -> {mb[p] / ((end - st.min()) * 1e-6) / 1e12:5.2f} TB/s")
    prev_end = end
