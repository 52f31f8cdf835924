"""First-token step in isolation: the q-only 1-token pass over an assembled
T-token cache + final norm + LM head (cake_final_logits, recompute=1), launched
back to back on one stream and timed with CUDA events; under ncu the launch
list gives the per-kernel split.
    T=32768 REPS=20 python tools/decode_bench.py"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200 import native  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(os.environ.get("T", "32768"))
REPS = int(os.environ.get("REPS", "20"))
preset = os.environ.get("PRESET", "llama3_8b")
rt = GpuRuntime(preset, max_tokens=T, max_chunk=512)
tier = rt.build_cache_tier(T, 512, 42)
lib = native.load()
lib.lib.cake_gpu_model.restype = ctypes.c_void_p
lib.lib.cake_gpu_model.argtypes = [ctypes.c_void_p]
model = lib.lib.cake_gpu_model(rt.h)
cl = native.load_cuda()
if os.environ.get("PREFETCH_KB") is not None:
    cl.cake_dec_set_prefetch(int(os.environ["PREFETCH_KB"]))
if os.environ.get("ATTN_WAVES") is not None:
    cl.cake_set_experiment(2, int(os.environ["ATTN_WAVES"]))  # CAKE_EXP_ATTN_MAX_WAVES
if os.environ.get("CHAIN") is not None:
    cl.cake_set_experiment(4, int(os.environ["CHAIN"]))  # CAKE_EXP_DEC_CHAIN
cl.cake_final_logits.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
if os.environ.get("IMPL"):  # e.g. tcgen05_alt: the 1-token attention on the tcgen05 kernel (before attention_q1)
    rt.set_attention_impl(os.environ["IMPL"])
r = rt.run(tier, T, 512, 42, mbps=256000, mode="io_only")
print(f"run: final step {r.final_step_ms:.3f} ms (in situ)", flush=True)
V = rt.vocab
tok = torch.tensor([7], dtype=torch.int32, device="cuda")
bt = torch.arange((T + 63) // 64, dtype=torch.int32, device="cuda")
logits = torch.empty(V, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()


def step():
    st = cl.cake_final_logits(model, T, tok.data_ptr(), 1, 0, bt.data_ptr(), logits.data_ptr(), s.cuda_stream)
    assert st == 0, st


for _ in range(3):
    step()
torch.cuda.synchronize()
import time  # noqa: E402
enq = []
for _ in range(5):  # host time to enqueue one step onto an idle stream (is the CPU ahead of the GPU?)
    t0 = time.perf_counter()
    step()
    enq.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
print(f"host enqueue of one step: {min(enq):.3f} ms (min of 5)", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / REPS
L, H, nh, nkv, hd, ffn, V = rt.dims
wbytes = 2 * L * (nh * hd * H + H * nh * hd + 3 * ffn * H) + 2 * V * H
kvbytes = T * 2 * L * nkv * hd * 2
print(f"first-token step T={T}: {ms:.3f} ms back to back; weights {wbytes/1e9:.2f} GB + KV {kvbytes/1e9:.2f} GB "
      f"-> {(wbytes + kvbytes) / (ms / 1e3) / 1e9:.0f} GB/s", flush=True)
