"""Clock-stamp trace of one CTA of the two-tile attention kernel (debug).
Runs an 8B-shape compute-only tier build of T tokens; the trace keeps the last
chunk's layer-5 attention (prefix T - 512)."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200 import native  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(os.environ.get("T", "8192"))
lib = native.load_cuda()
buf = torch.zeros(64 + 2 * 64 * 8, dtype=torch.int64, device="cuda")
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
rt.set_attention_impl(os.environ.get("IMPL", "tcgen05_2tile"))
lib.cake_debug_fa4_trace(ctypes.c_void_p(buf.data_ptr()), int(os.environ.get("LAYER", "5")))
rt.build_cache_tier(T, 512, 42)
torch.cuda.synchronize()
lib.cake_debug_fa4_trace(None, -1)
b = buf.cpu().tolist()
t0, nb = b[0], b[1]
print(f"blocks {nb}")
h = b[2:9]
print("entry->pdl_wait %d | ->mma start %d | ->softmax loop end %d | epilogue %d | ticket %d | combine %d | teardown %d"
      % (h[1] - h[0], t0 - h[1], h[2] - t0, h[3] - h[2], h[4] - h[3], h[5] - h[4], h[6] - h[5]))
tr = [[b[64 + i * 512 + j * 8: 64 + i * 512 + j * 8 + 8] for j in range(min(nb, 64))] for i in range(2)]
print("tile j | softmax: waitS ldtm max exp st+arr | mma: pv-wait-P  (cycles; start rel. to first S wait)")
for j in range(min(nb, 64)):
    for i in range(2):
        r = tr[i][j]
        print(f"{i} {j:3d} | {r[1]-r[0]:6d} {r[2]-r[1]:5d} {r[3]-r[2]:5d} {r[4]-r[3]:6d} {r[5]-r[4]:5d} | "
              f"{r[7]-r[6]:6d}   t={r[0]-tr[0][0][0]}")
