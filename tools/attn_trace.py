"""Clock-stamp trace of one CTA of the product (one-tile) attention kernel:
the last chunk's layer-5 attention of a compute-only 8B tier build of T tokens.
Per 128-key block and softmax group: wait for S, TMEM load, max + exchange
(named barrier), exponentials, store + arrive; and the MMA warp's wait for P."""
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
buf = torch.zeros(64 + 3 * 64 * 8, dtype=torch.int64, device="cuda")
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
rt.set_attention_impl(os.environ.get("IMPL", "tcgen05_1tile"))
lib.cake_debug_fa4_trace(ctypes.c_void_p(buf.data_ptr()), 5)
rt.build_cache_tier(T, 512, 42)
torch.cuda.synchronize()
lib.cake_debug_fa4_trace(None, -1)
b = buf.cpu().tolist()
nb = b[1]
print(f"blocks {nb}")
tr = [[b[64 + g * 512 + j * 8: 64 + g * 512 + j * 8 + 8] for j in range(min(nb, 64))] for g in range(2)]
print("g j | waitS ldtm max+xchg exp st+arr | mma: wait-P wait-V wait-K | t")
mm = [b[64 + 1024 + j * 8: 64 + 1024 + j * 8 + 8] for j in range(min(nb, 64))]
for j in range(min(nb, 64)):
    for g in range(2):
        r = tr[g][j]
        print(f"{g} {j:3d} | {r[1]-r[0]:6d} {r[2]-r[1]:5d} {r[3]-r[2]:6d} {r[4]-r[3]:6d} {r[5]-r[4]:5d} | "
              f"{(tr[0][j][7]-tr[0][j][6]) if g == 0 else 0:6d} {(mm[j][1]-mm[j][0]) if g == 0 else 0:6d} "
              f"{(mm[j][3]-mm[j][2]) if g == 0 else 0:6d} | {r[0]-tr[0][0][0]}")
print("MMA warp: cycles issuing S(j+1) MMAs (after K wait -> before P wait) and PV(j) MMAs (after V wait -> next K wait)")
for j in range(min(nb, 64) - 2):
    s_issue = tr[0][j][6] - mm[j + 1][3]
    pv_issue = mm[j + 2][2] - mm[j][1]
    print(f"{j:3d}  S-issue {s_issue:6d}  PV-issue {pv_issue:6d}")
