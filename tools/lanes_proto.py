"""Two compute lanes (prototype timing): consecutive chunks on two streams,
chunk k's layer l waiting on chunk k-1's layer l (one event per layer), so one
lane's kernel prologues/epilogue tails overlap the other lane's mainloops.
Times N chunks at prefix P on one stream vs two lanes (8B shape).

    python tools/lanes_proto.py [P=8192] [N=8] [GRAN=layer|half]"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = C.CDLL(os.path.join(ROOT, "paper_2410_03065_b200/_lib/libcake_cuda.so"))
vp = C.c_void_p


class Cfg(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("hidden", C.c_int), ("n_heads", C.c_int), ("n_kv_heads", C.c_int),
                ("head_dim", C.c_int), ("ffn", C.c_int), ("vocab", C.c_int), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float), ("page_tokens", C.c_int), ("max_chunk", C.c_int),
                ("max_tokens", C.c_longlong), ("spare_pages", C.c_int), ("tp_rank", C.c_int), ("tp_size", C.c_int),
                ("seed", C.c_ulonglong)]


P = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
Cn = 512
cfg = Cfg(32, 4096, 32, 8, 128, 14336, 128256, 500000.0, 1e-5, 64, Cn, P + N * Cn, 8, 0, 1, 42)
lib.cake_model_create.argtypes = [C.POINTER(Cfg), C.POINTER(vp)]
lib.cake_model_create_shared.argtypes = [C.POINTER(Cfg), vp, C.POINTER(vp)]
lib.cake_prefill_layers.argtypes = [vp, vp, C.c_longlong, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, vp]
ma, mb = vp(), vp()
assert lib.cake_model_create(C.byref(cfg), C.byref(ma)) == 0
assert lib.cake_model_create_shared(C.byref(cfg), ma, C.byref(mb)) == 0
torch.cuda.init()
pages = (P + N * Cn) // 64 + 8
bt = torch.arange(pages, dtype=torch.int32, device="cuda")
tok = torch.randint(0, 32000, (Cn,), dtype=torch.int32, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
L = 32


def run_seq(s):
    for k in range(N):
        assert lib.cake_prefill_layers(ma if k % 2 == 0 else mb, tok.data_ptr(), P + k * Cn, Cn, 0, L,
                                       bt.data_ptr(), None, 0, vp(s.cuda_stream)) == 0


def run_lanes(step):
    ev = [[torch.cuda.Event() for _ in range(L)] for _ in range(N)]
    for k0 in range(0, N, 2):
        for l0 in range(0, L, step):
            for k in (k0, k0 + 1):
                s, m = (sa, ma) if k % 2 == 0 else (sb, mb)
                if k > 0:
                    s.wait_event(ev[k - 1][min(L, l0 + step) - 1])
                assert lib.cake_prefill_layers(m, tok.data_ptr(), P + k * Cn, Cn, l0, min(L, l0 + step),
                                               bt.data_ptr(), None, 0, vp(s.cuda_stream)) == 0
                ev[k][min(L, l0 + step) - 1].record(s)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sa)
    sb.wait_event(e0)
    fn()
    done = torch.cuda.Event()
    done.record(sb)
    sa.wait_event(done)
    e1.record(sa)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(3):
    t_seq = timed(lambda: run_seq(sa))
    res = [f"seq {t_seq:.2f} ms ({t_seq / N:.3f}/chunk)"]
    for step in (1, 2, 4):
        t = timed(lambda: run_lanes(step))
        res.append(f"lanes(step {step}) {t:.2f} ms ({t / N:.3f}/chunk, {t_seq / t:.3f}x)")
    print(f"P={P} N={N}: " + "  ".join(res), flush=True)
