"""B200 bidirectional KV generator — Python handle on the native GpuContext.

    rt = GpuRuntime(PRESETS["llama3_8b"], max_tokens=32768)
    tier = rt.build_cache_tier(32768, 512, prompt_seed=42)      # pinned host DRAM tier
    res = rt.run(tier, 32768, 512, prompt_seed=42, mbps=64000, mode="cake")
    res.first_token_ms, res.merge_point, rt.logits()

Everything runs in libcake.so / libcake_cuda.so (C++ host runtime + sm_100a
kernels); there is no Python or CPU fallback — a missing library raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import native as N
from .cake import MODES, BandwidthTrace, ChunkStore, _opts, _records


def _cuda_error(cu) -> str:
    buf = C.create_string_buffer(512)
    cu.cake_cuda_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")

PRESETS = {
    # name: (n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab)
    "llama3_8b": (32, 4096, 32, 8, 128, 14336, 128256),
    "llama3_70b": (80, 8192, 64, 8, 128, 28672, 128256),
    "tiny": (2, 256, 4, 4, 64, 1024, 32000),
}


@dataclass
class GpuResult:
    mode: str
    kv_resident_ms: float
    first_token_ms: float
    final_step_ms: float
    device_ttft_ms: float
    merge_point: int
    n_chunks: int
    raced_chunk: int
    race_winner: int
    recomputed_last: bool
    kernel_launches: int
    h2d_bytes: int
    d2h_bytes: int
    compute_busy_ms: float
    io_busy_ms: float
    chunks: list = field(default_factory=list)


class Link:
    """One emulated cache-tier link shared by several GpuRuntimes (concurrent
    requests on one device): together their loaders deliver at the trace rate;
    the trace's time axis is the link's clock (t = 0 at creation / reset())."""

    def __init__(self, trace: BandwidthTrace | None = None, *, mbps: float | None = None):
        self.n = N.load()
        trace = trace or BandwidthTrace.constant(mbps)
        t, self._keep = trace.native()
        h = N.vp()
        self.n.call("cake_link_create", t, C.byref(h))
        self.h = h.value

    def reset(self):
        self.n.call("cake_link_reset", self.h)

    def reserved(self) -> tuple[int, int]:
        """(bits reserved so far, link clock in us)."""
        b, t = N.u64(), N.i64()
        self.n.call("cake_link_reserved_bits", self.h, C.byref(b), C.byref(t))
        return b.value, t.value

    def close(self):
        if getattr(self, "h", None):
            self.n.lib.cake_link_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GpuRuntime:
    def __init__(self, preset, *, n_layers: int | None = None, max_chunk: int = 512, max_tokens: int = 32768,
                 weight_seed: int = 1234, device: int = 0, tp_rank: int = 0, tp_size: int = 1, nccl_comm=None,
                 lookahead_layers: int = 0, profile_kernels: bool = False, race_margin_us: int = 0,
                 rope_theta: float = 500000.0, rms_eps: float = 1e-5, tp_shm: str | None = None,
                 compute_sms: int = 0, weights_from: "GpuRuntime | None" = None):
        self.n = N.load()
        dims = PRESETS[preset] if isinstance(preset, str) else tuple(preset)
        L, H, nh, nkv, hd, ffn, vocab = dims
        if n_layers is not None:
            L = n_layers
        self.dims = (L, H, nh, nkv, hd, ffn, vocab)
        cfg = N.CakeGpuConfig(L, H, nh, nkv, hd, ffn, vocab, rope_theta, rms_eps, max_chunk, max_tokens,
                              weight_seed, device, tp_rank, tp_size, nccl_comm, lookahead_layers,
                              1 if profile_kernels else 0, race_margin_us,
                              tp_shm.encode() if tp_shm else None, compute_sms,
                              weights_from.h if weights_from is not None else None)
        h = N.vp()
        self.n.call("cake_gpu_create", C.byref(cfg), C.byref(h))
        self.h = h.value
        self.vocab = vocab
        self.max_chunk = max_chunk
        self._parent = weights_from  # shared weights: the parent context must outlive this one
        self._link = None

    def tp_peer_handles(self) -> bytes:
        """This rank's CUDA IPC handles of its TP exchange buffers (peer-memory reduction)."""
        cu = N.load_cuda()
        buf = (C.c_uint8 * N.TP_PEER_HANDLE_BYTES)()
        if cu.cake_tp_peer_handles(self.n.lib.cake_gpu_model(self.h), buf, len(buf)) != 0:
            raise RuntimeError(f"cake_tp_peer_handles: {_cuda_error(cu)}")
        return bytes(buf)

    def tp_peer_open(self, handles: list) -> None:
        """Map every rank's exchange buffers (handles in rank order, this rank's included)."""
        cu = N.load_cuda()
        blob = b"".join(handles)
        if len(blob) != N.TP_PEER_HANDLE_BYTES * len(handles):
            raise ValueError("tp_peer_open: bad handle blobs")
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        if cu.cake_tp_peer_open(self.n.lib.cake_gpu_model(self.h), buf, len(handles)) != 0:
            raise RuntimeError(f"cake_tp_peer_open: {_cuda_error(cu)}")

    def close(self):
        if getattr(self, "h", None):
            self.n.lib.cake_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def attach_link(self, link: "Link | None"):
        """Pace later runs' loads through `link` (shared with other contexts) instead of
        their own trace; None detaches."""
        self.n.call("cake_gpu_set_link", self.h, link.h if link is not None else None)
        self._link = link

    @property
    def kv_bytes_per_token(self) -> int:
        out = N.u64()
        self.n.call("cake_gpu_kv_bytes_per_token", self.h, C.byref(out))
        return out.value

    def new_tier(self) -> ChunkStore:
        return ChunkStore(self.n, None, 2, pinned=True)

    def build_cache_tier(self, total_tokens: int, chunk_size: int, prompt_seed: int,
                         store: ChunkStore | None = None) -> ChunkStore:
        store = store or self.new_tier()
        self.n.call("cake_gpu_build_tier", self.h, store.h, total_tokens, chunk_size, prompt_seed)
        return store

    def set_codec(self, codec: str = "identity"):
        """Cache-tier codec for build_cache_tier and run: "identity" | "quant8"
        (reference codec.cpp:114-162; the GPU decodes inside the scatter)."""
        self.n.call("cake_gpu_set_codec", self.h, codec.encode())
        self.codec = codec

    def calibrate(self, total_tokens: int, chunk_size: int, prompt_seed: int):
        a, b = N.dbl(), N.dbl()
        self.n.call("cake_gpu_calibrate", self.h, total_tokens, chunk_size, prompt_seed, C.byref(a), C.byref(b))
        return a.value, b.value

    def run(self, store: ChunkStore, total_tokens: int, chunk_size: int, prompt_seed: int, *,
            mbps: float | None = None, trace: BandwidthTrace | None = None, mode: str = "cake",
            race: bool = True, quantum: int = 1 << 20, **opts) -> GpuResult:
        trace = trace or BandwidthTrace.constant(mbps)
        t, keep = trace.native()
        n = -(-total_tokens // chunk_size)
        recs = (N.CakeRecord * n)()
        res = N.CakeGpuResult()
        o = _opts(self.n, race_to_finish=race, throttle_quantum_bytes=quantum, token_budget=max(512, chunk_size),
                  **opts)
        self.n.call("cake_gpu_run", self.h, store.h, total_tokens, chunk_size, prompt_seed, t, MODES[mode],
                    C.byref(o), C.byref(res), recs)
        return GpuResult(mode, res.kv_resident_us / 1e3, res.first_token_us / 1e3, res.final_step_us / 1e3,
                         res.device_ttft_ms, res.merge_point, res.n_chunks, res.raced_chunk, res.race_winner,
                         bool(res.recomputed_last), res.kernel_launches, res.h2d_bytes, res.d2h_bytes,
                         res.compute_busy_us / 1e3, res.io_busy_us / 1e3, _records(recs, n))

    def logits(self) -> np.ndarray:
        out = np.empty(self.vocab, dtype=np.float32)
        self.n.call("cake_gpu_logits", self.h, out.ctypes.data, self.vocab)
        return out

    def poison(self, byte: int = 0xFF):
        """Test instrumentation: fill the paged KV pool (both page sets) and the
        device staging buffers with `byte` (0xFF = bf16 NaN) so a later run must
        write every page its block table references."""
        self.n.call("cake_gpu_poison", self.h, byte)

    def slices(self) -> tuple[np.ndarray, np.ndarray]:
        """Slice log of the last run (record_slices=True): (release time on the
        run clock in us, cumulative released bits) — reference transfer.hpp SliceEvent."""
        n = N.u64()
        self.n.call("cake_gpu_slices", self.h, None, None, 0, C.byref(n))
        at = np.zeros(n.value, dtype=np.int64)
        bits = np.zeros(n.value, dtype=np.uint64)
        if n.value:
            self.n.call("cake_gpu_slices", self.h, at.ctypes.data_as(C.POINTER(N.i64)),
                        bits.ctypes.data_as(C.POINTER(N.u64)), n.value, C.byref(n))
        return at, bits

    def read_chunk(self, token_start: int, token_count: int) -> bytes:
        L, H, nh, nkv, hd, ffn, vocab = self.dims
        nbytes = self.kv_bytes_per_token * token_count
        out = C.create_string_buffer(nbytes)
        self.n.call("cake_gpu_read_chunk", self.h, token_start, token_count, out, nbytes)
        return out.raw

    def set_attention_impl(self, impl: str):
        """"tcgen05" (product dispatch: softmax warpgroups on alternate key blocks),
        "tcgen05_1tile" (the column-split one-tile kernel), "mma_sync" (independent
        cross-check kernel); "tcgen05_2tile" / "tcgen05_dec" need an ATTN_VARIANTS=1 build."""
        self.n.call("cake_gpu_set_attention_impl", self.h,
                    {"tcgen05": 0, "mma_sync": 1, "tcgen05_1tile": 2, "tcgen05_2tile": 3,
                     "tcgen05_dec": 4, "tcgen05_alt": 5}[impl])

    def set_profiling(self, kernels="all", stride: int = 1):
        """Bracket launches of the named kernel classes with CUDA events ("all", None, or a list);
        stride n brackets every n-th launch of a class only."""
        self.n.call("cake_gpu_set_profiling_stride", self.h, stride)
        if kernels == "all":
            mask = -1
        elif not kernels:
            mask = 0
        else:
            mask = sum(1 << N.KERNEL_NAMES.index(k) for k in kernels)
        self.n.call("cake_gpu_set_profiling", self.h, mask)

    def kernel_stats(self, reset: bool = True) -> dict:
        arr = (N.CakeKernelStat * len(N.KERNEL_NAMES))()
        self.n.call("cake_gpu_kernel_stats", self.h, arr, 1 if reset else 0)
        return {name: {"launches": arr[i].launches, "ms": arr[i].total_ms, "flops": arr[i].flops,
                       "bytes": arr[i].bytes} for i, name in enumerate(N.KERNEL_NAMES)}
