"""Python mirror of the reference's cake:: interface for the hot path.

Names, argument meaning and error behaviour follow the reference headers
(proj/include/cake/{model,scheduler,store,codec,report}.hpp); every call goes
through the C ABI of a native library (`native.load()` = the B200 runtime).
Passing `lib=native.load(native.REF_LIB)` binds the same calls to the reference
built from source — that is how tests/test_parity_ref.py compares the two.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import native as N

MODES = {"cake": 0, "compute_only": 1, "io_only": 2}
SIDES = {0: "compute", 1: "io"}


@dataclass
class CostModel:
    alpha_ms: float = 0.0
    beta_ms_per_token: float = 0.0
    reference_chunk_size: int = 512


@dataclass
class BandwidthTrace:
    points: list  # [(at_us, mbps)]

    @staticmethod
    def constant(mbps: float) -> "BandwidthTrace":
        return BandwidthTrace([(0, float(mbps))])

    def native(self):
        return N.make_trace(self.points)


@dataclass
class ChunkRecord:
    index: int
    side: str
    start_us: int
    finish_us: int
    bytes: int


@dataclass
class RunReport:
    mode: str
    n_chunks: int
    ttft_us: int
    merge_point: int
    computed_fraction: float
    compute_busy_us: int
    io_busy_us: int
    chunks: list = field(default_factory=list)

    def event_csv(self) -> str:  # reference report.cpp:31-37 format
        rows = ["index,side,start_us,finish_us,bytes"]
        rows += [f"{r.index},{r.side},{r.start_us},{r.finish_us},{r.bytes}" for r in self.chunks]
        return "\n".join(rows) + "\n"

    def summary_line(self) -> str:  # reference report.cpp:45-52 format
        return f"{self.mode},{self.n_chunks},{self.ttft_us},{self.merge_point},{self.computed_fraction:.6f}"


@dataclass
class RunPlan:
    token_starts: list
    token_counts: list
    encoded_bytes: list
    uncompressed_bytes: list

    @property
    def n(self) -> int:
        return len(self.token_starts)


def _records(recs, n) -> list:
    return [ChunkRecord(recs[i].index, SIDES[recs[i].side], recs[i].start_us, recs[i].finish_us, recs[i].bytes)
            for i in range(n)]


def _opts(lib: N.Native, **kw) -> N.CakeRunOpts:
    o = N.CakeRunOpts()
    lib.lib.cake_run_opts_default(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown run option {k}")
        if k == "link":
            v = v.h if v is not None else None  # a runtime.Link
        setattr(o, k, v if v is None or isinstance(v, float) else int(v))
    return o


class Cake:
    """The cost laws, simulator, oracle, cache tier and codecs of one library."""

    def __init__(self, lib: N.Native | None = None):
        self.n = lib or N.load()

    # ---- cost laws (model.hpp)
    def time_to_transfer_bits(self, trace: BandwidthTrace, bits: int, start_us: int = 0) -> int:
        t, keep = trace.native()
        out = N.i64()
        self.n.call("cake_time_to_transfer_bits", t, bits, start_us, C.byref(out))
        return out.value

    def fetch_latency(self, trace: BandwidthTrace, nbytes: int, start_us: int = 0) -> int:
        t, keep = trace.native()
        out = N.i64()
        self.n.call("cake_fetch_latency", t, nbytes, start_us, C.byref(out))
        return out.value

    def compute_latency(self, cost: CostModel, token_start: int, token_count: int, power: float = 1.0) -> int:
        out = N.i64()
        self.n.call("cake_compute_latency", cost.alpha_ms, cost.beta_ms_per_token, cost.reference_chunk_size,
                    token_start, token_count, power, C.byref(out))
        return out.value

    def kv_bytes_per_token(self, n_layers, hidden, precision, kv_multiplier=2, override=0) -> int:
        out = N.u64()
        self.n.call("cake_kv_bytes_per_token", n_layers, hidden, precision, kv_multiplier, override, C.byref(out))
        return out.value

    def split_into_chunks(self, total_tokens: int, chunk_size: int):
        n = N.u32()
        self.n.call("cake_split_into_chunks", total_tokens, chunk_size, C.byref(n), None, None, 0)
        starts = (N.u64 * n.value)()
        counts = (N.u32 * n.value)()
        self.n.call("cake_split_into_chunks", total_tokens, chunk_size, C.byref(n), starts, counts, n.value)
        return list(zip(starts, counts))

    def oracle_best_split(self, compute_us: Sequence[int], fetch_us: Sequence[int]):
        c = (N.i64 * max(1, len(compute_us)))(*compute_us)
        f = (N.i64 * max(1, len(fetch_us)))(*fetch_us)
        k, t = N.u32(), N.i64()
        self.n.call("cake_oracle_best_split", c, len(compute_us), f, len(fetch_us), C.byref(k), C.byref(t))
        return k.value, t.value

    # ---- scheduler (scheduler.hpp)
    def run_sim_planned(self, plan: RunPlan, cost: CostModel, trace: BandwidthTrace, mode: str = "cake",
                        power: float = 1.0, **opts) -> RunReport:
        n = plan.n
        t, keep = trace.native()
        recs = (N.CakeRecord * n)()
        s = N.CakeSummary()
        o = _opts(self.n, **opts)
        self.n.call("cake_sim_run", n, (N.u64 * n)(*plan.token_starts), (N.u32 * n)(*plan.token_counts),
                    (N.u64 * n)(*plan.encoded_bytes), (N.u64 * n)(*plan.uncompressed_bytes), cost.alpha_ms,
                    cost.beta_ms_per_token, cost.reference_chunk_size, t, MODES[mode], power, C.byref(o),
                    C.byref(s), recs)
        return RunReport(mode, s.n_chunks, s.ttft_us, s.merge_point, s.computed_fraction, s.compute_busy_us,
                         s.io_busy_us, _records(recs, n))

    def run(self, store: "ChunkStore", total_tokens: int, chunk_size: int, profile: tuple, codec: str,
            cost: CostModel, trace: BandwidthTrace, mode: str = "cake", clock: str = "sim", seed: int = 0,
            power: float = 1.0, **opts) -> RunReport:
        """reference run(request, profile, cost, trace, codec, mode, clock, store, seed, options)."""
        n_layers, hidden, precision = profile
        n = -(-total_tokens // chunk_size)
        t, keep = trace.native()
        recs = (N.CakeRecord * n)()
        s = N.CakeSummary()
        o = _opts(self.n, **opts)
        self.n.call("cake_run_store", store.h, total_tokens, chunk_size, n_layers, hidden, precision,
                    codec.encode(), cost.alpha_ms, cost.beta_ms_per_token, cost.reference_chunk_size, t,
                    MODES[mode], 1 if clock == "live" else 0, seed, power, C.byref(o), C.byref(s), recs)
        return RunReport(mode, s.n_chunks, s.ttft_us, s.merge_point, s.computed_fraction, s.compute_busy_us,
                         s.io_busy_us, _records(recs, n))

    # ---- cache tier (store.hpp)
    def chain_hash(self, prev: bytes | None, tokens: Sequence[int]) -> bytes:
        toks = np.ascontiguousarray(tokens, dtype=np.uint32)
        out = C.create_string_buffer(32)
        self.n.call("cake_chain_hash", prev, toks.ctypes.data, toks.size, out)
        return out.raw

    def token_stream(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint32)
        self.n.call("cake_token_stream", seed, count, out.ctypes.data)
        return out

    def synth_payload(self, seed: int, chunk_index: int, nbytes: int) -> bytes:
        out = C.create_string_buffer(max(nbytes, 1))
        self.n.call("cake_synth_payload", seed, chunk_index, nbytes, out)
        return out.raw[:nbytes]

    def codec_encoded_size(self, codec: str, raw: int) -> int:
        out = N.u64()
        self.n.call("cake_codec_encoded_size", codec.encode(), raw, C.byref(out))
        return out.value

    def codec_encode(self, codec: str, payload: bytes) -> bytes:
        cap = self.codec_encoded_size(codec, len(payload))
        out = C.create_string_buffer(max(cap, 1))
        n = N.u64()
        self.n.call("cake_codec_encode", codec.encode(), payload, len(payload), out, cap, C.byref(n))
        return out.raw[:n.value]

    def codec_decode(self, codec: str, encoded: bytes, original_len: int) -> bytes:
        out = C.create_string_buffer(max(original_len, 1))
        self.n.call("cake_codec_decode", codec.encode(), encoded, len(encoded), original_len, out, original_len)
        return out.raw[:original_len]

    def fp16_from_float(self, f: float) -> int:
        return self.n.lib.cake_fp16_from_float(f)

    def fp16_to_float(self, h: int) -> float:
        return self.n.lib.cake_fp16_to_float(h)

    def store(self, root: str | None, create: int = 2, pinned: bool = False) -> "ChunkStore":
        return ChunkStore(self.n, root, create, pinned)


class ChunkStore:
    """reference ChunkStore (files + manifest.v1), or a memory-resident tier when root is None."""

    def __init__(self, lib: N.Native, root: str | None, create: int = 2, pinned: bool = False):
        self.n = lib
        h = N.vp()
        self.n.call("cake_store_open", (root or "").encode(), create, 1 if pinned else 0, C.byref(h))
        self.h = h.value

    def close(self):
        if self.h:
            self.n.lib.cake_store_close(self.h)
            self.h = None

    def set_direct_io(self, on: bool = True):
        """File-backed stores: read aligned slices with O_DIRECT (B200 extension)."""
        self.n.call("cake_store_set_direct_io", self.h, 1 if on else 0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def entry_count(self) -> int:
        out = N.u64()
        self.n.call("cake_store_entry_count", self.h, C.byref(out))
        return out.value

    def populate(self, total_tokens, chunk_size, profile, codec="identity", seed=0, sparse=False) -> list:
        n_layers, hidden, precision = profile
        n = -(-total_tokens // chunk_size)
        keys = C.create_string_buffer(32 * n)
        self.n.call("cake_store_populate", self.h, total_tokens, chunk_size, n_layers, hidden, precision,
                    codec.encode(), seed, 1 if sparse else 0, keys)
        return [keys.raw[32 * i:32 * (i + 1)] for i in range(n)]

    def put(self, key: bytes, payload: bytes, token_count: int, codec="identity", uncompressed=None):
        self.n.call("cake_store_put", self.h, key, payload, len(payload), token_count, codec.encode(),
                    len(payload) if uncompressed is None else uncompressed)

    def get(self, key: bytes) -> bytes:
        n = N.u64()
        self.n.call("cake_store_get", self.h, key, None, 0, C.byref(n))
        out = C.create_string_buffer(max(n.value, 1))
        self.n.call("cake_store_get", self.h, key, out, n.value, C.byref(n))
        return out.raw[:n.value]

    def make_resident(self, pinned=True):
        self.n.call("cake_store_make_resident", self.h, 1 if pinned else 0)
