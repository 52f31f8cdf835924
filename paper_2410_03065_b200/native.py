"""ctypes bindings of the C ABIs (include/cake_c.h over libcake.so, include/cake_cuda.h
over libcake_cuda.so).

`load(path)` binds any library exporting the cake_c.h surface: the B200 runtime
(default) or — for parity tests only — the reference compiled from its own sources
(oracle/_ref/libcake_ref.so, same capi.cpp built with -DCAKE_REFERENCE_BUILD).
The product path never falls back: if the B200 library is missing, importing the
GPU runtime raises.
"""
from __future__ import annotations

import ctypes as C
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
B200_LIB = os.path.join(LIB_DIR, "libcake.so")
CUDA_LIB = os.path.join(LIB_DIR, "libcake_cuda.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libcake_ref.so")

i64, u64, u32, i32, dbl, vp = C.c_int64, C.c_uint64, C.c_uint32, C.c_int32, C.c_double, C.c_void_p


class CakeTrace(C.Structure):
    _fields_ = [("at_us", C.POINTER(i64)), ("mbps", C.POINTER(dbl)), ("n", C.c_int)]


class CakeRecord(C.Structure):
    _fields_ = [("index", u32), ("side", i32), ("start_us", i64), ("finish_us", i64), ("bytes", u64)]


class CakeRunOpts(C.Structure):
    _fields_ = [("compute_enabled", C.c_int), ("io_enabled", C.c_int), ("token_budget", u32),
                ("throttle_quantum_bytes", u64), ("decode_us_per_byte", dbl), ("jitter_max_us", u32),
                ("jitter_seed", u64), ("race_to_finish", C.c_int), ("cached_prefix", C.c_int),
                ("record_slices", C.c_int), ("race_force", C.c_int), ("race_hold", C.c_int), ("link", vp)]


class CakeSummary(C.Structure):
    _fields_ = [("ttft_us", i64), ("merge_point", u32), ("n_chunks", u32), ("computed_fraction", dbl),
                ("compute_busy_us", i64), ("io_busy_us", i64)]


class CakeGpuConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("hidden", C.c_int), ("n_heads", C.c_int), ("n_kv_heads", C.c_int),
                ("head_dim", C.c_int), ("ffn", C.c_int), ("vocab", C.c_int), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float), ("max_chunk", C.c_int), ("max_tokens", C.c_longlong),
                ("weight_seed", C.c_ulonglong), ("device", C.c_int), ("tp_rank", C.c_int), ("tp_size", C.c_int),
                ("nccl_comm", vp), ("lookahead_layers", C.c_int), ("profile_kernels", C.c_int),
                ("race_margin_us", i64), ("tp_shm", C.c_char_p), ("compute_sms", C.c_int),
                ("weights_from", vp)]


class CakeGpuResult(C.Structure):
    _fields_ = [("kv_resident_us", i64), ("first_token_us", i64), ("final_step_us", i64),
                ("device_ttft_ms", dbl), ("merge_point", u32), ("n_chunks", u32), ("raced_chunk", C.c_int),
                ("race_winner", C.c_int), ("recomputed_last", C.c_int), ("kernel_launches", C.c_longlong),
                ("h2d_bytes", u64), ("d2h_bytes", u64), ("compute_busy_us", i64), ("io_busy_us", i64)]


class CakeKernelStat(C.Structure):
    _fields_ = [("launches", C.c_longlong), ("total_ms", dbl), ("flops", dbl), ("bytes", dbl)]


KERNEL_NAMES = ["embed", "rmsnorm", "gemm_qkv", "attention", "gemm_o", "gemm_gu", "gemm_down", "allreduce",
                "lm_head", "kv_scatter", "dec_proj", "dec_attn"]

P = C.POINTER
_SIGS = {
    "cake_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "cake_time_to_transfer_bits": (C.c_int, [CakeTrace, u64, i64, P(i64)]),
    "cake_fetch_latency": (C.c_int, [CakeTrace, u64, i64, P(i64)]),
    "cake_compute_latency": (C.c_int, [dbl, dbl, u32, u64, u32, dbl, P(i64)]),
    "cake_kv_bytes_per_token": (C.c_int, [u32, u32, u32, u32, u64, P(u64)]),
    "cake_split_into_chunks": (C.c_int, [u64, u32, P(u32), P(u64), P(u32), u32]),
    "cake_oracle_best_split": (C.c_int, [P(i64), u32, P(i64), u32, P(u32), P(i64)]),
    "cake_run_opts_default": (None, [P(CakeRunOpts)]),
    "cake_sim_run": (C.c_int, [u32, P(u64), P(u32), P(u64), P(u64), dbl, dbl, u32, CakeTrace, C.c_int, dbl,
                               P(CakeRunOpts), P(CakeSummary), P(CakeRecord)]),
    "cake_store_open": (C.c_int, [C.c_char_p, C.c_int, C.c_int, P(vp)]),
    "cake_store_close": (C.c_int, [vp]),
    "cake_store_set_direct_io": (C.c_int, [vp, C.c_int]),
    "cake_store_entry_count": (C.c_int, [vp, P(u64)]),
    "cake_store_populate": (C.c_int, [vp, u64, u32, u32, u32, u32, C.c_char_p, u64, C.c_int, vp]),
    "cake_store_put": (C.c_int, [vp, vp, vp, u64, u32, C.c_char_p, u64]),
    "cake_store_get": (C.c_int, [vp, vp, vp, u64, P(u64)]),
    "cake_store_make_resident": (C.c_int, [vp, C.c_int]),
    "cake_chain_hash": (C.c_int, [vp, vp, u64, vp]),
    "cake_token_stream": (C.c_int, [u64, u64, vp]),
    "cake_synth_payload": (C.c_int, [u64, u32, u64, vp]),
    "cake_codec_encoded_size": (C.c_int, [C.c_char_p, u64, P(u64)]),
    "cake_codec_encode": (C.c_int, [C.c_char_p, vp, u64, vp, u64, P(u64)]),
    "cake_codec_decode": (C.c_int, [C.c_char_p, vp, u64, u64, vp, u64]),
    "cake_fp16_from_float": (C.c_uint16, [C.c_float]),
    "cake_fp16_to_float": (C.c_float, [C.c_uint16]),
    "cake_run_store": (C.c_int, [vp, u64, u32, u32, u32, u32, C.c_char_p, dbl, dbl, u32, CakeTrace, C.c_int,
                                 C.c_int, u64, dbl, P(CakeRunOpts), P(CakeSummary), P(CakeRecord)]),
    "cake_gpu_create": (C.c_int, [P(CakeGpuConfig), P(vp)]),
    "cake_link_create": (C.c_int, [CakeTrace, P(vp)]),
    "cake_link_destroy": (C.c_int, [vp]),
    "cake_link_reset": (C.c_int, [vp]),
    "cake_link_reserved_bits": (C.c_int, [vp, P(u64), P(i64)]),
    "cake_gpu_set_link": (C.c_int, [vp, vp]),
    "cake_gpu_destroy": (C.c_int, [vp]),
    "cake_gpu_kv_bytes_per_token": (C.c_int, [vp, P(u64)]),
    "cake_gpu_build_tier": (C.c_int, [vp, vp, u64, u32, u64]),
    "cake_gpu_set_codec": (C.c_int, [vp, C.c_char_p]),
    "cake_gpu_calibrate": (C.c_int, [vp, u64, u32, u64, P(dbl), P(dbl)]),
    "cake_gpu_run": (C.c_int, [vp, vp, u64, u32, u64, CakeTrace, C.c_int, P(CakeRunOpts), P(CakeGpuResult),
                               P(CakeRecord)]),
    "cake_gpu_logits": (C.c_int, [vp, vp, C.c_int]),
    "cake_gpu_read_chunk": (C.c_int, [vp, u64, u32, vp, u64]),
    "cake_gpu_kernel_stats": (C.c_int, [vp, P(CakeKernelStat), C.c_int]),
    "cake_gpu_set_profiling": (C.c_int, [vp, C.c_int]),
    "cake_gpu_set_profiling_stride": (C.c_int, [vp, C.c_int]),
    "cake_gpu_set_attention_impl": (C.c_int, [vp, C.c_int]),
    "cake_gpu_poison": (C.c_int, [vp, C.c_int]),
    "cake_gpu_slices": (C.c_int, [vp, P(i64), P(u64), u64, P(u64)]),
    "cake_gpu_model": (vp, [vp]),
    "cake_gpu_compute_stream": (vp, [vp]),
    "cake_tp_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, P(vp)]),
    "cake_tp_destroy": (C.c_int, [vp]),
    "cake_tp_begin_run": (C.c_int, [vp, u64, u32]),
    "cake_tp_end_run": (C.c_int, [vp]),
    "cake_tp_publish_compute": (C.c_int, [vp, u32]),
    "cake_tp_end_compute": (C.c_int, [vp]),
    "cake_tp_next_compute": (C.c_int, [vp, u32, P(u32), P(C.c_int)]),
    "cake_tp_publish_io": (C.c_int, [vp, u32]),
    "cake_tp_end_io": (C.c_int, [vp]),
    "cake_tp_next_io": (C.c_int, [vp, u32, P(u32), P(C.c_int)]),
    "cake_tp_shard_landed": (C.c_int, [vp, u32]),
    "cake_tp_wait_all_landed": (C.c_int, [vp, u32]),
    "cake_tp_publish_decided": (C.c_int, [vp, u32, C.c_int]),
    "cake_tp_decided": (C.c_int, [vp, u32, P(C.c_int)]),
    "cake_tp_publish_final": (C.c_int, [vp, C.c_int, C.c_int, C.c_int]),
    "cake_tp_wait_final": (C.c_int, [vp, P(C.c_int), P(C.c_int), P(C.c_int)]),
}


class CakeError(RuntimeError):
    pass


class MissingKeyError(CakeError):
    pass


class CorruptChunkError(CakeError):
    pass


class StoreError(CakeError):
    pass


class Native:
    """One loaded library exporting (a subset of) cake_c.h."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make` / __graft_entry__.build())")
        self.path = path
        self.lib = C.CDLL(path, mode=os.RTLD_LOCAL)
        self.available = set()
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, name, None)
            if fn is None:
                continue
            fn.restype, fn.argtypes = res, args
            self.available.add(name)

    def error(self) -> str:
        buf = C.create_string_buffer(2048)
        self.lib.cake_last_error(buf, 2048)
        return buf.value.decode(errors="replace")

    def call(self, name: str, *args):
        st = getattr(self.lib, name)(*args)
        if st == 0:
            return
        msg = f"{name}: {self.error()}"
        if st == -1:
            raise ValueError(msg)
        if st == -2:
            raise RuntimeError("logic_error: " + msg)
        if st == -3:
            raise MissingKeyError(msg)
        if st == -4:
            raise CorruptChunkError(msg)
        if st == -5:
            raise StoreError(msg)
        raise CakeError(msg)


_cache: dict[str, Native] = {}


def load(path: str | None = None) -> Native:
    path = path or B200_LIB
    if path not in _cache:
        _cache[path] = Native(path)
    return _cache[path]


def load_cuda():
    """libcake_cuda.so (the thin CUDA layer) with its exported symbols typed minimally."""
    if not os.path.exists(CUDA_LIB):
        raise FileNotFoundError(f"{CUDA_LIB} not built")
    lib = C.CDLL(CUDA_LIB, mode=os.RTLD_LOCAL)
    lib.cake_gemm.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp]
    lib.cake_cuda_last_error.argtypes = [C.c_char_p, C.c_size_t]
    lib.cake_kv_chunk_bytes.restype = C.c_longlong
    lib.cake_kv_chunk_bytes.argtypes = [vp, C.c_int]
    lib.cake_kv_scatter.argtypes = [vp, vp, C.c_longlong, C.c_int, vp, C.c_longlong, C.c_longlong, vp]
    lib.cake_kv_gather.argtypes = [vp, vp, C.c_longlong, C.c_int, vp, vp]
    lib.cake_kv_q8_bytes.restype = C.c_longlong
    lib.cake_kv_q8_bytes.argtypes = [vp, C.c_int]
    lib.cake_kv_scatter_q8.argtypes = [vp, vp, C.c_longlong, C.c_int, vp, vp]
    lib.cake_kv_encode_q8.argtypes = [vp, vp, C.c_int, vp, vp]
    lib.cake_prefill_group.argtypes = [C.POINTER(vp), C.c_int, vp, C.c_longlong, C.c_int, vp, vp]
    lib.cake_final_logits.argtypes = [vp, C.c_longlong, vp, C.c_int, C.c_int, vp, vp, vp]
    lib.cake_nccl_unique_id.argtypes = [vp]
    lib.cake_nccl_init.argtypes = [C.POINTER(vp), vp, C.c_int, C.c_int]
    lib.cake_attention_debug.argtypes = [vp, vp, C.c_longlong, C.c_int, C.c_int, vp, vp, vp]
    lib.cake_tp_peer_handles.argtypes = [vp, vp, C.c_size_t]
    lib.cake_tp_peer_open.argtypes = [vp, vp, C.c_int]
    return lib


TP_PEER_HANDLE_BYTES = 512  # include/cake_cuda.h CAKE_TP_PEER_HANDLE_BYTES


def make_trace(points):
    """points: [(at_us, mbps), ...] -> (CakeTrace, keepalive)."""
    at = (i64 * len(points))(*[int(p[0]) for p in points])
    mb = (dbl * len(points))(*[float(p[1]) for p in points])
    return CakeTrace(C.cast(at, P(i64)), C.cast(mb, P(dbl)), len(points)), (at, mb)
