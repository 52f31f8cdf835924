"""ctypes handle on oracle/_lib/libllama_ref.so (CPU transformer oracle).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_lib", "libllama_ref.so")


class RefConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("hidden", C.c_int), ("n_heads", C.c_int), ("n_kv_heads", C.c_int),
                ("head_dim", C.c_int), ("ffn", C.c_int), ("vocab", C.c_int), ("rope_theta", C.c_float),
                ("rms_eps", C.c_float), ("seed", C.c_ulonglong), ("threads", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise FileNotFoundError(f"{LIB} not built (make -C oracle)")
        _lib = C.CDLL(LIB)
        vp = C.c_void_p
        _lib.ref_create.restype = vp
        _lib.ref_create.argtypes = [C.POINTER(RefConfig), C.c_longlong, C.c_longlong]
        _lib.ref_destroy.argtypes = [vp]
        _lib.ref_begin_chunk.argtypes = [vp, vp, C.c_longlong, C.c_int]
        _lib.ref_run_layers.argtypes = [vp, C.c_int, C.c_int]
        _lib.ref_final_logits.argtypes = [vp, C.c_int, vp]
        _lib.ref_last_token_logits.argtypes = [vp, C.c_int32, C.c_longlong, vp]
        _lib.ref_load_chunk.argtypes = [vp, vp, C.c_longlong, C.c_int]
        _lib.ref_kv.restype = C.POINTER(C.c_float)
        _lib.ref_kv.argtypes = [vp]
        _lib.ref_weight_bits.restype = C.c_uint16
        _lib.ref_weight_bits.argtypes = [C.c_ulonglong, C.c_uint32, C.c_uint64, C.c_float]
    return _lib


class LlamaRef:
    """dims = (n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab)."""

    def __init__(self, dims, max_tokens, seed=1234, threads=0, cache_weight_bytes=8 << 30,
                 rope_theta=500000.0, rms_eps=1e-5):
        self.dims = dims
        L, H, nh, nkv, hd, ffn, vocab = dims
        cfg = RefConfig(L, H, nh, nkv, hd, ffn, vocab, rope_theta, rms_eps, seed, threads)
        self.h = lib().ref_create(C.byref(cfg), max_tokens, cache_weight_bytes)
        if not self.h:
            raise MemoryError("ref_create failed")
        self.max_tokens = max_tokens

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_destroy(self.h)
            self.h = None

    def prefill_chunk(self, tokens, start, layers=None):
        toks = np.ascontiguousarray(tokens, dtype=np.int32)
        assert lib().ref_begin_chunk(self.h, toks.ctypes.data, start, toks.size) == 0
        L = self.dims[0]
        l0, l1 = layers if layers is not None else (0, L)
        assert lib().ref_run_layers(self.h, l0, l1) == 0

    def final_logits(self, row):
        out = np.empty(self.dims[6], dtype=np.float32)
        assert lib().ref_final_logits(self.h, row, out.ctypes.data) == 0
        return out

    def last_token_logits(self, token, T):
        out = np.empty(self.dims[6], dtype=np.float32)
        assert lib().ref_last_token_logits(self.h, int(token), T, out.ctypes.data) == 0
        return out

    def load_chunk(self, tier_bytes: bytes, start, length):
        buf = np.frombuffer(tier_bytes, dtype=np.uint16)
        assert lib().ref_load_chunk(self.h, buf.ctypes.data, start, length) == 0

    def kv(self) -> np.ndarray:
        L, H, nh, nkv, hd, ffn, vocab = self.dims
        n = L * 2 * nkv * self.max_tokens * hd
        arr = np.ctypeslib.as_array(lib().ref_kv(self.h), shape=(n,))
        return arr.reshape(L, 2, nkv, self.max_tokens, hd)

    def chunk_tier(self, start, length) -> np.ndarray:
        """This oracle's KV of tokens [start, start+length) in the cache-tier layout, fp32."""
        return np.ascontiguousarray(self.kv()[:, :, :, start:start + length, :])


def weight_bits(seed, tensor_id, index, scale):
    return lib().ref_weight_bits(seed, tensor_id, index, scale)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)
