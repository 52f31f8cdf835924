"""Numpy restatement of the CPU transformer oracle, for sizes the plain-C loops
cannot reach in a test (full-depth Llama-3-8B, 70B dimensions, 32K prefixes).

TEST INFRASTRUCTURE ONLY — imported by tests/ (never by the product path).

Same model and the same bf16 rounding points as oracle/llama_ref.c (checked
against it in tests/test_oracle_pinned.py, and both against
transformers.LlamaForCausalLM goldens in tests/golden/hf_*.npz):

  h      = embed[token]                                  (bf16 values, fp32 residual)
  xn     = bf16(h * rsqrt(mean(h^2) + eps))              (gamma = 1)
  q, k   = bf16(rope(xn @ Wq^T)), bf16(rope(xn @ Wk^T))  (rotate-half RoPE, theta)
  v      = bf16(xn @ Wv^T)
  attn   = bf16(softmax(q k^T / sqrt(hd), causal) v)     (GQA: q head h reads kv head h // G)
  h     += attn @ Wo^T
  xn     = bf16(norm(h)); act = bf16(silu(xn @ Wg^T) * (xn @ Wu^T)); h += act @ Wd^T
  logits = bf16(norm(h_last)) @ Wlm^T

Weights come from the same counter-hash generator (ref_weight_matrix_bits in
libllama_ref.so, bit-identical to the GPU's weight_value). The reference has
no model (proj/src/compute.cpp:48-49 sleeps), so none of this cites it.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

import llama_oracle

W_Q, W_K, W_V, W_O, W_GATE, W_UP, W_DOWN = range(7)
TID_EMBED = 1 << 20
TID_LMHEAD = (1 << 20) + 1


def _lib():
    lib = llama_oracle.lib()
    if not hasattr(lib, "_np_ready"):
        lib.ref_weight_matrix_bits.argtypes = [C.c_ulonglong, C.c_uint32, C.c_longlong, C.c_longlong, C.c_float,
                                               C.c_void_p]
        lib.ref_round_bf16.argtypes = [C.c_void_p, C.c_longlong]
        lib._np_ready = True
    return lib


def weight_bits(seed, tid, rows, cols, scale) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.uint16)
    _lib().ref_weight_matrix_bits(seed, tid, rows, cols, scale, out.ctypes.data)
    return out


def weight(seed, tid, rows, cols, scale) -> np.ndarray:
    return llama_oracle.bf16_to_f32(weight_bits(seed, tid, rows, cols, scale)).reshape(rows, cols)


def round_bf16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    _lib().ref_round_bf16(x.ctypes.data, x.size)
    return x


class LlamaNp:
    """dims = (n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab)."""

    def __init__(self, dims, max_tokens, seed=1234, rope_theta=500000.0, rms_eps=1e-5, cache_layers=False):
        self.dims = tuple(dims)
        L, H, nh, nkv, hd, ffn, V = self.dims
        self.max_tokens = max_tokens
        self.seed = seed
        self.eps = np.float32(rms_eps)
        self.G = nh // nkv
        self.s_h = np.float32(1.0 / np.sqrt(np.float32(H)))
        self.s_o = np.float32(1.0 / np.sqrt(np.float32(nh * hd)))
        self.s_f = np.float32(1.0 / np.sqrt(np.float32(ffn)))
        # the same per-layer KV cache layout as llama_ref.c: [L][2][nkv][pos][hd], fp32 values of bf16
        self.kv = np.zeros((L, 2, nkv, max_tokens, hd), dtype=np.float32)
        half = hd // 2
        i = np.arange(half, dtype=np.float64)
        inv = np.power(np.float64(rope_theta), -2.0 * i / hd)
        ang = np.arange(max_tokens, dtype=np.float64)[:, None] * inv[None, :]
        self.cos = np.cos(ang).astype(np.float32)
        self.sin = np.sin(ang).astype(np.float32)
        self.cache_layers = cache_layers
        self._layers = {}
        self.h = None
        self.start = 0

    # ---- weights (scales as llama_ref.c gen_layer)
    def layer(self, l):
        if l in self._layers:
            return self._layers[l]
        L, H, nh, nkv, hd, F, V = self.dims
        s = self.seed
        w = {
            "q": weight(s, 16 * l + W_Q, nh * hd, H, self.s_h),
            "k": weight(s, 16 * l + W_K, nkv * hd, H, self.s_h),
            "v": weight(s, 16 * l + W_V, nkv * hd, H, self.s_h),
            "o": weight(s, 16 * l + W_O, H, nh * hd, self.s_o),
            "g": weight(s, 16 * l + W_GATE, F, H, self.s_h),
            "u": weight(s, 16 * l + W_UP, F, H, self.s_h),
            "d": weight(s, 16 * l + W_DOWN, H, F, self.s_f),
        }
        if self.cache_layers:
            self._layers[l] = w
        return w

    def embed(self, tokens) -> np.ndarray:
        H = self.dims[1]
        lib = _lib()
        out = np.empty((len(tokens), H), dtype=np.uint16)
        for i, t in enumerate(np.asarray(tokens, dtype=np.int64)):
            # row t of the (vocab, H) table: a (1, H) block at logical offset t*H
            out[i] = _row_bits(lib, self.seed, TID_EMBED, int(t), H, 1.0)
        return llama_oracle.bf16_to_f32(out).reshape(len(tokens), H)

    # ---- math at llama_ref.c's rounding points
    def norm(self, h):
        ss = np.einsum("ij,ij->i", h.astype(np.float64), h.astype(np.float64))
        r = (np.float32(1.0) / np.sqrt((ss / h.shape[1]).astype(np.float32) + self.eps)).astype(np.float32)
        return round_bf16(h * r[:, None])

    def rope(self, x, pos0):
        T = x.shape[0]
        half = self.dims[4] // 2
        c = self.cos[pos0:pos0 + T][:, None, :]
        s = self.sin[pos0:pos0 + T][:, None, :]
        a, b = x[..., :half], x[..., half:]
        return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)

    def attention(self, l, q, pos0):
        """q: [T, nh, hd] at positions pos0.. over cached keys [0, pos0 + t]."""
        L, H, nh, nkv, hd, F, V = self.dims
        T = q.shape[0]
        end = pos0 + T
        scale = np.float32(1.0 / np.sqrt(np.float32(hd)))
        out = np.empty((T, nh, hd), dtype=np.float32)
        qpos = pos0 + np.arange(T)[:, None]
        kpos = np.arange(end)[None, :]
        mask = kpos > qpos
        for g in range(nkv):
            K = self.kv[l, 0, g, :end]
            Vv = self.kv[l, 1, g, :end]
            for j in range(self.G):
                h = g * self.G + j
                s = (q[:, h, :] @ K.T) * scale
                s[mask] = -np.inf
                m = s.max(axis=1, keepdims=True)
                p = np.exp(s - m)
                den = p.sum(axis=1, keepdims=True, dtype=np.float64)
                out[:, h, :] = (p / den.astype(np.float32)) @ Vv
        return round_bf16(out.reshape(T, nh * hd))

    def block(self, l, q_only=False):
        L, H, nh, nkv, hd, F, V = self.dims
        w = self.layer(l)
        T, pos0 = self.h.shape[0], self.start
        xn = self.norm(self.h)
        q = round_bf16(self.rope((xn @ w["q"].T).reshape(T, nh, hd), pos0))
        if not q_only:
            k = round_bf16(self.rope((xn @ w["k"].T).reshape(T, nkv, hd), pos0))
            v = round_bf16(xn @ w["v"].T).reshape(T, nkv, hd)
            self.kv[l, 0, :, pos0:pos0 + T] = k.transpose(1, 0, 2)
            self.kv[l, 1, :, pos0:pos0 + T] = v.transpose(1, 0, 2)
        at = self.attention(l, q.reshape(T, nh, hd), pos0)
        self.h += at @ w["o"].T
        xn = self.norm(self.h)
        g = xn @ w["g"].T
        u = xn @ w["u"].T
        act = round_bf16(g / (np.float32(1.0) + np.exp(-g)) * u)
        self.h += act @ w["d"].T

    # ---- driver (mirrors llama_oracle.LlamaRef)
    def prefill(self, tokens, start, layers=None):
        """Tokens at positions [start, start+len): every layer (or [l0, l1)), KV cached."""
        self.h = self.embed(tokens)
        self.start = start
        l0, l1 = layers if layers is not None else (0, self.dims[0])
        for l in range(l0, l1):
            self.block(l)

    def final_logits(self, row):
        L, H, nh, nkv, hd, F, V = self.dims
        xn = self.norm(self.h[row:row + 1])
        wl = weight(self.seed, TID_LMHEAD, V, H, self.s_h)
        return (xn @ wl.T)[0]

    def last_token_logits(self, token, T):
        """First-token step over a complete cache: q-only pass of position T-1."""
        self.h = self.embed([token])
        self.start = T - 1
        for l in range(self.dims[0]):
            self.block(l, q_only=True)
        return self.final_logits(0)

    def load_chunk(self, tier_bytes: bytes, start, length):
        L, H, nh, nkv, hd, F, V = self.dims
        a = llama_oracle.bf16_to_f32(np.frombuffer(tier_bytes, dtype=np.uint16)).reshape(L, 2, nkv, length, hd)
        self.kv[:, :, :, start:start + length] = a

    def chunk_tier(self, start, length) -> np.ndarray:
        return np.ascontiguousarray(self.kv[:, :, :, start:start + length, :])


def _row_bits(lib, seed, tid, row, cols, scale):
    """bf16 bits of row `row` of a (*, cols) tensor: logical indices [row*cols, (row+1)*cols)."""
    out = np.empty(cols, dtype=np.uint16)
    if not hasattr(lib, "_row_ready"):
        lib.ref_weight_row_bits.argtypes = [C.c_ulonglong, C.c_uint32, C.c_longlong, C.c_longlong, C.c_float,
                                            C.c_void_p]
        lib._row_ready = True
    lib.ref_weight_row_bits(seed, tid, row, cols, scale, out.ctypes.data)
    return out
