"""numpy restatement of the reference's quant8 cache-tier codec.

TEST INFRASTRUCTURE ONLY (checker for tests/; never imported by the product).

Reference: proj/src/codec.cpp:114-143 (quant8_encode), :145-162 (quant8_decode).
One (lo, hi) pair per chunk, stored as fp16; one byte per element,
level = lroundf((v - lo) / range * 255) clamped to [0, 255]; decode
lo + level / 255 * range. Every float32 operation is done in the same order
as the reference (numpy float32 arithmetic rounds per op, like the reference's
scalar code on x86-64 without FMA contraction).

`elem` selects the element type: "f16" is the reference's own payload (pinned
bit-exact against oracle/_ref/libcake_ref.so in tests/test_q8_oracle.py);
"bf16" is the B200 build's KV tier (the cache is bf16), where values read as
bf16 and decode rounds to bf16 (RNE) instead of fp16.
"""
from __future__ import annotations

import numpy as np


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def _values(payload: bytes | np.ndarray, elem: str) -> np.ndarray:
    h = np.frombuffer(payload, dtype=np.uint16) if isinstance(payload, (bytes, bytearray)) else payload
    if elem == "f16":
        return h.view(np.float16).astype(np.float32)
    if elem == "bf16":
        return bf16_bits_to_f32(h)
    raise ValueError(elem)


def q8_encode(payload: bytes | np.ndarray, elem: str = "f16") -> bytes:
    """codec.cpp:114-143."""
    v = _values(payload, elem)
    n = v.size
    lo = np.float32(v.min()) if n else np.float32(0.0)  # :118-126 running min/max
    hi = np.float32(v.max()) if n else np.float32(0.0)
    hdr = np.array([lo, hi], dtype=np.float32).astype(np.float16).view(np.uint16)  # :128 fp16_from_float
    rng = np.float32(hi - lo)  # :131
    if rng <= np.float32(0.0):  # :134-136
        levels = np.zeros(n, dtype=np.uint8)
    else:
        t = ((v - lo) / rng) * np.float32(255.0)  # :138, float32 per op
        q = np.floor(t.astype(np.float64) + 0.5)  # lroundf: half away from zero (t >= 0)
        levels = np.clip(q, 0, 255).astype(np.uint8)  # :140
    return hdr.tobytes() + levels.tobytes()


def q8_decode(encoded: bytes, original_len: int, elem: str = "f16") -> bytes:
    """codec.cpp:145-162; elem "bf16" rounds the result to bf16 instead of fp16."""
    n = original_len // 2
    if original_len % 2 or len(encoded) != 4 + n:
        raise ValueError("quant8: length mismatch")
    hdr = np.frombuffer(encoded[:4], dtype=np.uint16).view(np.float16).astype(np.float32)
    lo = np.float32(hdr[0])
    rng = np.float32(np.float32(hdr[1]) - lo)  # :153
    q = np.frombuffer(encoded[4:], dtype=np.uint8).astype(np.float32)
    if rng <= np.float32(0.0):
        v = np.full(n, lo, dtype=np.float32)
    else:
        v = lo + (q / np.float32(255.0)) * rng  # :158
    if elem == "f16":
        return v.astype(np.float16).tobytes()
    return f32_to_bf16_bits(v).tobytes()
