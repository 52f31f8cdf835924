"""quant8 tier codec: the oracle (oracle/kvcodec.py) pinned to the reference.

* golden vectors produced by the reference library (tests/golden/q8_golden.json,
  tests/golden/make_q8_golden.py) -> oracle bit-exact, encode and decode;
* the live reference library (oracle/_ref) and this build's host codec
  (libcake.so, codec.cpp) on seeded random payloads -> oracle bit-exact;
* the bf16 variant the GPU tier uses: the reference's properties
  (proj/tests/test_codec.cpp:81-109: constant payloads exact, error bound).
"""
import json
import os

import numpy as np
import pytest

import kvcodec

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "q8_golden.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c["name"])
def test_oracle_matches_reference_golden(case):
    payload = bytes.fromhex(case["payload"])
    enc = kvcodec.q8_encode(payload, "f16")
    assert enc == bytes.fromhex(case["encoded"])
    assert kvcodec.q8_decode(enc, len(payload), "f16") == bytes.fromhex(case["decoded"])


def _random_payloads(seed, count=12):
    rng = np.random.default_rng(seed)
    for i in range(count):
        n = int(rng.integers(1, 5000))
        scale = 10.0 ** rng.uniform(-4, 4)
        yield (rng.standard_normal(n) * scale).astype(np.float16).tobytes()


def test_oracle_matches_reference_lib(cake_ref):
    for p in _random_payloads(7):
        enc = cake_ref.codec_encode("quant8", p)
        assert kvcodec.q8_encode(p, "f16") == enc
        assert kvcodec.q8_decode(enc, len(p), "f16") == cake_ref.codec_decode("quant8", enc, len(p))


def test_host_codec_matches_oracle(cake_b200):
    for p in _random_payloads(8):
        enc = cake_b200.codec_encode("quant8", p)
        assert enc == kvcodec.q8_encode(p, "f16")
        assert cake_b200.codec_decode("quant8", enc, len(p)) == kvcodec.q8_decode(enc, len(p), "f16")


def test_bf16_variant_properties():
    rng = np.random.default_rng(3)
    const = kvcodec.f32_to_bf16_bits(np.full(4096, 0.3125, np.float32))
    dec = kvcodec.q8_decode(kvcodec.q8_encode(const, "bf16"), const.nbytes, "bf16")
    assert dec == const.tobytes()
    for _ in range(10):
        x = kvcodec.f32_to_bf16_bits((rng.standard_normal(8192) * rng.uniform(0.01, 20)).astype(np.float32))
        enc = kvcodec.q8_encode(x, "bf16")
        assert len(enc) == x.nbytes // 2 + 4
        y = kvcodec.bf16_bits_to_f32(np.frombuffer(kvcodec.q8_decode(enc, x.nbytes, "bf16"), np.uint16))
        v = kvcodec.bf16_bits_to_f32(x)
        span = v.max() - v.min()
        # half a level + the bf16 rounding of the result (and of the fp16 header)
        bound = span / 255 / 2 + np.abs(v).max() * 2.0 ** -8 + span * 2.0 ** -10
        assert np.abs(y - v).max() <= bound


def _dual_payloads(seed, count=12):
    """Values exactly representable in BOTH fp16 and bf16 (8 significant bits, fp16 normal range), so the
    reference's fp16 payload and the B200 tier's bf16 payload carry the same numbers."""
    rng = np.random.default_rng(seed)
    for _ in range(count):
        n = int(rng.integers(1, 5000))
        mant = rng.integers(128, 256, n)  # 8-bit significand
        expo = rng.integers(-10, 8, n)
        sign = rng.choice([-1.0, 1.0], n)
        v = (sign * mant * np.exp2(expo - 7.0)).astype(np.float32)
        yield v


def test_bf16_variant_pinned_to_reference_lib(cake_ref):
    """The bf16 tier encoding (the GPU's, bit-exact to kvcodec in tests/test_gpu_q8.py) equals the
    reference library's fp16 encoding of the same values (codec.cpp:114-143: the levels and the fp16
    (lo, hi) header depend only on the values); decoded values are the same fp32 result of
    codec.cpp:158 rounded to bf16 instead of fp16, so they agree within the two roundings."""
    for v in _dual_payloads(11):
        f16 = v.astype(np.float16)
        bf = kvcodec.f32_to_bf16_bits(v)
        assert np.array_equal(f16.astype(np.float32), v) and np.array_equal(kvcodec.bf16_bits_to_f32(bf), v)
        ref_enc = cake_ref.codec_encode("quant8", f16.tobytes())
        enc = kvcodec.q8_encode(bf, "bf16")
        assert enc == ref_enc
        y16 = np.frombuffer(cake_ref.codec_decode("quant8", ref_enc, f16.nbytes), np.float16).astype(np.float64)
        ybf = kvcodec.bf16_bits_to_f32(np.frombuffer(kvcodec.q8_decode(enc, bf.nbytes, "bf16"), np.uint16))
        tol = np.abs(y16) * (2.0 ** -8 + 2.0 ** -11) + 2.0 ** -24
        assert np.all(np.abs(ybf.astype(np.float64) - y16) <= tol)
