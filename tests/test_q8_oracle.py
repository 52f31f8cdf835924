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
