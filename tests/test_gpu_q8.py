"""quant8 cache tier on the GPU vs the oracle.

* tier build: the GPU encoder (cake_kv_encode_q8) over every chunk's bf16 KV
  == oracle/kvcodec.py q8_encode(elem="bf16") of the identity tier's bytes, bit-exact;
* load: an io-only run from the quant8 tier assembles exactly
  q8_decode(elem="bf16") of each chunk (decode fused into the scatter), bit-exact;
* bidirectional run from the quant8 tier: first-token logits stay close to the
  identity tier's (quantisation error only; cosine >= 0.99) with half the bytes loaded.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (2, 512, 8, 2, 64, 1024, 32000)
T, C, SEED = 1024, 256, 42


@pytest.fixture(scope="module")
def q8setup():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    rt = GpuRuntime(DIMS, max_tokens=T, max_chunk=C)
    tier_id = rt.build_cache_tier(T, C, SEED)
    rt.set_codec("quant8")
    tier_q8 = rt.build_cache_tier(T, C, SEED)
    cake = Cake()
    toks = cake.token_stream(SEED, T)
    keys, prev = [], None
    for s in range(0, T, C):
        prev = cake.chain_hash(prev, toks[s:s + C])
        keys.append(prev)
    return rt, tier_id, tier_q8, keys


def test_gpu_encode_matches_oracle(q8setup):
    import kvcodec

    rt, tier_id, tier_q8, keys = q8setup
    for k in keys:
        raw = tier_id.get(k)
        enc = tier_q8.get(k)
        assert len(enc) == len(raw) // 2 + 4
        assert enc == kvcodec.q8_encode(np.frombuffer(raw, np.uint16), "bf16")


def test_gpu_decode_scatter_matches_oracle(q8setup):
    import kvcodec

    rt, tier_id, tier_q8, keys = q8setup
    r = rt.run(tier_q8, T, C, SEED, mbps=8000, mode="io_only")
    # every loaded byte is the quant8 payload; the only other upload is the prompt's token ids
    assert r.h2d_bytes == sum(len(tier_q8.get(k)) for k in keys) + 4 * T
    for i, k in enumerate(keys):
        raw_len = len(tier_id.get(k))
        want = kvcodec.q8_decode(tier_q8.get(k), raw_len, "bf16")
        assert rt.read_chunk(i * C, C) == want, i


def test_bidirectional_from_q8_tier(q8setup):
    rt, tier_id, tier_q8, keys = q8setup
    rt.set_codec("identity")
    rt.run(tier_id, T, C, SEED, mbps=8000, mode="io_only")
    want = rt.logits()
    rt.set_codec("quant8")
    r = rt.run(tier_q8, T, C, SEED, mbps=8000, mode="cake")
    got = rt.logits()
    assert np.isfinite(got).all()
    cosv = float(np.dot(got, want) / (np.linalg.norm(got) * np.linalg.norm(want)))
    assert cosv >= 0.99, cosv
    assert r.merge_point <= r.n_chunks
