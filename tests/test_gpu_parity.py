"""GPU hot path vs the CPU oracle (oracle/llama_ref.c) on identical seeded inputs.

Tolerances (bf16 storage, fp32 accumulate; stated per SURVEY.md §8c):
  computed KV       max |gpu - cpu| / max|cpu| <= 2e-2 per layer tensor (bf16 ulp is 2^-8 = 3.9e-3;
                    rounding differences compound through the layers)
  first-token logits  rel err <= 2e-2, cosine >= 0.999, top-1 equal
  loaded KV          bit-exact vs the cache tier
  assembled cache    bit-exact across merge points (deterministic kernels)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CONFIGS = {
    # name: (dims, T, chunk)
    "tiny": ((2, 256, 4, 4, 64, 1024, 32000), 2048, 256),
    "gqa_hd64": ((2, 512, 8, 2, 64, 1024, 32000), 1024, 256),
    "gqa_hd128": ((2, 1024, 8, 2, 128, 2048, 32768), 1024, 512),
    # GQA 8:1 (the Llama-3-70B grouping: 16 tokens x 8 heads per 128-row tile)
    "gqa8_hd128": ((2, 1024, 16, 2, 128, 2048, 32768), 1024, 256),
}


def top1_ok(got, want, tol=2e-2):
    """GPU arg-max is the oracle's arg-max, or a near-tie within the stated tolerance."""
    return want[int(got.argmax())] >= want.max() - tol * np.abs(want).max()


def rel(a, b):
    return float(np.abs(a - b).max() / (np.abs(b).max() + 1e-12))


def cos(a, b):
    return float(np.dot(a, b) / (np.linalg.norm(a) * np.linalg.norm(b)))


@pytest.fixture(scope="module", params=list(CONFIGS))
def setup(request):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import llama_oracle
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    dims, T, C = CONFIGS[request.param]
    seed = 42
    rt = GpuRuntime(dims, max_tokens=T, max_chunk=C)
    tier = rt.build_cache_tier(T, C, seed)
    toks = Cake().token_stream(seed, T).astype(np.int32)
    ref = llama_oracle.LlamaRef(dims, T)
    for s in range(0, T, C):
        ref.prefill_chunk(toks[s:s + C], s)
    return {"rt": rt, "tier": tier, "ref": ref, "toks": toks, "T": T, "C": C, "dims": dims,
            "ref_logits": ref.final_logits(C - 1)}


def _chunk_kv(rt, s, c):
    import llama_oracle

    L, H, nh, nkv, hd, ffn, V = rt.dims
    b = np.frombuffer(rt.read_chunk(s, c), dtype=np.uint16)
    return llama_oracle.bf16_to_f32(b).reshape(L, 2, nkv, c, hd)


def test_computed_kv_matches_oracle(setup):
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.run(setup["tier"], T, C, 42, mbps=1000, mode="compute_only")
    kv = setup["ref"].kv()
    for s in range(0, T, C):
        got = _chunk_kv(rt, s, C)
        want = kv[:, :, :, s:s + C, :]
        for layer in range(got.shape[0]):
            assert rel(got[layer], want[layer]) <= 2e-2, (s, layer)


@pytest.mark.parametrize("mode", ["compute_only", "io_only"])
def test_first_token_logits_match_oracle(setup, mode):
    rt = setup["rt"]
    r = rt.run(setup["tier"], setup["T"], setup["C"], 42, mbps=4000, mode=mode)
    lg, want = rt.logits(), setup["ref_logits"]
    assert r.recomputed_last == (mode == "io_only")
    assert rel(lg, want) <= 2e-2
    assert cos(lg, want) >= 0.999
    assert top1_ok(lg, want)


def test_loaded_kv_bit_exact(setup):
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    from paper_2410_03065_b200.cake import Cake

    r = rt.run(setup["tier"], T, C, 42, mbps=40000, mode="io_only")
    assert r.merge_point == 0
    toks = setup["toks"].astype(np.uint32)
    prev = None
    for s in range(0, T, C):
        key = Cake().chain_hash(prev, toks[s:s + C])
        prev = key
        assert rt.read_chunk(s, C) == setup["tier"].get(key)


@pytest.mark.parametrize("mbps", [200, 2000, 20000, 200000])
def test_assembled_cache_independent_of_merge_point(setup, mbps):
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.run(setup["tier"], T, C, 42, mbps=mbps, mode="compute_only")
    base = [rt.read_chunk(s, C) for s in range(0, T, C)]
    r = rt.run(setup["tier"], T, C, 42, mbps=mbps, mode="cake")
    assert sorted(c.index for c in r.chunks) == list(range(T // C))
    assert all((c.side == "compute") == (c.index < r.merge_point) for c in r.chunks)
    for i, s in enumerate(range(0, T, C)):
        assert rt.read_chunk(s, C) == base[i], (mbps, i, r.merge_point)
    lg = rt.logits()
    assert top1_ok(lg, setup["ref_logits"])
    assert rel(lg, setup["ref_logits"]) <= 2e-2


def test_tcgen05_attention_matches_mma_sync_kernel(setup):
    """The two independent attention kernels agree on the whole computed cache
    (bf16 P in both; only accumulation order differs)."""
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.set_attention_impl("mma_sync")
    rt.run(setup["tier"], T, C, 42, mbps=1000, mode="compute_only")
    mma = [_chunk_kv(rt, s, C) for s in range(0, T, C)]
    lg_mma = rt.logits()
    rt.set_attention_impl("tcgen05")
    rt.run(setup["tier"], T, C, 42, mbps=1000, mode="compute_only")
    tc = [_chunk_kv(rt, s, C) for s in range(0, T, C)]
    for a, b in zip(tc, mma):
        assert rel(a, b) <= 2e-2
    assert rel(rt.logits(), lg_mma) <= 2e-2


@pytest.mark.parametrize("other", ["tcgen05_2tile", "tcgen05_dec"])
def test_two_tile_attention_matches_one_tile_kernel(setup, other):
    """The two-tile (ping-pong) tcgen05 kernel, and the one-tile kernel with
    decoupled softmax groups, against the one-tile tcgen05 kernel."""
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.set_attention_impl("tcgen05_1tile")
    rt.run(setup["tier"], T, C, 42, mbps=1000, mode="compute_only")
    one = [_chunk_kv(rt, s, C) for s in range(0, T, C)]
    lg_one = rt.logits()
    rt.set_attention_impl(other)
    rt.run(setup["tier"], T, C, 42, mbps=1000, mode="compute_only")
    two = [_chunk_kv(rt, s, C) for s in range(0, T, C)]
    lg_two = rt.logits()
    rt.set_attention_impl("tcgen05")
    for a, b in zip(two, one):
        assert rel(a, b) <= 2e-2
    assert rel(lg_two, lg_one) <= 2e-2


@pytest.mark.parametrize("mode", ["cake", "io_only"])
def test_partially_cached_prompt(setup, mode):
    """Only a prefix of the prompt is in the tier (cached_prefix): the bidirectional
    phase covers it, the uncached suffix is computed after it. The assembled cache
    and the first-token logits are bit-identical to a full compute-only run."""
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.run(setup["tier"], T, C, 42, mbps=1000, mode="compute_only")
    want_kv = [rt.read_chunk(s, C) for s in range(0, T, C)]
    want = rt.logits()
    cached = T // 2
    part = rt.build_cache_tier(cached, C, 42)
    r = rt.run(part, T, C, 42, mbps=1000, mode=mode, cached_prefix=True)
    assert r.n_chunks == T // C
    assert sorted(c.index for c in r.chunks) == list(range(T // C))
    assert all(c.side == "compute" for c in r.chunks if c.index >= cached // C)
    assert r.merge_point <= cached // C
    assert not r.recomputed_last  # the computed suffix holds the last token's hidden state
    assert [rt.read_chunk(s, C) for s in range(0, T, C)] == want_kv
    assert np.array_equal(rt.logits(), want)
    with pytest.raises(Exception):
        rt.run(part, T, C, 42, mbps=1000, mode=mode)  # without the option a missing chunk is an error


@pytest.mark.parametrize("direct", [False, True])
def test_file_tier(setup, tmp_path, direct):
    """Cache tier on local disk in the reference's file format (one file per
    chunk + manifest), read by the loader with buffered or O_DIRECT reads:
    the assembled cache and the logits equal the pinned-memory tier's."""
    from paper_2410_03065_b200.cake import ChunkStore

    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.run(setup["tier"], T, C, 42, mbps=8000, mode="io_only")
    want_kv = [rt.read_chunk(s, C) for s in range(0, T, C)]
    want = rt.logits()
    fs = ChunkStore(rt.n, str(tmp_path / f"tier{int(direct)}"), create=1)
    rt.build_cache_tier(T, C, 42, store=fs)
    fs.set_direct_io(direct)
    for mode in ("io_only", "cake"):
        r = rt.run(fs, T, C, 42, mbps=8000, mode=mode)
        assert sorted(c.index for c in r.chunks) == list(range(T // C))
        assert [rt.read_chunk(s, C) for s in range(0, T, C)] == want_kv
        assert np.array_equal(rt.logits(), want)
    fs.close()


def test_sm_share_compute_stream(setup):
    """GPU-share emulation: a runtime whose compute stream owns a fraction of
    the SMs (green context). Launches are sized for the partition (split
    counts, persistent grids), so its sums run in another order than the
    full-GPU runtime's: within tolerance of it, and bit-identical to itself
    wherever the merge point lands."""
    from paper_2410_03065_b200.runtime import GpuRuntime

    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.run(setup["tier"], T, C, 42, mbps=1000, mode="compute_only")
    full_kv = [_chunk_kv(rt, s, C) for s in range(0, T, C)]
    full = rt.logits()
    small = GpuRuntime(setup["dims"], max_tokens=T, max_chunk=C, compute_sms=16)
    try:
        tier = small.build_cache_tier(T, C, 42)
        small.run(tier, T, C, 42, mbps=1000, mode="compute_only")
        base = [small.read_chunk(s, C) for s in range(0, T, C)]
        base_lg = small.logits()
        for a, b in zip([_chunk_kv(small, s, C) for s in range(0, T, C)], full_kv):
            assert rel(a, b) <= 2e-2
        assert rel(base_lg, full) <= 2e-2
        r = small.run(tier, T, C, 42, mbps=1000, mode="cake")
        assert sorted(c.index for c in r.chunks) == list(range(T // C))
        assert [small.read_chunk(s, C) for s in range(0, T, C)] == base
        tier.close()
    finally:
        small.close()
