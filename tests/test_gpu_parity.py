"""GPU hot path vs the CPU oracle (oracle/llama_ref.c, pinned to
transformers.LlamaForCausalLM by tests/test_oracle_pinned.py) on identical
seeded inputs.

Every run starts from a POISONED device: the whole paged pool (both page
sets) and the staging buffers are filled with 0xFF bytes (bf16 NaN) first,
so a page a run should have written but did not shows up as NaN logits or a
byte mismatch — nothing can pass on bytes an earlier run left behind.

Tolerances (bf16 storage, fp32 accumulate):
  computed KV        RMS(gpu - cpu) / RMS(cpu) <= 2^-7 per layer tensor
  first-token logits RMS-normalised error <= 2^-7, cosine >= 0.999, the same top-1
  loaded KV          bit-exact vs the cache tier
  assembled cache    bit-exact across merge points and race outcomes (deterministic kernels)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2.0 ** -7
NAN = 0xFF  # poison byte: 0xFFFF is a bf16 NaN

CONFIGS = {
    # name: (dims, T, chunk, prompt seed)
    "tiny": ((2, 256, 4, 4, 64, 1024, 32000), 2048, 256, 44),
    "gqa_hd64": ((2, 512, 8, 2, 64, 1024, 32000), 1024, 256, 42),
    "gqa_hd128": ((2, 1024, 8, 2, 128, 2048, 32768), 1024, 512, 45),
    # GQA 8:1 (the Llama-3-70B grouping: 16 tokens x 8 heads per 128-row tile)
    "gqa8_hd128": ((2, 1024, 16, 2, 128, 2048, 32768), 1024, 256, 45),
}
# Prompt seeds are chosen so the oracle's top-1 is DECIDABLE at bf16: its lead over
# the runner-up is >= MIN_MARGIN of the logits' RMS (seed 42 on gqa_hd128 has a
# 0.2% lead, inside the bf16 noise, and flips with any change of summation order).
MIN_MARGIN = 0.02


def rms_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)))


def cos(a, b):
    return float(np.dot(a, b) / (np.linalg.norm(a) * np.linalg.norm(b)))


def top1_margin(want):
    w = np.sort(np.asarray(want, np.float64))[::-1]
    return float((w[0] - w[1]) / np.sqrt(np.mean(w ** 2)))


def logits_ok(got, want):
    assert top1_margin(want) >= MIN_MARGIN, ("ill-posed top-1 check: pick another prompt seed", top1_margin(want))
    assert np.isfinite(got).all()
    assert rms_rel(got, want) <= TOL, rms_rel(got, want)
    assert cos(got, want) >= 0.999
    assert int(got.argmax()) == int(want.argmax())


def prun(rt, *a, **k):
    """A run from a poisoned pool."""
    rt.poison(NAN)
    return rt.run(*a, **k)


@pytest.fixture(scope="module", params=list(CONFIGS))
def setup(request):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import llama_oracle
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    dims, T, C, seed = CONFIGS[request.param]
    rt = GpuRuntime(dims, max_tokens=T, max_chunk=C)
    rt.poison(NAN)
    tier = rt.build_cache_tier(T, C, seed)
    toks = Cake().token_stream(seed, T).astype(np.int32)
    ref = llama_oracle.LlamaRef(dims, T)
    for s in range(0, T, C):
        ref.prefill_chunk(toks[s:s + C], s)
    keys, prev = [], None
    for s in range(0, T, C):
        prev = Cake().chain_hash(prev, toks[s:s + C].astype(np.uint32))
        keys.append(prev)
    prun(rt, tier, T, C, seed, mbps=1000, mode="compute_only")
    base_kv = [rt.read_chunk(s, C) for s in range(0, T, C)]
    base_logits = rt.logits()
    prun(rt, tier, T, C, seed, mbps=64000, mode="io_only")
    io_logits = rt.logits()
    return {"rt": rt, "tier": tier, "ref": ref, "toks": toks, "T": T, "C": C, "dims": dims, "keys": keys, "seed": seed,
            "ref_logits": ref.final_logits(C - 1), "base_kv": base_kv, "base_logits": base_logits,
            "io_logits": io_logits}


def _chunk_kv(rt, s, c):
    import llama_oracle

    L, H, nh, nkv, hd, ffn, V = rt.dims
    b = np.frombuffer(rt.read_chunk(s, c), dtype=np.uint16)
    return llama_oracle.bf16_to_f32(b).reshape(L, 2, nkv, c, hd)


def test_tier_holds_the_computed_cache(setup):
    """build_cache_tier wrote the bytes a poisoned compute-only run computes."""
    for i, key in enumerate(setup["keys"]):
        assert setup["tier"].get(key) == setup["base_kv"][i], i


def test_computed_kv_matches_oracle(setup):
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    prun(rt, setup["tier"], T, C, setup["seed"], mbps=1000, mode="compute_only")
    kv = setup["ref"].kv()
    for s in range(0, T, C):
        got = _chunk_kv(rt, s, C)
        want = kv[:, :, :, s:s + C, :]
        assert np.isfinite(got).all(), s
        for layer in range(got.shape[0]):
            for k in range(2):
                assert rms_rel(got[layer, k], want[layer, k]) <= TOL, (s, layer, k, rms_rel(got[layer, k], want[layer, k]))


@pytest.mark.parametrize("mode", ["compute_only", "io_only"])
def test_first_token_logits_match_oracle(setup, mode):
    rt = setup["rt"]
    r = prun(rt, setup["tier"], setup["T"], setup["C"], setup["seed"], mbps=4000, mode=mode)
    assert r.recomputed_last == (mode == "io_only")
    logits_ok(rt.logits(), setup["ref_logits"])


def test_loaded_kv_bit_exact(setup):
    """I/O-only from a poisoned pool: every page was landed by the loader, byte for byte."""
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    r = prun(rt, setup["tier"], T, C, setup["seed"], mbps=40000, mode="io_only")
    assert r.merge_point == 0
    assert all(c.side == "io" for c in r.chunks)
    for i, s in enumerate(range(0, T, C)):
        assert rt.read_chunk(s, C) == setup["tier"].get(setup["keys"][i]), i
    assert np.array_equal(rt.logits(), setup["io_logits"])


@pytest.mark.parametrize("mbps", [200, 2000, 20000, 200000])
def test_assembled_cache_independent_of_merge_point(setup, mbps):
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    r = prun(rt, setup["tier"], T, C, setup["seed"], mbps=mbps, mode="cake")
    assert sorted(c.index for c in r.chunks) == list(range(T // C))
    for i, s in enumerate(range(0, T, C)):
        assert rt.read_chunk(s, C) == setup["base_kv"][i], (mbps, i, r.merge_point)
    want = setup["io_logits"] if r.recomputed_last else setup["base_logits"]
    assert np.array_equal(rt.logits(), want)
    logits_ok(rt.logits(), setup["ref_logits"])


# Forced boundary races (RunOptions::race_force / race_hold test hooks):
#   compute racer: a slow link keeps the loader on its first chunk while the
#   compute side runs out of chunks and contests it into the spare page set;
#   io racer: a fast link (one slice per chunk) lands the suffix while the
#   compute side is still on its last claimed chunk, which the loader contests.
# The hold decides who commits first; the assembled cache (through the final
# block table) and the logits must be those of the single-sided runs.
RACES = {
    "compute_racer_wins": dict(race_force=1, race_hold=1, mbps=100, racer="compute", winner=0),
    "compute_racer_loses": dict(race_force=1, race_hold=0, mbps=100, racer="compute", winner=1),
    "io_racer_wins": dict(race_force=2, race_hold=0, mbps=1_000_000, racer="io", winner=1),
    "io_racer_loses": dict(race_force=2, race_hold=1, mbps=1_000_000, racer="io", winner=0),
}


@pytest.mark.parametrize("case", list(RACES))
def test_forced_boundary_race(setup, case):
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    spec = RACES[case]
    n = T // C
    quantum = (1 << 20) if spec["racer"] == "compute" else rt.kv_bytes_per_token * C
    r = prun(rt, setup["tier"], T, C, setup["seed"], mbps=spec["mbps"], mode="cake", quantum=quantum,
             race_force=spec["race_force"], race_hold=spec["race_hold"])
    assert r.raced_chunk >= 0, case
    assert r.race_winner == spec["winner"], (case, r.raced_chunk, r.race_winner)
    if spec["racer"] == "compute":
        assert r.raced_chunk == n - 1  # the loader's first (slow) chunk
    else:
        assert r.raced_chunk < n - 1
    sides = {c.index: c.side for c in r.chunks}
    assert sorted(sides) == list(range(n))
    assert sides[r.raced_chunk] == ("compute" if spec["winner"] == 0 else "io")
    for i, s in enumerate(range(0, T, C)):
        assert rt.read_chunk(s, C) == setup["base_kv"][i], (case, i, r.raced_chunk)
    lg = rt.logits()
    want = setup["io_logits"] if r.recomputed_last else setup["base_logits"]
    assert np.array_equal(lg, want), case
    logits_ok(lg, setup["ref_logits"])


def test_tcgen05_attention_matches_mma_sync_kernel(setup):
    """The two independent attention kernels agree on the whole computed cache
    (bf16 P in both; only accumulation order differs)."""
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.set_attention_impl("mma_sync")
    try:
        prun(rt, setup["tier"], T, C, setup["seed"], mbps=1000, mode="compute_only")
        mma = [_chunk_kv(rt, s, C) for s in range(0, T, C)]
        lg_mma = rt.logits()
    finally:
        rt.set_attention_impl("tcgen05")
    for i, s in enumerate(range(0, T, C)):
        assert rms_rel(mma[i], _base(setup, i)) <= TOL
    assert rms_rel(lg_mma, setup["base_logits"]) <= TOL


def test_one_tile_kernel_matches_product(setup):
    """The column-split one-tile tcgen05 kernel (attention_tc.cuh, impl 2) against the product
    kernel (softmax warpgroups on alternate key blocks, attention_alt.cuh): the whole computed
    cache and the logits (same bf16 P; the per-group running max / the final merge differ)."""
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    rt.set_attention_impl("tcgen05_1tile")
    try:
        prun(rt, setup["tier"], T, C, setup["seed"], mbps=1000, mode="compute_only")
        one = [_chunk_kv(rt, s, C) for s in range(0, T, C)]
        lg = rt.logits()
    finally:
        rt.set_attention_impl("tcgen05")
    for i in range(len(one)):
        assert rms_rel(one[i], _base(setup, i)) <= TOL
    logits_ok(lg, setup["ref_logits"])


def _base(setup, i):
    import llama_oracle

    L, H, nh, nkv, hd, ffn, V = setup["dims"]
    C = setup["C"]
    return llama_oracle.bf16_to_f32(np.frombuffer(setup["base_kv"][i], dtype=np.uint16)).reshape(L, 2, nkv, C, hd)


@pytest.mark.parametrize("mode", ["cake", "io_only"])
def test_partially_cached_prompt(setup, mode):
    """Only a prefix of the prompt is in the tier (cached_prefix): the bidirectional
    phase covers it, the uncached suffix is computed after it. The assembled cache
    and the first-token logits are bit-identical to a full compute-only run."""
    rt, T, C = setup["rt"], setup["T"], setup["C"]
    cached = T // 2
    part = rt.build_cache_tier(cached, C, setup["seed"])
    r = prun(rt, part, T, C, setup["seed"], mbps=1000, mode=mode, cached_prefix=True)
    assert r.n_chunks == T // C
    assert sorted(c.index for c in r.chunks) == list(range(T // C))
    assert all(c.side == "compute" for c in r.chunks if c.index >= cached // C)
    assert r.merge_point <= cached // C
    assert not r.recomputed_last  # the computed suffix holds the last token's hidden state
    assert [rt.read_chunk(s, C) for s in range(0, T, C)] == setup["base_kv"]
    assert np.array_equal(rt.logits(), setup["base_logits"])
    with pytest.raises(Exception):
        rt.run(part, T, C, setup["seed"], mbps=1000, mode=mode)  # without the option a missing chunk is an error


@pytest.mark.parametrize("direct", [False, True])
def test_file_tier(setup, tmp_path, direct):
    """Cache tier on local disk in the reference's file format (one file per
    chunk + manifest), read by the loader with buffered or O_DIRECT reads:
    the assembled cache and the logits equal the pinned-memory tier's."""
    from paper_2410_03065_b200.cake import ChunkStore

    rt, T, C = setup["rt"], setup["T"], setup["C"]
    fs = ChunkStore(rt.n, str(tmp_path / f"tier{int(direct)}"), create=1)
    rt.build_cache_tier(T, C, setup["seed"], store=fs)
    fs.set_direct_io(direct)
    for mode in ("io_only", "cake"):
        r = prun(rt, fs, T, C, setup["seed"], mbps=8000, mode=mode)
        assert sorted(c.index for c in r.chunks) == list(range(T // C))
        assert [rt.read_chunk(s, C) for s in range(0, T, C)] == setup["base_kv"]
        assert np.array_equal(rt.logits(), setup["io_logits"] if r.recomputed_last else setup["base_logits"])
    fs.close()


def test_sm_share_compute_stream(setup):
    """GPU-share emulation: a runtime whose compute stream owns a fraction of
    the SMs (green context). Launches are sized for the partition (split
    counts, persistent grids), so its sums run in another order than the
    full-GPU runtime's: within tolerance of it, and bit-identical to itself
    wherever the merge point lands."""
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C = setup["T"], setup["C"]
    small = GpuRuntime(setup["dims"], max_tokens=T, max_chunk=C, compute_sms=16)
    try:
        small.poison(NAN)
        tier = small.build_cache_tier(T, C, setup["seed"])
        prun(small, tier, T, C, setup["seed"], mbps=1000, mode="compute_only")
        base = [small.read_chunk(s, C) for s in range(0, T, C)]
        base_lg = small.logits()
        for i, s in enumerate(range(0, T, C)):
            assert rms_rel(_chunk_kv(small, s, C), _base(setup, i)) <= TOL
        assert rms_rel(base_lg, setup["base_logits"]) <= TOL
        r = prun(small, tier, T, C, setup["seed"], mbps=1000, mode="cake")
        assert sorted(c.index for c in r.chunks) == list(range(T // C))
        assert [small.read_chunk(s, C) for s in range(0, T, C)] == base
        tier.close()
    finally:
        small.close()


RAGGED = {
    # T not a multiple of the chunk, nor of the 64-token page: a short last chunk ending mid-page
    "tiny_ragged": ((2, 256, 4, 4, 64, 1024, 32000), 1000, 256),
    "gqa8_ragged": ((2, 1024, 16, 2, 128, 2048, 32768), 1000, 256),
}


@pytest.mark.parametrize("name", list(RAGGED))
def test_ragged_prompt(name):
    """Short last chunk. The pool is poisoned with a finite pattern (0x5A5A):
    the tail page's unwritten slots are read as masked keys, so they must be
    ignored, not merely zero."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import llama_oracle
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    dims, T, C = RAGGED[name]
    rt = GpuRuntime(dims, max_tokens=1024, max_chunk=C)
    try:
        rt.poison(0x5A)
        tier = rt.build_cache_tier(T, C, 42)
        toks = Cake().token_stream(42, T).astype(np.int32)
        ref = llama_oracle.LlamaRef(dims, T)
        starts = list(range(0, T, C))
        for s in starts:
            ref.prefill_chunk(toks[s:s + C], s)
        want = ref.final_logits(T - starts[-1] - 1)
        kv = ref.kv()
        lens = [min(C, T - s) for s in starts]
        for mode in ("compute_only", "io_only", "cake"):
            rt.poison(0x5A)
            r = rt.run(tier, T, C, 42, mbps=2000, mode=mode)
            assert r.n_chunks == len(starts)
            logits_ok(rt.logits(), want)
            for s, n in zip(starts, lens):
                got = llama_oracle.bf16_to_f32(np.frombuffer(rt.read_chunk(s, n), dtype=np.uint16))
                got = got.reshape(dims[0], 2, dims[3], n, dims[4])
                assert rms_rel(got, kv[:, :, :, s:s + n]) <= TOL, (mode, s)
        tier.close()
    finally:
        rt.close()
