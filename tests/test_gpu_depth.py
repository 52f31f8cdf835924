"""Deep and long parity at the BASELINE model shapes, against the numpy oracle
(oracle/llama_np.py — the C oracle's restatement, both pinned to
transformers.LlamaForCausalLM by tests/test_oracle_pinned.py).

* Llama-3-8B, all 32 layers, T = 1024: every layer's computed KV and the
  first-token logits (compute-only, I/O-only and bidirectional runs).
* Llama-3-8B, 2 layers, T = 32768: the attention over long prefixes — split-KV
  with many splits, the fixed-order combine, and the 32K first-token step. The
  oracle starts from the GPU's own cache tier for the prefix (loaded KV is
  bit-exact, checked separately) and computes the chunk at 16K and the last
  chunk itself; the first-token step is checked on the loaded 32K cache.
* Llama-3-70B dimensions (H 8192, 64 q / 8 kv heads, FFN 28672), 2 layers.

Every GPU run starts from a NaN-poisoned pool (see test_gpu_parity.py).
Tolerances: RMS-normalised error <= 2^-7, cosine >= 0.999, identical top-1.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2.0 ** -7
L8B = (32, 4096, 32, 8, 128, 14336, 128256)
L70B = (80, 8192, 64, 8, 128, 28672, 128256)


def rms_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)))


def cos(a, b):
    return float(np.dot(a, b) / (np.linalg.norm(a) * np.linalg.norm(b)))


MIN_MARGIN = 0.02  # the oracle's top-1 lead over the runner-up, in logits RMS (see test_gpu_parity.py)


def logits_ok(got, want, what=""):
    w = np.sort(np.asarray(want, np.float64))[::-1]
    margin = float((w[0] - w[1]) / np.sqrt(np.mean(w ** 2)))
    assert margin >= MIN_MARGIN, ("ill-posed top-1 check: pick another prompt seed", what, margin)
    assert np.isfinite(got).all(), what
    e = rms_rel(got, want)
    assert e <= TOL, (what, e)
    assert cos(got, want) >= 0.999, what
    assert int(got.argmax()) == int(want.argmax()), (what, int(got.argmax()), int(want.argmax()))


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _kv(rt, s, c):
    import llama_oracle

    L, H, nh, nkv, hd, ffn, V = rt.dims
    return llama_oracle.bf16_to_f32(np.frombuffer(rt.read_chunk(s, c), dtype=np.uint16)).reshape(L, 2, nkv, c, hd)


def _keys(toks, C):
    from paper_2410_03065_b200.cake import Cake

    keys, prev = [], None
    for s in range(0, len(toks), C):
        prev = Cake().chain_hash(prev, toks[s:s + C].astype(np.uint32))
        keys.append(prev)
    return keys


def _full_depth(dims, T, C, seed, n_layers=None):
    import llama_np
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    L = n_layers or dims[0]
    dims = (L,) + tuple(dims[1:])
    rt = GpuRuntime(dims, max_tokens=T, max_chunk=C)
    rt.poison(0xFF)
    tier = rt.build_cache_tier(T, C, seed)
    toks = Cake().token_stream(seed, T).astype(np.int32)
    ref = llama_np.LlamaNp(dims, T)
    ref.prefill(toks, 0)
    want = ref.final_logits(T - 1)
    kv_errs = []
    for mode in ("compute_only", "io_only", "cake"):
        rt.poison(0xFF)
        r = rt.run(tier, T, C, seed, mbps=64000, mode=mode)
        assert sorted(c.index for c in r.chunks) == list(range(T // C))
        logits_ok(rt.logits(), want, mode)
        if mode == "compute_only":
            for s in range(0, T, C):
                got = _kv(rt, s, C)
                assert np.isfinite(got).all()
                for layer in range(L):
                    for k in range(2):
                        e = rms_rel(got[layer, k], ref.kv[layer, k, :, s:s + C])
                        kv_errs.append(e)
                        assert e <= TOL, (s, layer, k, e)
    tier.close()
    rt.close()
    return max(kv_errs)


def test_8b_full_depth_vs_oracle(gpu):
    """All 32 layers of the Llama-3-8B shape, 1024 tokens in two 512-token chunks."""
    worst = _full_depth(L8B, 1024, 512, 7)
    print(f"8B 32-layer worst per-layer KV rms err {worst:.2e}")


def test_70b_dims_two_layers_vs_oracle(gpu):
    """Llama-3-70B dimensions (H 8192, 64/8 heads, FFN 28672, vocab 128256), 2 layers."""
    worst = _full_depth(L70B, 1024, 512, 11, n_layers=2)
    print(f"70B-dim 2-layer worst per-layer KV rms err {worst:.2e}")


def test_8b_long_prefix_vs_oracle(gpu):
    """2 layers of the 8B shape at T = 32768 (64 chunks of 512)."""
    import llama_np
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C, seed = 32768, 512, 42
    dims = (2,) + L8B[1:]
    n = T // C
    rt = GpuRuntime(dims, max_tokens=T, max_chunk=C)
    rt.poison(0xFF)
    tier = rt.build_cache_tier(T, C, seed)
    toks = Cake().token_stream(seed, T).astype(np.int32)
    keys = _keys(toks, C)
    ref = llama_np.LlamaNp(dims, T)
    for i in range(n - 1):
        ref.load_chunk(tier.get(keys[i]), i * C, C)

    # the chunk at 16K and the last chunk, computed by the oracle over the GPU's prefix
    def kv_of(i):
        import llama_oracle

        return llama_oracle.bf16_to_f32(np.frombuffer(tier.get(keys[i]), dtype=np.uint16)).reshape(2, 2, 8, C, 128)

    mid = n // 2
    ref.prefill(toks[mid * C:(mid + 1) * C], mid * C)
    got, want = kv_of(mid), ref.chunk_tier(mid * C, C)
    for layer in range(2):
        for k in range(2):
            assert rms_rel(got[layer, k], want[layer, k]) <= TOL, ("mid", layer, k)
    ref.load_chunk(tier.get(keys[mid]), mid * C, C)  # back to the GPU's bytes for the prefix
    ref.prefill(toks[T - C:], T - C)
    got, want = kv_of(n - 1), ref.chunk_tier(T - C, C)
    for layer in range(2):
        for k in range(2):
            assert rms_rel(got[layer, k], want[layer, k]) <= TOL, ("last", layer, k)
    want_logits = ref.final_logits(C - 1)

    rt.poison(0xFF)
    r = rt.run(tier, T, C, seed, mbps=256000, mode="compute_only")
    logits_ok(rt.logits(), want_logits, "compute_only")
    for i in (0, mid, n - 1):
        assert rt.read_chunk(i * C, C) == tier.get(keys[i])

    # first-token step over the loaded 32K cache (the recompute path: split-KV decode + combine)
    ref.load_chunk(tier.get(keys[n - 1]), T - C, C)
    want_step = ref.last_token_logits(int(toks[T - 1]), T)
    rt.poison(0xFF)
    r = rt.run(tier, T, C, seed, mbps=256000, mode="io_only")
    assert r.recomputed_last
    for i in range(n):
        assert rt.read_chunk(i * C, C) == tier.get(keys[i]), i
    logits_ok(rt.logits(), want_step, "io_only 32K first-token step")

    rt.poison(0xFF)
    r = rt.run(tier, T, C, seed, mbps=64000, mode="cake")
    assert sorted(c.index for c in r.chunks) == list(range(n))
    for i in range(n):
        assert rt.read_chunk(i * C, C) == tier.get(keys[i]), (i, r.merge_point)
    logits_ok(rt.logits(), want_step if r.recomputed_last else want_logits, "cake")
    tier.close()
    rt.close()
