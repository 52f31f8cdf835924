"""Llama-3-8B shape on the B200.

(oracle parity at this shape: tests/test_gpu_depth.py)

* full depth, BASELINE config sizes (32K context): size-independent properties —
  every loaded chunk bit-exact vs the cache tier, the assembled cache bit-identical
  to the compute-only cache wherever the merge point lands, exactly-once coverage,
  and bidirectional TTFT <= min(compute-only, I/O-only) at each emulated bandwidth.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (32, 4096, 32, 8, 128, 14336, 128256)


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def test_8b_full_32k_properties(gpu):
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C, seed = 32768, 512, 42
    rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=C)
    rt.calibrate(T, C, seed)
    tier = rt.build_cache_tier(T, C, seed)
    n = T // C
    rt.poison(0xFF)
    c_only = rt.run(tier, T, C, seed, mbps=64000, mode="compute_only")
    sample = sorted({0, 1, n // 2, n - 2, n - 1})
    base = {i: rt.read_chunk(i * C, C) for i in sample}
    toks = Cake().token_stream(seed, T).astype(np.uint32)
    keys, prev = [], None
    for s in range(0, T, C):
        prev = Cake().chain_hash(prev, toks[s:s + C])
        keys.append(prev)
    for i in sample:  # the tier was written by the same kernels: computed == stored
        assert base[i] == tier.get(keys[i])
    for mbps in (16000, 64000, 256000):
        io_only = rt.run(tier, T, C, seed, mbps=mbps, mode="io_only")
        rt.poison(0xFF)
        r = rt.run(tier, T, C, seed, mbps=mbps, mode="cake")
        assert sorted(c.index for c in r.chunks) == list(range(n))
        assert all((c.side == "compute") == (c.index < r.merge_point) for c in r.chunks)
        for i in range(n):  # from a poisoned pool: every chunk landed or computed in this run
            assert rt.read_chunk(i * C, C) == (base[i] if i in base else tier.get(keys[i])), (mbps, i, r.merge_point)
        # bidirectional never loses to the better single-sided mode (small slack for device jitter)
        assert r.device_ttft_ms <= min(c_only.device_ttft_ms, io_only.device_ttft_ms) * 1.03 + 1.0, \
            (mbps, r.device_ttft_ms, c_only.device_ttft_ms, io_only.device_ttft_ms)
