"""Concurrent requests on one B200 (paper_2410_03065_b200/serve.py): two
contexts sharing one weight copy and one emulated link serve a mix of prompts
at the same time. Every request's assembled cache is byte-identical, and its
first-token logits bit-identical, to the same prompt served alone — from a
NaN-poisoned pool — whatever the other request did to the link and the SMs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (2, 512, 8, 2, 64, 1024, 32000)
T, C = 1024, 256
SEEDS = [42, 45, 46, 47]


@pytest.fixture(scope="module")
def server():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_03065_b200.serve import GpuServer

    srv = GpuServer(DIMS, workers=2, mbps=400, max_tokens=T, max_chunk=C)
    yield srv
    srv.close()


def test_concurrent_requests_match_solo(server):
    from paper_2410_03065_b200.serve import Request

    rt = server.primary
    tiers, base_kv, base_lg, io_lg = {}, {}, {}, {}
    for s in SEEDS:
        tiers[s] = rt.build_cache_tier(T, C, s)
    rt.attach_link(None)  # solo references: the request alone on its own 400 mbps link
    for s in SEEDS:
        rt.poison(0xFF)
        rt.run(tiers[s], T, C, s, mbps=400, mode="compute_only")
        base_kv[s] = [rt.read_chunk(o, C) for o in range(0, T, C)]
        base_lg[s] = rt.logits()
        rt.poison(0xFF)
        rt.run(tiers[s], T, C, s, mbps=40000, mode="io_only")
        io_lg[s] = rt.logits()
        assert [rt.read_chunk(o, C) for o in range(0, T, C)] == base_kv[s]
    rt.attach_link(server.link)
    for w in server.runtimes:
        w.poison(0xFF)

    modes = ["io_only", "cake", "io_only", "cake"]
    reqs = [Request(tiers[s], T, C, s, mode=m) for s, m in zip(SEEDS, modes)]
    checked = []

    def after(sv, w):
        s = SEEDS[sv.index]
        got = [w.read_chunk(o, C) for o in range(0, T, C)]
        assert got == base_kv[s], (sv.index, sv.worker)
        want = io_lg[s] if sv.result.recomputed_last else base_lg[s]
        assert np.array_equal(sv.logits, want), (sv.index, sv.worker)
        checked.append(sv.index)
        w.poison(0xFF)  # the next request on this context starts from NaN pages

    out = server.serve(reqs, keep_logits=True, after=after)
    assert sorted(checked) == list(range(len(reqs)))
    assert {sv.worker for sv in out} == {0, 1}
    # the two contexts ran at the same time
    by_w = {w: [sv for sv in out if sv.worker == w] for w in (0, 1)}
    assert any(a.start_ms < b.end_ms and b.start_ms < a.end_ms for a in by_w[0] for b in by_w[1])
    # every io-landed byte went through the one link
    io_bytes = sum(c.bytes for sv in out for c in sv.result.chunks if c.side == "io")
    bits, _ = server.link.reserved()
    assert bits >= io_bytes * 8 > 0


def test_shared_link_halves_each_requests_rate(server):
    """Two I/O-only requests at once on one link take about twice as long as one."""
    from paper_2410_03065_b200.serve import Request

    rt = server.primary
    tiers = [rt.build_cache_tier(T, C, s) for s in SEEDS[:2]]
    solo = server.serve([Request(tiers[0], T, C, SEEDS[0], mode="io_only")])[0]
    pair = server.serve([Request(t, T, C, s, mode="io_only") for t, s in zip(tiers, SEEDS[:2])])
    assert {sv.worker for sv in pair} == {0, 1}
    slowest = max(sv.result.kv_resident_ms for sv in pair)
    assert slowest >= 1.6 * solo.result.kv_resident_ms, (slowest, solo.result.kv_resident_ms)
