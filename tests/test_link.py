"""One emulated link shared by concurrent loaders (cake/transfer.hpp SharedLink,
C ABI cake_link_*): the multi-request mix's bandwidth model, on the CPU live
path (threads + throttle + real store reads, reference proj/src/transfer.cpp:174-228).

* alone, a loader attached to the link runs at the trace rate (the same gate
  law as its own budget);
* two loaders on one link together deliver at the trace rate: each takes about
  twice as long, and the link's clock never runs ahead of the bits it granted.
"""
import threading

from paper_2410_03065_b200.cake import BandwidthTrace, CostModel
from paper_2410_03065_b200.runtime import Link

PROFILE = (2, 256, 2)  # 2048 B of KV per token
T, C = 2048, 256       # 8 chunks of 512 KiB
MBPS = 400.0           # 50 MB/s: 4 MiB per request in ~84 ms
Q = 64 << 10


def _store(lib, tmp_path, name, seed):
    s = lib.store(str(tmp_path / name), create=1)
    s.populate(T, C, PROFILE, "identity", seed=seed)
    return s


def _io_only(lib, store, seed, **kw):
    return lib.run(store, T, C, PROFILE, "identity", CostModel(12.0, 0.02, C), BandwidthTrace.constant(MBPS),
                   "io_only", "live", seed, throttle_quantum_bytes=Q, **kw)


def test_link_alone_matches_own_budget(tmp_path, cake_b200):
    s = _store(cake_b200, tmp_path, "a", 1)
    own = _io_only(cake_b200, s, 1)
    link = Link(mbps=MBPS)
    shared = _io_only(cake_b200, s, 1, link=link)
    assert sorted(c.index for c in shared.chunks) == list(range(T // C))
    assert abs(shared.ttft_us - own.ttft_us) <= 0.1 * own.ttft_us + 5000, (shared.ttft_us, own.ttft_us)
    bits, _ = link.reserved()
    assert bits == T * 2048 * 8
    link.close()


def test_two_loaders_share_the_rate(tmp_path, cake_b200):
    stores = [_store(cake_b200, tmp_path, f"s{i}", 10 + i) for i in range(2)]
    solo = _io_only(cake_b200, stores[0], 10)
    link = Link(mbps=MBPS)
    out = [None, None]

    def go(i):
        out[i] = _io_only(cake_b200, stores[i], 10 + i, link=link)

    th = [threading.Thread(target=go, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    bits, now_us = link.reserved()
    total = 2 * T * 2048 * 8
    assert bits == total
    for r in out:
        assert sorted(c.index for c in r.chunks) == list(range(T // C))
        # interleaved on one link: each request waits for the other's slices
        assert r.ttft_us >= 1.6 * solo.ttft_us, (r.ttft_us, solo.ttft_us)
    # the link granted `total` bits at MBPS: its clock is at least that far along
    # (less the one quantum a stalled source may bank)
    assert now_us >= total / MBPS - Q * 8 / MBPS - 1000, (now_us, total / MBPS)
    link.close()
