"""B200 library vs the reference library (built from /root/reference sources) on the
same seeded inputs: identical results for every deterministic call, store interop
in both directions, identical error classes. Skips when oracle/_ref is absent."""
import os
import random

import pytest

from paper_2410_03065_b200.cake import BandwidthTrace, CostModel, RunPlan
from paper_2410_03065_b200.native import CorruptChunkError, MissingKeyError


def rand_plan(rng):
    n = 1 + rng.randrange(64)
    chunk = 1 + rng.randrange(1024)
    per_token = 1000 + rng.randrange(1000000)
    counts = [chunk] * n
    if rng.randrange(3) == 0:
        counts[-1] = 1 + rng.randrange(chunk)
    starts = [sum(counts[:i]) for i in range(n)]
    b = [per_token * c for c in counts]
    return RunPlan(starts, counts, b, b), CostModel(0.1 + rng.randrange(500) / 10, rng.randrange(50) / 1000, chunk)


def test_sim_fuzz_identical(cake_b200, cake_ref):
    rng = random.Random(99)
    for _ in range(300):
        plan, cost = rand_plan(rng)
        trace = BandwidthTrace.constant(100 + rng.randrange(39900))
        power = rng.choice([0.1, 0.5, 1.0])
        dec = rng.choice([0.0, 0.001])
        for mode in ("cake", "io_only", "compute_only"):
            kw = dict(token_budget=max(512, cost.reference_chunk_size), decode_us_per_byte=dec)
            a = cake_b200.run_sim_planned(plan, cost, trace, mode, power, **kw)
            b = cake_ref.run_sim_planned(plan, cost, trace, mode, power, **kw)
            assert a == b


def test_dynamic_trace_fetch_identical(cake_b200, cake_ref):
    rng = random.Random(5)
    for _ in range(300):
        pts, t = [], 0
        for _ in range(1 + rng.randrange(5)):
            rate = rng.choice([100 + rng.randrange(50000), 100.5 + rng.random() * 5000])
            pts.append((t, rate))
            t += 1 + rng.randrange(3000000)
        tr = BandwidthTrace(pts)
        bits = rng.randrange(1 << 40)
        start = rng.randrange(5000000)
        assert cake_b200.time_to_transfer_bits(tr, bits, start) == cake_ref.time_to_transfer_bits(tr, bits, start)


def test_errors_match(cake_b200, cake_ref):
    for lib in (cake_b200, cake_ref):
        with pytest.raises(ValueError):
            lib.split_into_chunks(0, 512)
        with pytest.raises(ValueError):
            lib.compute_latency(CostModel(1, 0, 512), 0, 512, 0.0)
        with pytest.raises(ValueError):
            lib.oracle_best_split([1, 2], [1])
        with pytest.raises(ValueError):
            lib.fetch_latency(BandwidthTrace([(5, 100.0)]), 10)


@pytest.mark.parametrize("writer,reader", [("ref", "b200"), ("b200", "ref")])
def test_store_interop(tmp_path, cake_b200, cake_ref, writer, reader):
    libs = {"ref": cake_ref, "b200": cake_b200}
    root = str(tmp_path / "store")
    w = libs[writer].store(root, create=1)
    keys = w.populate(3000, 512, (2, 256, 2), "identity", seed=11)
    qkeys = libs[writer].store(str(tmp_path / "q8"), create=1).populate(1024, 256, (2, 128, 2), "quant8", seed=3)
    w.close()
    r = libs[reader].store(root, create=0)
    assert r.entry_count() == len(keys)
    for i, k in enumerate(keys):
        n = (512 if i < len(keys) - 1 else 3000 - 512 * (len(keys) - 1)) * 2 * 2 * 256 * 2
        assert r.get(k) == libs[writer].synth_payload(11, i, n)
    with pytest.raises(MissingKeyError):
        r.get(b"\x00" * 32)
    assert len(qkeys) == 4


def test_truncated_chunk_is_corrupt(tmp_path, cake_b200, cake_ref):
    for name, lib in (("b", cake_b200), ("r", cake_ref)):
        root = tmp_path / name
        s = lib.store(str(root), create=1)
        keys = s.populate(1024, 512, (1, 64, 2), "identity", seed=1)
        s.close()
        hx = keys[0].hex()
        path = root / hx[:2] / (hx + ".kv")
        data = path.read_bytes()
        path.write_bytes(data[:-10])
        with pytest.raises(CorruptChunkError):
            lib.store(str(root), create=0)


def test_live_modeled_run_same_split(tmp_path, cake_b200, cake_ref):
    """Live (threads + throttle + real file reads, modeled compute) on both
    implementations: same exactly-once coverage and a merge point within one
    chunk of the simulator's (live timing jitter)."""
    for lib in (cake_b200, cake_ref):
        s = lib.store(str(tmp_path / ("s" + str(id(lib)))), create=1)
        s.populate(2048, 256, (2, 256, 2), "identity", seed=42)
        cost = CostModel(12.0, 0.02, 256)
        tr = BandwidthTrace.constant(400)
        sim = lib.run(s, 2048, 256, (2, 256, 2), "identity", cost, tr, "cake", "sim", 42,
                      throttle_quantum_bytes=64 << 10)
        live = lib.run(s, 2048, 256, (2, 256, 2), "identity", cost, tr, "cake", "live", 42,
                       throttle_quantum_bytes=64 << 10)
        assert sorted(c.index for c in live.chunks) == list(range(8))
        assert abs(live.merge_point - sim.merge_point) <= 1


def test_cached_prefix_plan(tmp_path, cake_b200):
    """B200 extension (RunOptions::cached_prefix): a store holding only the first
    chunks of the prompt. Without the option the run fails like the reference
    (MissingKeyError for the first absent chunk); with it the plan splits into the
    cached prefix and an uncached suffix, which only a GPU live run can compute;
    on a fully cached prompt the option changes nothing."""
    s = cake_b200.store(str(tmp_path / "part"), create=1)
    s.populate(1024, 256, (2, 256, 2), "identity", seed=42)  # chunks 0..3 of an 8-chunk prompt
    cost = CostModel(12.0, 0.02, 256)
    tr = BandwidthTrace.constant(400)
    with pytest.raises(MissingKeyError):
        cake_b200.run(s, 2048, 256, (2, 256, 2), "identity", cost, tr, "cake", "sim", 42)
    with pytest.raises(ValueError, match="GPU live run"):
        cake_b200.run(s, 2048, 256, (2, 256, 2), "identity", cost, tr, "cake", "sim", 42, cached_prefix=True)
    full = cake_b200.run(s, 1024, 256, (2, 256, 2), "identity", cost, tr, "cake", "sim", 42)
    opt = cake_b200.run(s, 1024, 256, (2, 256, 2), "identity", cost, tr, "cake", "sim", 42, cached_prefix=True)
    assert (full.ttft_us, full.merge_point) == (opt.ttft_us, opt.merge_point)
    # a prompt whose first chunk is absent has no cached prefix at all
    empty = cake_b200.store(str(tmp_path / "none"), create=1)
    with pytest.raises(MissingKeyError):
        cake_b200.run(empty, 1024, 256, (2, 256, 2), "identity", cost, tr, "cake", "sim", 42, cached_prefix=True)
