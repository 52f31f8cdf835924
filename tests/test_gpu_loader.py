"""The loader and scheduler on the GPU path, held to the reference's own
acceptance bars (proj/tests/acceptance.cpp), plus config 5's mid-run
bandwidth change.

* C6 analogue (acceptance.cpp:250-323, transfer.hpp SliceEvent): with the
  GPU sink (every released slice -> cudaMemcpyAsync into HBM), the released
  bits never run ahead of the trace integral by more than one quantum, and
  every 100 ms window on a 5 ms grid delivers 0.9-1.1 x the link rate.
* C2 analogue (acceptance.cpp:126-169): 60 jittered bidirectional GPU runs,
  each covering every chunk exactly once with a consistent merge point, and
  each assembling the same (bit-identical) cache from a poisoned pool.
* Config 5 (BASELINE.json, reference dynamic traces model.cpp:100-171): the
  link drops 8x mid-run; the merge point follows it and the bidirectional
  TTFT stays <= min(compute-only, I/O-only) under the same trace.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("mbps,quantum", [(2000, 1 << 20), (5000, 2 << 20), (10000, 4 << 20)])
def test_throttle_fidelity_on_the_gpu_sink(gpu, mbps, quantum):
    from paper_2410_03065_b200.cake import BandwidthTrace, Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C = 32768, 512
    rt = GpuRuntime("llama3_8b", n_layers=4, max_tokens=T, max_chunk=C)  # 16 KiB/token: a 512 MiB tier
    try:
        tier = rt.build_cache_tier(T, C, 42)
        total = rt.kv_bytes_per_token * T
        best = None
        for attempt in range(2):  # one retry absorbs a host deschedule, as the reference does
            r = rt.run(tier, T, C, 42, mbps=mbps, mode="io_only", quantum=quantum, record_slices=True)
            at, bits = rt.slices()
            assert len(at) == -(-total // quantum) and int(bits[-1]) == total * 8
            assert sorted(c.index for c in r.chunks) == list(range(T // C))
            # cumulative bound: never ahead of the integral by more than one quantum
            ahead = (bits.astype(np.float64) - mbps * at.astype(np.float64)).max()
            lead = Cake().fetch_latency(BandwidthTrace.constant(mbps), quantum, 0)
            begin, end, window = int(at[0]) - lead, int(at[-1]), 100_000
            lo, hi = 1.0, 1.0

            def cum(t):
                i = np.searchsorted(at, t, side="right")
                return 0 if i == 0 else int(bits[i - 1])

            for t in range(max(begin, 0), end - window + 1, 5000):
                ratio = (cum(t + window) - cum(t)) / (mbps * window)
                lo, hi = min(lo, ratio), max(hi, ratio)
            best = (ahead, lo, hi)
            if ahead <= quantum * 8 and lo >= 0.9 and hi <= 1.1:
                break
        ahead, lo, hi = best
        print(f"{mbps} mbps: ahead {ahead / 8 / 1024:.0f} KiB, windows [{lo:.3f}, {hi:.3f}]")
        assert ahead <= quantum * 8
        assert 0.9 <= lo and hi <= 1.1
        tier.close()
    finally:
        rt.close()


def test_jittered_runs_cover_every_chunk_once(gpu):
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C = 2048, 256
    rt = GpuRuntime("tiny", max_tokens=T, max_chunk=C)
    try:
        tier = rt.build_cache_tier(T, C, 5)
        rt.poison(0xFF)
        rt.run(tier, T, C, 5, mbps=4000, mode="compute_only")
        base = [rt.read_chunk(s, C) for s in range(0, T, C)]
        merges = set()
        for i in range(60):
            rt.poison(0xFF)
            r = rt.run(tier, T, C, 5, mbps=4000, mode="cake", jitter_max_us=400, jitter_seed=1000 + i)
            recs = sorted(r.chunks, key=lambda c: c.index)
            assert [c.index for c in recs] == list(range(T // C)), i
            assert all((c.side == "io") == (c.index >= r.merge_point) for c in recs), (i, r.merge_point)
            assert [rt.read_chunk(s, C) for s in range(0, T, C)] == base, (i, r.merge_point, r.raced_chunk)
            merges.add(r.merge_point)
        print(f"merge points seen: {sorted(merges)}")
        tier.close()
    finally:
        rt.close()


def test_merge_point_follows_a_mid_run_bandwidth_drop(gpu):
    from paper_2410_03065_b200.cake import BandwidthTrace
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C = 16384, 512
    rt = GpuRuntime("llama3_8b", n_layers=8, max_tokens=T, max_chunk=C)  # 32 KiB/token, 16 MiB chunks
    try:
        rt.calibrate(T, C, 42)
        tier = rt.build_cache_tier(T, C, 42)
        steady = BandwidthTrace.constant(128000)                    # 16 GB/s
        step = BandwidthTrace([(0, 128000.0), (10_000, 16000.0)])  # 16 -> 2 GB/s after 10 ms

        def best(trace, mode):
            return min((rt.run(tier, T, C, 42, trace=trace, mode=mode) for _ in range(2)),
                       key=lambda r: r.device_ttft_ms)

        r_steady = best(steady, "cake")
        r_step = best(step, "cake")
        c_only = best(step, "compute_only")
        io_only = best(step, "io_only")
        print(f"merge steady {r_steady.merge_point} -> step {r_step.merge_point}; TTFT {r_step.device_ttft_ms:.2f} ms "
              f"vs compute-only {c_only.device_ttft_ms:.2f}, io-only {io_only.device_ttft_ms:.2f}")
        assert r_step.merge_point > r_steady.merge_point  # slower link: compute takes more chunks
        assert sorted(c.index for c in r_step.chunks) == list(range(T // C))
        assert r_step.device_ttft_ms <= min(c_only.device_ttft_ms, io_only.device_ttft_ms) * 1.03 + 0.5
        tier.close()
    finally:
        rt.close()
