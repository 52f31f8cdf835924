"""bench.py host logic (no GPU): the workload config both arms print, and the
TTFT roofline (the reference's oracle_best_split over ideal chunk times)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_both_arms_share_the_workload_config():
    a = bench.workload_config(32768, 512, 64000.0, 1)
    b = dict(bench.workload_config(32768, 512, 64000.0, 1), parallelism="host CPU")
    for k in ("workload", "model", "seq_len", "chunk", "link_mbps"):
        assert a[k] == b[k]
    assert "8 GB/s" in a["workload"] and a["parallelism"] == "1 GPU"
    assert bench.workload_config(32768, 512, 64000.0, 4)["parallelism"].startswith("tp4")


def test_roofline_bounds_and_split():
    r = bench.ttft_roofline_ms(bench.DIMS_8B, 32768, 512, 64000.0, 1368.1, 6650.0)
    assert r["n_chunks"] == 64
    assert 0 <= r["k_star"] <= 64
    # bidirectional is no worse than either side alone, and beats both at 8 GB/s
    assert r["bidir_ms"] <= min(r["compute_only_ms"], r["io_only_ms"]) + 1e-6
    assert r["bidir_ms"] < 0.6 * min(r["compute_only_ms"], r["io_only_ms"])
    # I/O-only = chunk bytes over the emulated link (+ the first-token step)
    kv_tok = 2 * 32 * 8 * 128 * 2
    assert abs(r["io_only_ms"] - (32768 * kv_tok / 8e9 * 1e3)) < 10.0


def test_roofline_tp_scales_both_sides():
    one = bench.ttft_roofline_ms(bench.DIMS_8B, 16384, 512, 64000.0, 1368.1, 6650.0)
    two = bench.ttft_roofline_ms(bench.DIMS_8B, 16384, 512, 64000.0, 1368.1, 6650.0, tp=2)
    assert two["compute_only_ms"] < 0.55 * one["compute_only_ms"]
    assert two["io_only_ms"] < 0.55 * one["io_only_ms"]
