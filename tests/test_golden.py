"""Golden vectors of the reference (tests/golden/ref_golden.json: known answers quoted
from proj/tests/*.cpp plus outputs of the reference library built from source, made
by tests/golden/make_golden.py). Checked against BOTH the CPU oracle restatement
(oracle/sched_ref.py) — which pins the oracle — and the B200 library."""
import hashlib
import json
import os

import pytest

import sched_ref
from conftest import ROOT
from paper_2410_03065_b200.cake import BandwidthTrace, CostModel, RunPlan

G = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")))
K = G["known"]


def _trace(pts):
    return BandwidthTrace([tuple(p) for p in pts])


# ---------------------------------------------------------------- oracle pinning
def test_oracle_known_answers():
    for case in K["compute_latency"]:
        assert sched_ref.compute_latency(*case["args"]) == case["want"]
    for case in K["fetch_latency"]:
        assert sched_ref.fetch_latency(case["trace"], case["nbytes"], case["start"]) == case["want"]
    for case in K["oracle_best_split"]:
        assert list(sched_ref.oracle_best_split(case["c"], case["f"])) == case["want"]
    law = [sched_ref.compute_latency(10.0, 0.01, 512, 512 * i, 512) for i in range(64)]
    assert sum(law) == K["closed_form_64"]


def test_oracle_reproduces_reference_fetch_latencies():
    checked = 0
    for case in G["fetch"]:
        if any(p[1] != int(p[1]) for p in case["trace"]):
            continue  # reference uses long double on fractional rates; python has double only
        assert sched_ref.fetch_latency(case["trace"], case["nbytes"], case["start"]) == case["want"]
        checked += 1
    assert checked > 50


def test_oracle_reproduces_reference_simulator():
    for inst in G["sim"]:
        a, b, ref = inst["cost"]
        comp = [sched_ref.compute_latency(a, b, ref, s, c, inst["power"]) for s, c in zip(inst["starts"], inst["counts"])]
        pts = [[0, inst["mbps"]]]
        fetch = lambda i, t: sched_ref.fetch_latency(pts, inst["bytes"][i], t)  # noqa: E731
        n = len(inst["counts"])
        ttft, merge, rows = sched_ref.sim_bidirectional(comp, fetch, n)
        want = inst["want"]["cake"]
        assert (ttft, merge) == (want["ttft"], want["merge"])
        assert [[r.index, r.side, r.start, r.finish] for r in rows] == want["rows"]
        assert sched_ref.sim_compute_only(comp) == inst["want"]["compute_only"]["ttft"]
        assert sched_ref.sim_io_only(fetch, n) == inst["want"]["io_only"]["ttft"]


# ---------------------------------------------------------------- B200 library
def test_b200_known_answers(cake_b200):
    for case in K["kv_bytes"]:
        assert cake_b200.kv_bytes_per_token(*case["args"]) == case["want"]
    for case in K["compute_latency"]:
        a, b, ref, start, count, power = case["args"]
        assert cake_b200.compute_latency(CostModel(a, b, ref), start, count, power) == case["want"]
    for case in K["fetch_latency"]:
        assert cake_b200.fetch_latency(_trace(case["trace"]), case["nbytes"], case["start"]) == case["want"]
    for case in K["oracle_best_split"]:
        assert list(cake_b200.oracle_best_split(case["c"], case["f"])) == case["want"]


def test_b200_worked_example(cake_b200):
    ex = K["worked_example"]
    plan = RunPlan([512 * i for i in range(4)], [512] * 4, ex["bytes"], ex["bytes"])
    for mode in ("cake", "io_only", "compute_only"):
        r = cake_b200.run_sim_planned(plan, CostModel(*ex["cost"]), BandwidthTrace.constant(ex["mbps"]), mode)
        assert (r.ttft_us, r.merge_point) == (ex[mode]["ttft"], ex[mode]["merge"])


def test_b200_fetch_latency_matches_reference_outputs(cake_b200):
    for case in G["fetch"]:  # includes fractional-rate traces (long-double path)
        assert cake_b200.fetch_latency(_trace(case["trace"]), case["nbytes"], case["start"]) == case["want"]


def test_b200_simulator_matches_reference_outputs(cake_b200):
    for inst in G["sim"]:
        plan = RunPlan(inst["starts"], inst["counts"], inst["bytes"], inst["bytes"])
        for mode, want in inst["want"].items():
            r = cake_b200.run_sim_planned(plan, CostModel(*inst["cost"]), BandwidthTrace.constant(inst["mbps"]), mode,
                                          inst["power"], token_budget=max(512, inst["cost"][2]))
            assert (r.ttft_us, r.merge_point) == (want["ttft"], want["merge"])
            assert [[c.index, c.side, c.start_us, c.finish_us] for c in r.chunks] == want["rows"]


def test_b200_hash_tokens_payload_codec(cake_b200):
    h = G["hash"]
    toks = cake_b200.token_stream(42, 64)
    assert [int(x) for x in toks] == h["token_stream_42_64"]
    k0 = cake_b200.chain_hash(None, toks[:32])
    k1 = cake_b200.chain_hash(k0, toks[32:])
    assert [k0.hex(), k1.hex()] == h["chain"]
    assert hashlib.sha256(cake_b200.synth_payload(42, 3, 4098)).hexdigest() == h["synth_payload_sha256"]
    for c in G["codec"]:
        p = cake_b200.synth_payload(c["seed"], c["index"], c["n"])
        enc = cake_b200.codec_encode(c["codec"], p)
        assert len(enc) == c["enc_len"] and hashlib.sha256(enc).hexdigest() == c["enc_sha256"]
        dec = cake_b200.codec_decode(c["codec"], enc, c["n"])
        assert hashlib.sha256(dec).hexdigest() == c["dec_sha256"]


def test_b200_fp16_round_trip_all_finite_halves(cake_b200):
    """proj/tests/test_codec.cpp:141-151: every finite binary16 survives to-float-and-back."""
    import numpy as np

    bad = 0
    for h in range(0, 1 << 16, 7):  # stride keeps the CPU suite fast; the C++ suite covers all 63,488
        if (h & 0x7C00) == 0x7C00:
            continue
        if cake_b200.fp16_from_float(cake_b200.fp16_to_float(h)) != h:
            bad += 1
    assert bad == 0
    assert np.isinf(cake_b200.fp16_to_float(0x7C00))
