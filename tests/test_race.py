"""Race-to-finish at the merge boundary, on the virtual clock.

The reference guarantees TTFT <= min(baselines) + one chunk (the
slack is real — BASELINE.md §2: 13.7 ms cake vs 10.2 ms io_only at 4000 mbps).
With the boundary race the bound is strict: TTFT <= min(compute_only, io_only),
every chunk still has exactly one committed source, and with the race off the
library is bit-identical to the reference (tests/test_golden.py)."""
import random

import sched_ref
from paper_2410_03065_b200.cake import BandwidthTrace, CostModel, RunPlan


def fuzz(rng):
    n = 1 + rng.randrange(64)
    chunk = 1 + rng.randrange(1024)
    per_token = 1000 + rng.randrange(1000000)
    counts = [chunk] * n
    if rng.randrange(3) == 0:
        counts[-1] = 1 + rng.randrange(chunk)
    starts = [sum(counts[:i]) for i in range(n)]
    b = [per_token * c for c in counts]
    cost = CostModel(0.1 + rng.randrange(500) / 10, rng.randrange(50) / 1000, chunk)
    return RunPlan(starts, counts, b, b), cost, BandwidthTrace.constant(100 + rng.randrange(39900)), \
        rng.choice([0.1, 0.25, 0.5, 1.0])


def test_strict_dominance_and_exactly_once(cake_b200):
    rng = random.Random(2024)
    strict_wins = 0
    for _ in range(600):
        plan, cost, trace, power = fuzz(rng)
        kw = dict(token_budget=max(512, cost.reference_chunk_size))
        race = cake_b200.run_sim_planned(plan, cost, trace, "cake", power, race_to_finish=True, **kw)
        greedy = cake_b200.run_sim_planned(plan, cost, trace, "cake", power, **kw)
        c_only = cake_b200.run_sim_planned(plan, cost, trace, "compute_only", power, **kw)
        io_only = cake_b200.run_sim_planned(plan, cost, trace, "io_only", power, **kw)
        assert sorted(c.index for c in race.chunks) == list(range(plan.n))
        assert race.ttft_us <= min(c_only.ttft_us, io_only.ttft_us)
        assert race.ttft_us <= greedy.ttft_us
        # the committed split is a prefix + suffix at merge_point
        assert all((c.side == "compute") == (c.index < race.merge_point) for c in race.chunks)
        strict_wins += race.ttft_us < greedy.ttft_us
    assert strict_wins > 0  # the race actually matters on some instances


def test_reference_counterexample_is_fixed(cake_b200):
    """BASELINE.md §2 config-1 shape at 4000 mbps: greedy cake (12.0 ms sim) loses to
    io_only (8.4 ms sim); with the race the loader takes chunk 0 too."""
    counts = [256] * 8
    b = [256 * 2048] * 8
    plan = RunPlan([256 * i for i in range(8)], counts, b, b)
    cost = CostModel(12.0, 0.02, 256)
    tr = BandwidthTrace.constant(4000)
    greedy = cake_b200.run_sim_planned(plan, cost, tr, "cake")
    io = cake_b200.run_sim_planned(plan, cost, tr, "io_only")
    race = cake_b200.run_sim_planned(plan, cost, tr, "cake", race_to_finish=True)
    assert greedy.ttft_us > io.ttft_us
    assert race.ttft_us <= io.ttft_us
    assert race.merge_point == 0


def test_library_race_matches_oracle_restatement(cake_b200):
    rng = random.Random(7)
    for _ in range(300):
        plan, cost, trace, power = fuzz(rng)
        r = cake_b200.run_sim_planned(plan, cost, trace, "cake", power, race_to_finish=True,
                                      token_budget=max(512, cost.reference_chunk_size))
        comp = [sched_ref.compute_latency(cost.alpha_ms, cost.beta_ms_per_token, cost.reference_chunk_size, s, c,
                                          power) for s, c in zip(plan.token_starts, plan.token_counts)]
        pts = trace.points
        fetch = lambda i, t: sched_ref.fetch_latency(pts, plan.encoded_bytes[i], t)  # noqa: E731
        ttft, merge, rows = sched_ref.sim_bidirectional(comp, fetch, plan.n, race=True)
        assert (r.ttft_us, r.merge_point) == (ttft, merge)
        assert [[c.index, c.side, c.start_us, c.finish_us] for c in r.chunks] == \
            [[x.index, x.side, x.start, x.finish] for x in rows]
