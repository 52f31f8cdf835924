"""Pure-Python restatement of the reference scheduler's decision model.

TEST INFRASTRUCTURE ONLY (checker for tests/; never imported by the product).
Each function cites the reference file:line it restates. Pinned by
tests/test_golden.py against the reference's own golden values
(proj/tests/test_model.cpp, test_scheduler.cpp, test_compute.cpp) and, when
oracle/_ref is built, against the reference library itself.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


def _is_whole(x: float) -> bool:  # proj/src/model.cpp:102
    return x == math.floor(x) and 0.0 < x < 9.0e15


def time_to_transfer_bits(points, bits: int, start: int) -> int:
    """proj/src/model.cpp:105-167. points: [(at_us, mbps)] sorted, first at 0."""
    if start < 0:
        raise ValueError("start_time must be >= 0")
    if bits == 0:
        return 0
    i = len(points) - 1
    while i > 0 and points[i][0] > start:
        i -= 1
    exact = all(_is_whole(p[1]) for p in points)
    elapsed, cursor = 0, start
    if exact:  # :105-128 integer path
        rem = bits
        while True:
            rate = int(points[i][1])
            if i + 1 < len(points):
                seg_end = points[i + 1][0]
                cap = (seg_end - cursor) * rate
                if cap < rem:
                    rem -= cap
                    elapsed += seg_end - cursor
                    cursor = seg_end
                    i += 1
                    continue
            return elapsed + (rem + rate - 1) // rate
    # :130-156 real path (python float = double; the reference uses long double,
    # so this branch is only compared on cases without sub-ulp ties)
    rem = float(bits)
    while True:
        rate = float(points[i][1])
        if i + 1 < len(points):
            seg_end = points[i + 1][0]
            cap = rate * (seg_end - cursor)
            if cap < rem:
                rem -= cap
                elapsed += seg_end - cursor
                cursor = seg_end
                i += 1
                continue
        need = rem / rate
        return elapsed + max(math.ceil(need - 1e-7), 0)


def fetch_latency(points, nbytes: int, start: int = 0) -> int:  # proj/src/model.cpp:169-171
    return time_to_transfer_bits(points, nbytes * 8, start)


def compute_latency(alpha, beta, ref, token_start, token_count, power=1.0) -> int:  # proj/src/model.cpp:90-98
    ms = (alpha + beta * token_start) * (token_count / ref) / power
    return int(math.floor(ms * 1000.0 + 0.5)) if ms * 1000.0 >= 0 else -int(math.floor(-ms * 1000.0 + 0.5))


def oracle_best_split(c, f):  # proj/src/scheduler.cpp:71-87
    n = len(c)
    suffix = [0] * (n + 1)
    for i in range(n - 1, -1, -1):
        suffix[i] = suffix[i + 1] + f[i]
    best_k, best_t = 0, suffix[0]
    prefix = 0
    for k in range(1, n + 1):
        prefix += c[k - 1]
        t = max(prefix, suffix[k])
        if t < best_t:
            best_k, best_t = k, t
    return best_k, best_t


@dataclass
class Rec:
    index: int
    side: str
    start: int
    finish: int


def sim_bidirectional(compute_us, fetch_fn, n, race=False):
    """proj/src/scheduler.cpp:164-202 (greedy event loop, ties to compute),
    plus — race=True — the boundary race-to-finish this build adds (one
    contested chunk; earlier completion commits).  fetch_fn(i, start) -> µs.
    Returns (ttft, merge_point, records)."""
    recs = {}
    cn, io = 0, n - 1
    c_free = io_free = 0
    while cn <= io:
        if c_free <= io_free:
            recs[cn] = Rec(cn, "compute", c_free, c_free + compute_us[cn])
            c_free += compute_us[cn]
            cn += 1
        else:
            d = fetch_fn(io, io_free)
            recs[io] = Rec(io, "io", io_free, io_free + d)
            io_free += d
            io -= 1
    merge = io + 1
    if race:
        if merge >= 1 and io_free < c_free:
            k = merge - 1
            done = io_free + fetch_fn(k, io_free)
            if done < c_free:
                recs[k] = Rec(k, "io", io_free, done)
                merge = k
        elif merge < n and c_free < io_free:
            k = merge
            done = c_free + compute_us[k]
            if done < io_free:
                recs[k] = Rec(k, "compute", c_free, done)
                merge = k + 1
    ttft = max(r.finish for r in recs.values())
    return ttft, merge, [recs[i] for i in range(n)]


def sim_compute_only(compute_us):  # proj/src/scheduler.cpp:126-141
    return sum(compute_us)


def sim_io_only(fetch_fn, n):  # proj/src/scheduler.cpp:143-158
    t = 0
    for i in range(n - 1, -1, -1):
        t += fetch_fn(i, t)
    return t
