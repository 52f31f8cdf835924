#!/usr/bin/env python3
"""BASELINE config 5 with CONCURRENT requests: a mix of long prompts (4K-128K
tokens, varying cached-prefix fraction) on the Llama-3-8B shape arriving over
time at one B200, served by `--workers` contexts that share one weight copy and
ONE emulated link (paper_2410_03065_b200/serve.py), with the link's bandwidth
stepping down mid-mix. The same arrivals are served with 1 worker (requests one
at a time, the round-1 tools/mix.py setting) for comparison.

    python tools/serve_mix.py [--requests T:frac:arrival_ms,...] [--trace 0:16,300:4] [--workers 1,2,3]

One JSON line per (workers, request), then one summary line per worker count.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_03065_b200.cake import BandwidthTrace  # noqa: E402
from paper_2410_03065_b200.serve import GpuServer, Request  # noqa: E402


def parse_trace(spec):
    pts = []
    for item in spec.split(","):
        t_ms, gbps = item.split(":")
        pts.append((int(float(t_ms) * 1000), float(gbps) * 8000.0))
    return BandwidthTrace(pts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests",
                    default="32768:0.75:0,4096:1.0:50,65536:0.5:100,16384:0.5:150,131072:0.25:200,8192:1.0:250")
    ap.add_argument("--trace", default="0:16,300:4")
    ap.add_argument("--workers", default="1,2,3")
    ap.add_argument("--chunk", type=int, default=512)
    args = ap.parse_args()
    C = args.chunk
    reqs = [(int(t), float(f), float(a)) for t, f, a in (x.split(":") for x in args.requests.split(","))]
    trace = parse_trace(args.trace)
    Tmax = max(t for t, _, _ in reqs)
    counts = [int(w) for w in args.workers.split(",")]
    srv = GpuServer("llama3_8b", workers=max(counts), trace=trace, max_tokens=Tmax, max_chunk=C)
    for rt in srv.runtimes:
        rt.calibrate(8192, C, 1)
    tiers = []
    for i, (T, frac, _) in enumerate(reqs):
        cached = max(C, int(T * frac) // C * C)
        tiers.append((srv.primary.build_cache_tier(cached, C, 100 + i), cached))
    every = srv.runtimes
    for W in counts:
        srv.runtimes = every[:W]
        requests = [Request(tiers[i][0], T, C, 100 + i, arrival_ms=a, options={"cached_prefix": True})
                    for i, (T, _, a) in enumerate(reqs)]
        srv.serve(requests)  # warm-up pass
        out = srv.serve(requests)
        for sv in out:
            T = reqs[sv.index][0]
            r = sv.result
            print(json.dumps({
                "workers": W, "request": sv.index, "tokens": T, "cached_tokens": tiers[sv.index][1],
                "arrival_ms": sv.arrival_ms, "start_ms": sv.start_ms, "end_ms": sv.end_ms,
                "ttft_ms": sv.ttft_ms, "queue_ms": sv.start_ms - sv.arrival_ms, "run_ttft_ms": r.first_token_ms,
                "device_ttft_ms": r.device_ttft_ms, "merge_point": r.merge_point,
                "cached_chunks": tiers[sv.index][1] // C, "n_chunks": r.n_chunks, "worker": sv.worker,
                "raced": r.raced_chunk, "race_winner": r.race_winner,
            }), flush=True)
        print(json.dumps({
            "workers": W, "summary": True, "requests": len(out),
            "trace_gbps": [(t / 1000, m / 8000) for t, m in trace.points],
            "mean_ttft_ms": statistics.mean(sv.ttft_ms for sv in out),
            "p50_ttft_ms": statistics.median(sv.ttft_ms for sv in out),
            "max_ttft_ms": max(sv.ttft_ms for sv in out),
            "makespan_ms": max(sv.end_ms for sv in out),
        }), flush=True)
    srv.runtimes = every
    for t, _ in tiers:
        t.close()
    srv.close()


if __name__ == "__main__":
    main()
