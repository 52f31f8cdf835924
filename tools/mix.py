#!/usr/bin/env python3
"""BASELINE config 5: a mix of long prompts (4K-128K tokens, varying cached-prefix
fraction) on the Llama-3-8B shape, one B200, with the emulated I/O bandwidth
stepping down mid-request, so the merge point has to move at run time.

Each request is served three ways on the same GPU and the same cache tier:
  cake          bidirectional over the cached prefix (compute forward from token 0,
                loads backward from the prefix end, runtime merge point), then the
                uncached suffix computed;
  compute_only  the whole prompt computed;
  io_only       the cached prefix loaded, the suffix computed.
Every run uses the same piecewise-constant trace (reference BandwidthTrace,
proj/include/cake/model.hpp:58-77; proj/configs/traces/step.csv is the same
shape): --trace "0:16,120:4" = 16 GB/s from arrival, 4 GB/s from t = 120 ms.
The cake run is repeated with the trace's first rate held constant, to show
the merge point the step change moved.

    python tools/mix.py [--requests 4096:1.0,16384:0.5,32768:0.75,65536:1.0,131072:0.25]
                        [--trace 0:16,120:4] [--chunk 512]

One JSON line per request on stdout.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_03065_b200.cake import BandwidthTrace  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402


def parse_trace(spec):
    pts = []
    for item in spec.split(","):
        t_ms, gbps = item.split(":")
        pts.append((int(float(t_ms) * 1000), float(gbps) * 8000.0))  # mbps = bits per us
    return BandwidthTrace(pts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", default="4096:1.0,16384:0.5,32768:0.75,65536:1.0,131072:0.25")
    ap.add_argument("--trace", default="0:16,120:4")
    ap.add_argument("--chunk", type=int, default=512)
    args = ap.parse_args()
    C = args.chunk
    reqs = [(int(t), float(f)) for t, f in (x.split(":") for x in args.requests.split(","))]
    trace = parse_trace(args.trace)
    steady = BandwidthTrace([(0, trace.points[0][1])])
    rt = GpuRuntime("llama3_8b", max_tokens=max(t for t, _ in reqs), max_chunk=C)
    rt.calibrate(min(32768, max(t for t, _ in reqs)), C, 1)
    for i, (T, frac) in enumerate(reqs):
        seed = 100 + i
        cached = max(C, int(T * frac) // C * C)
        tier = rt.build_cache_tier(cached, C, seed)
        best = {}
        for mode in ("compute_only", "io_only", "cake"):
            runs = [rt.run(tier, T, C, seed, trace=trace, mode=mode, cached_prefix=True) for _ in range(2)]
            best[mode] = min(runs, key=lambda r: r.device_ttft_ms)
        st = min((rt.run(tier, T, C, seed, trace=steady, mode="cake", cached_prefix=True) for _ in range(2)),
                 key=lambda r: r.device_ttft_ms)
        ck, co, io = best["cake"], best["compute_only"], best["io_only"]
        print(json.dumps({
            "request": i, "tokens": T, "cached_tokens": cached, "cached_fraction": cached / T,
            "trace_gbps": [(t / 1000, m / 8000) for t, m in trace.points],
            "ttft_cake_ms": ck.device_ttft_ms, "ttft_compute_only_ms": co.device_ttft_ms,
            "ttft_io_only_ms": io.device_ttft_ms, "e2e_cake_ms": ck.first_token_ms,
            "ratio_vs_min": ck.device_ttft_ms / min(co.device_ttft_ms, io.device_ttft_ms),
            "merge_point": ck.merge_point, "cached_chunks": cached // C, "n_chunks": ck.n_chunks,
            "raced": ck.raced_chunk, "race_winner": ck.race_winner,
            "steady_trace_merge_point": st.merge_point, "steady_trace_ttft_ms": st.device_ttft_ms,
        }), flush=True)
        tier.close()
    rt.close()


if __name__ == "__main__":
    main()
