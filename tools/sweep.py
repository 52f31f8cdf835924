#!/usr/bin/env python3
"""BASELINE config 3: Llama-3-8B shape, context {8K, 32K, 64K} x emulated link
{1..32 GB/s}: bidirectional vs GPU compute-only vs GPU I/O-only TTFT on 1 B200.

One JSON line per (context, link) point on stdout:
  ttft_{cake,compute_only,io_only}_ms  device TTFT (run anchor -> logits event), best of --reps
  e2e_cake_ms                          host-clock TTFT (request -> logits in host memory)
  ratio_vs_min                         cake / min(compute_only, io_only)   (target <= 1)
  roofline_ms / frac                   bench.ttft_roofline_ms (oracle_best_split over ideal chunk times)

    python tools/sweep.py [--contexts 8192,32768,65536] [--gbps 1,2,4,8,16,32] [--reps 2] [--codec quant8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="8192,32768,65536")
    ap.add_argument("--gbps", default="1,2,4,8,16,32")
    ap.add_argument("--chunk", type=int, default=512)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--codec", default="identity")
    args = ap.parse_args()
    peak_s, _, hbm, _ = bench.load_peaks()
    C = args.chunk
    for T in [int(x) for x in args.contexts.split(",")]:
        rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=C)
        rt.set_codec(args.codec)
        rt.calibrate(T, C, 42)
        tier = rt.build_cache_tier(T, C, 42)
        for gb in [float(x) for x in args.gbps.split(",")]:
            mbps = gb * 8000.0
            best = {}
            for mode in ("compute_only", "io_only", "cake"):
                runs = [rt.run(tier, T, C, 42, mbps=mbps, mode=mode) for _ in range(args.reps)]
                best[mode] = min(runs, key=lambda r: r.device_ttft_ms)
            roof = bench.ttft_roofline_ms(bench.DIMS_8B, T, C, mbps * (2 if args.codec == "quant8" else 1),
                                          peak_s, hbm)
            ck, co, io = best["cake"], best["compute_only"], best["io_only"]
            line = {"context": T, "link_GBps": gb, "codec": args.codec, "chunk": C,
                    "ttft_cake_ms": ck.device_ttft_ms, "ttft_compute_only_ms": co.device_ttft_ms,
                    "ttft_io_only_ms": io.device_ttft_ms, "e2e_cake_ms": ck.first_token_ms,
                    "ratio_vs_min": ck.device_ttft_ms / min(co.device_ttft_ms, io.device_ttft_ms),
                    "merge_point": ck.merge_point, "n_chunks": ck.n_chunks, "raced": ck.raced_chunk,
                    "race_winner": ck.race_winner, "roofline_ms": roof["bidir_ms"],
                    "frac": roof["bidir_ms"] / ck.device_ttft_ms, "k_star": roof["k_star"]}
            print(json.dumps(line), flush=True)
        rt.close()
        del tier


if __name__ == "__main__":
    main()
