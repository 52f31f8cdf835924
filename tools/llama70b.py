#!/usr/bin/env python3
"""BASELINE config 4 at TP = 1: the Llama-3-70B shape (80 layers, H 8192,
64 q / 8 KV heads, FFN 28672) fits one B200 (141 GB of bf16 weights + a 10 GB
32K paged KV cache), so the whole bidirectional run of one 70B prompt can be
measured on the single GPU this pool provides. (The head-sharded TP path is
tested on one device with tests/test_gpu_tp.py.)

    python tools/llama70b.py [--tokens 32768] [--gbps 8]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

DIMS_70B = (80, 8192, 64, 8, 128, 28672, 128256)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--gbps", default="8")
    args = ap.parse_args()
    T, C = args.tokens, 512
    t0 = time.time()
    rt = GpuRuntime("llama3_70b", max_tokens=T, max_chunk=C)
    init_s = time.time() - t0
    rt.calibrate(min(T, 8192), C, 42)
    t0 = time.time()
    tier = rt.build_cache_tier(T, C, 42)
    tier_s = time.time() - t0
    peak_s, _, hbm, _ = bench.load_peaks()
    for gb in [float(x) for x in args.gbps.split(",")]:
        mbps = gb * 8000.0
        best = {m: min((rt.run(tier, T, C, 42, mbps=mbps, mode=m) for _ in range(2)), key=lambda r: r.device_ttft_ms)
                for m in ("compute_only", "io_only", "cake")}
        ck, co, io = best["cake"], best["compute_only"], best["io_only"]
        roof = bench.ttft_roofline_ms(DIMS_70B, T, C, mbps, peak_s, hbm)
        print(json.dumps({"model": "llama-3-70b-shape", "tp": 1, "tokens": T, "link_GBps": gb,
                          "ttft_cake_ms": ck.device_ttft_ms, "ttft_compute_only_ms": co.device_ttft_ms,
                          "ttft_io_only_ms": io.device_ttft_ms,
                          "ratio_vs_min": ck.device_ttft_ms / min(co.device_ttft_ms, io.device_ttft_ms),
                          "merge_point": ck.merge_point, "n_chunks": ck.n_chunks, "final_step_ms": ck.final_step_ms,
                          "roofline_ms": roof["bidir_ms"], "frac": roof["bidir_ms"] / ck.device_ttft_ms,
                          "compute_only_roofline_ms": roof["compute_only_ms"], "model_init_s": init_s,
                          "tier_build_s": tier_s}), flush=True)


if __name__ == "__main__":
    main()
