#!/usr/bin/env python3
"""GPU-share emulation. The reference scales its modeled
chunk latency by a power fraction p (proj/src/model.cpp:94-96);
the paper's partial-power runs report the largest gains of bidirectional KV
generation there. Here the compute stream is confined to a
fraction of the B200's SMs (a green context over an SM partition,
GpuRuntime(compute_sms=...)); the loader keeps the copy engines and the rest.

One JSON line per (SM share, context, link): TTFT of bidirectional vs GPU
compute-only vs I/O-only on the same partition and tier.

    python tools/gpu_share.py [--shares 0.1,0.25,0.5,1.0] [--contexts 14336,32768] [--gbps 8]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shares", default="0.1,0.25,0.5,1.0")
    ap.add_argument("--contexts", default="14336,32768")
    ap.add_argument("--gbps", default="8")
    ap.add_argument("--chunk", type=int, default=512)
    args = ap.parse_args()
    C = args.chunk
    ctxs = [int(x) for x in args.contexts.split(",")]
    for share in [float(x) for x in args.shares.split(",")]:
        sms = 0 if share >= 1.0 else max(8, int(round(148 * share)))
        rt = GpuRuntime("llama3_8b", max_tokens=max(ctxs), max_chunk=C, compute_sms=sms)
        for T in ctxs:
            rt.calibrate(T, C, 42)
            tier = rt.build_cache_tier(T, C, 42)
            for gb in [float(x) for x in args.gbps.split(",")]:
                mbps = gb * 8000.0
                best = {m: min((rt.run(tier, T, C, 42, mbps=mbps, mode=m) for _ in range(2)),
                               key=lambda r: r.device_ttft_ms) for m in ("compute_only", "io_only", "cake")}
                ck, co, io = best["cake"], best["compute_only"], best["io_only"]
                print(json.dumps({"sm_share": share, "compute_sms": sms or 148, "tokens": T, "link_GBps": gb,
                                  "ttft_cake_ms": ck.device_ttft_ms, "ttft_compute_only_ms": co.device_ttft_ms,
                                  "ttft_io_only_ms": io.device_ttft_ms,
                                  "reduction_vs_compute_only": 1 - ck.device_ttft_ms / co.device_ttft_ms,
                                  "reduction_vs_io_only": 1 - ck.device_ttft_ms / io.device_ttft_ms,
                                  "merge_point": ck.merge_point, "n_chunks": ck.n_chunks}), flush=True)
            tier.close()
        rt.close()


if __name__ == "__main__":
    main()
