#!/usr/bin/env python3
"""the cache tier on local disk (reference file format:
<root>/<hh>/<digest>.kv + manifest.v1) instead of pinned DRAM. Builds an 8B
32K tier under --root, then loads it with no emulated throttle (the link is
the disk + PCIe) through buffered reads (page cache: after the build the
files are hot) and O_DIRECT reads (every run reads the disk), io-only and
bidirectional. One JSON line per (read mode, run mode).

    python tools/file_tier.py [--root /tmp/cake_tier] [--tokens 32768]"""
import argparse
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.cake import ChunkStore  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--root", default="/tmp/cake_tier")
    ap.add_argument("--tokens", type=int, default=32768)
    args = ap.parse_args()
    T, C = args.tokens, 512
    shutil.rmtree(args.root, ignore_errors=True)
    df = subprocess.run(["df", "-h", os.path.dirname(args.root) or "/"], capture_output=True, text=True).stdout
    rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=C)
    rt.calibrate(T, C, 42)
    fs = ChunkStore(rt.n, args.root, create=1)
    rt.build_cache_tier(T, C, 42, store=fs)
    tier_bytes = T * rt.kv_bytes_per_token
    unthrottled = 8e6  # 1 TB/s "link": the loader runs at the disk / PCIe rate
    for direct in (False, True):
        fs.set_direct_io(direct)
        for mode in ("io_only", "cake"):
            runs = [rt.run(fs, T, C, 42, mbps=unthrottled, mode=mode) for _ in range(2)]
            r = min(runs, key=lambda x: x.device_ttft_ms)
            io_chunks = [c for c in r.chunks if c.side == "io"]
            io_bytes = sum(c.bytes for c in io_chunks)
            io_ms = max((c.finish_us for c in io_chunks), default=0) / 1e3
            print(json.dumps({"read": "O_DIRECT" if direct else "buffered (page cache)", "mode": mode,
                              "tokens": T, "tier_bytes": tier_bytes, "ttft_ms": r.device_ttft_ms,
                              "e2e_ms": r.first_token_ms, "merge_point": r.merge_point, "n_chunks": r.n_chunks,
                              "loaded_bytes": io_bytes,
                              "io_finish_ms": [(c.index, round(c.finish_us / 1e3, 1)) for c in
                                               sorted(io_chunks, key=lambda c: c.finish_us)],
                              "load_GBps": io_bytes / (io_ms / 1e3) / 1e9 if io_ms > 0 else None}), flush=True)
    print(json.dumps({"disk": df.strip().splitlines()[-1] if df else None}))
    fs.close()
    shutil.rmtree(args.root, ignore_errors=True)


if __name__ == "__main__":
    main()
