"""Per-chunk timeline of bidirectional runs (8B, 32K, 8 GB/s): which side
delivered each chunk and when, the merge, the race, and the gap between the
last delivery and the first token.
    python tools/run_timeline.py [T=32768] [mbps=64000] [reps=3]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
mbps = float(sys.argv[2]) if len(sys.argv) > 2 else 64000.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
rt.calibrate(T, 512, 42)
tier = rt.build_cache_tier(T, 512, 42)
for rep in range(reps):
    r = rt.run(tier, T, 512, 42, mbps=mbps, mode="cake")
    ch = sorted(r.chunks, key=lambda c: c.finish_us)
    comp = [c for c in ch if c.side == "compute"]
    io = [c for c in ch if c.side == "io"]
    print(f"rep {rep}: device TTFT {r.device_ttft_ms:.2f} ms, kv resident {r.kv_resident_ms:.2f}, final step "
          f"{r.final_step_ms:.2f}, merge {r.merge_point}, raced {r.raced_chunk} won by {r.race_winner}")
    print(f"  compute: {len(comp)} chunks, first start {comp[0].start_us / 1e3:.2f} ms, last finish "
          f"{comp[-1].finish_us / 1e3:.2f} ms (chunk {comp[-1].index})")
    print(f"  io:      {len(io)} chunks, first finish {io[0].finish_us / 1e3:.2f} ms, last finish "
          f"{io[-1].finish_us / 1e3:.2f} ms (chunk {io[-1].index}); link-only time {len(io) * 512 * 131072 * 8 / mbps / 1e3:.2f} ms")
