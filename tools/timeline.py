"""Per-chunk timeline of one bidirectional run (which side finishes when, the
gap before the first token)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(os.environ.get("T", "32768"))
mbps = float(os.environ.get("MBPS", "64000"))
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
rt.calibrate(T, 512, 42)
tier = rt.build_cache_tier(T, 512, 42)
for rep in range(3):
    r = rt.run(tier, T, 512, 42, mbps=mbps, mode="cake")
comp = sorted((c for c in r.chunks if c.side == "compute"), key=lambda c: c.index)
io = sorted((c for c in r.chunks if c.side == "io"), key=lambda c: c.index)
print(f"device TTFT {r.device_ttft_ms:.2f} ms, kv resident {r.kv_resident_ms:.2f}, final step {r.final_step_ms:.2f}, "
      f"merge {r.merge_point}/{r.n_chunks}, raced {r.raced_chunk} winner {r.race_winner}")
print("compute: " + " ".join(f"{c.index}:{c.start_us/1e3:.1f}-{c.finish_us/1e3:.1f}" for c in comp[-4:]))
print("io:      " + " ".join(f"{c.index}:{c.finish_us/1e3:.1f}" for c in io[:4]))
durs = [(c.finish_us - c.start_us) / 1e3 for c in comp]
print("compute chunk ms: " + " ".join(f"{d:.1f}" for d in durs))
