"""First-token step cost: an io-only run (every chunk loaded, so the 1-token
pass over the assembled cache runs) with every kernel class event-bracketed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(os.environ.get("T", "32768"))
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
tier = rt.build_cache_tier(T, 512, 42)
if os.environ.get("IMPL"):
    rt.set_attention_impl(os.environ["IMPL"])
for _ in range(2):
    r = rt.run(tier, T, 512, 42, mbps=256000, mode="io_only")
print(f"unprofiled: final step {r.final_step_ms:.3f} ms, kv resident {r.kv_resident_ms:.2f} ms")
rt.kernel_stats(reset=True)
rt.set_profiling("all")
r = rt.run(tier, T, 512, 42, mbps=256000, mode="io_only")
st = rt.kernel_stats(reset=True)
rt.set_profiling(None)
print(f"profiled: final step {r.final_step_ms:.3f} ms")
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 else 0
        print(f"  {k:12s} {v['launches']:5d} launches {v['ms']:8.3f} ms  {gbs:7.0f} GB/s")
