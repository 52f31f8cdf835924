"""Attention split policy A/B inside an 8B compute-only run: the product's
one-wave rule (128 CTAs of 148 SMs at C = 512) against multi-wave split-KV
(CAKE_EXP_ATTN_MAX_WAVES), per-class event-bracketed time and the run's TTFT.

    python tools/attn_waves.py [T=32768] [waves=1,2,4,7]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200 import native as N  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
waves = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,7").split(",")]
cl = N.load_cuda()
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
tier = rt.build_cache_tier(T, 512, 42)
if os.environ.get("IMPL"):
    rt.set_attention_impl(os.environ["IMPL"])  # e.g. tcgen05_s3
for rep in range(2):
    for w in waves:
        cl.cake_set_experiment(2, w)
        rt.set_profiling(["attention"])
        rt.kernel_stats(reset=True)
        r1 = rt.run(tier, T, 512, 42, mbps=64000, mode="compute_only")
        st = rt.kernel_stats(reset=True)["attention"]
        rt.set_profiling(None)
        r2 = rt.run(tier, T, 512, 42, mbps=64000, mode="compute_only")
        print(f"T={T} max_waves={w}: attention {st['ms']:.1f} ms over {st['launches']} launches "
              f"({st['flops'] / st['ms'] / 1e9:.0f} TF/s bracketed); compute-only TTFT {r2.device_ttft_ms:.1f} ms",
              flush=True)
cl.cake_set_experiment(2, 1)
