"""Experiment build (make ATTN_VARIANTS=1): an attention variant against the
product kernel on the parity configs of tests/test_gpu_parity.py — computed
KV (RMS-normalised error) and first-token logits.
    IMPL=tcgen05_alt python tools/attn_variant_check.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import llama_oracle  # noqa: E402
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

CONFIGS = {
    "tiny": ((2, 256, 4, 4, 64, 1024, 32000), 2048, 256, 44),
    "gqa_hd64": ((2, 512, 8, 2, 64, 1024, 32000), 1024, 256, 42),
    "gqa_hd128": ((2, 1024, 8, 2, 128, 2048, 32768), 1024, 512, 45),
    "gqa8_hd128": ((2, 1024, 16, 2, 128, 2048, 32768), 1024, 256, 45),
    "8b_2layer_8k": ((2, 4096, 32, 8, 128, 14336, 128256), 8192, 512, 42),
}
impl = os.environ.get("IMPL", "tcgen05_alt")


def rms_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)))


worst = 0.0
for name, (dims, T, C, seed) in CONFIGS.items():
    rt = GpuRuntime(dims, max_tokens=T, max_chunk=C)
    tier = rt.build_cache_tier(T, C, seed)
    out = {}
    for im in ("tcgen05", impl):
        rt.set_attention_impl(im)
        for mode in ("compute_only", "io_only"):
            rt.poison(0xFF)
            rt.run(tier, T, C, seed, mbps=64000, mode=mode)
            out[(im, mode)] = (rt.logits().copy(),
                               [llama_oracle.bf16_to_f32(np.frombuffer(rt.read_chunk(s, C), np.uint16))
                                for s in range(0, T, C)])
    rt.set_attention_impl("tcgen05")
    for mode in ("compute_only", "io_only"):
        lg0, kv0 = out[("tcgen05", mode)]
        lg1, kv1 = out[(impl, mode)]
        e_kv = max(rms_rel(a, b) for a, b in zip(kv1, kv0))
        e_lg = rms_rel(lg1, lg0)
        worst = max(worst, e_kv, e_lg)
        print(f"{name:14s} {mode:12s} kv rms rel {e_kv:.2e}  logits rms rel {e_lg:.2e}  "
              f"top1 {'same' if lg0.argmax() == lg1.argmax() else 'DIFF'}  finite {np.isfinite(lg1).all()}", flush=True)
    rt.close()
print(f"worst {worst:.2e} (bar 2^-7 = {2 ** -7:.2e}): {'OK' if worst <= 2 ** -7 else 'FAIL'}")
