"""GPU probe: end-to-end bidirectional runs (tiny vs CPU oracle; 8B timings)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402
from paper_2410_03065_b200.cake import Cake  # noqa: E402
import llama_oracle  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / (np.abs(b).max() + 1e-12))


def tiny():
    T, CH, SEED = 2048, 256, 42
    rt = GpuRuntime("tiny", max_tokens=T, max_chunk=256)
    t0 = time.time()
    tier = rt.build_cache_tier(T, CH, SEED)
    print(f"tiny tier built in {time.time()-t0:.2f}s, entries={tier.entry_count()}", flush=True)
    toks = Cake().token_stream(SEED, T).astype(np.int32)
    # oracle
    ref = llama_oracle.LlamaRef(rt.dims, T)
    for s in range(0, T, CH):
        ref.prefill_chunk(toks[s:s + CH], s)
    ref_logits = ref.final_logits(CH - 1)
    ref_kv = ref.kv()
    res_all = {}
    for mode, mbps in [("compute_only", 4000), ("io_only", 4000), ("cake", 100), ("cake", 1000), ("cake", 4000),
                       ("cake", 40000)]:
        r = rt.run(tier, T, CH, SEED, mbps=mbps, mode=mode, quantum=64 << 10)
        lg = rt.logits()
        print(f"{mode:13s} @{mbps:6d} mbps: first_token={r.first_token_ms:8.2f} ms kv_resident={r.kv_resident_ms:8.2f} "
              f"merge={r.merge_point} race={r.raced_chunk}/{r.race_winner} recompute={r.recomputed_last} "
              f"final={r.final_step_ms:.2f}ms launches={r.kernel_launches} logits_rel={rel(lg, ref_logits):.3e} "
              f"top1 {lg.argmax()} vs {ref_logits.argmax()}", flush=True)
        res_all[(mode, mbps)] = lg
    # assembled KV vs oracle
    worst = 0.0
    for s in range(0, T, CH):
        b = np.frombuffer(rt.read_chunk(s, CH), dtype=np.uint16)
        g = llama_oracle.bf16_to_f32(b).reshape(rt.dims[0], 2, rt.dims[3], CH, rt.dims[4])
        worst = max(worst, rel(g, ref_kv[:, :, :, s:s + CH, :]))
    print(f"assembled KV vs oracle rel max: {worst:.3e}")
    # tier bytes = GPU computed KV for chunk 0
    k0 = Cake().chain_hash(None, toks[:CH].astype(np.uint32))
    print("tier chunk0 == readback:", tier.get(k0) == rt.read_chunk(0, CH))


def llama8b(T=8192, layers=None):
    CH, SEED = 512, 42
    t0 = time.time()
    rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512, n_layers=layers)
    print(f"8B model ({rt.dims[0]} layers) created in {time.time()-t0:.1f}s", flush=True)
    t0 = time.time()
    a, b = rt.calibrate(T, CH, SEED)
    print(f"calibrate: alpha={a:.3f} ms beta={b*1e3:.4f} us/token  ({time.time()-t0:.1f}s)", flush=True)
    t0 = time.time()
    tier = rt.build_cache_tier(T, CH, SEED)
    print(f"tier built {time.time()-t0:.1f}s", flush=True)
    for mode, mbps in [("compute_only", 64000), ("io_only", 64000), ("cake", 64000), ("cake", 8000),
                       ("cake", 256000)]:
        for rep in range(2):
            r = rt.run(tier, T, CH, SEED, mbps=mbps, mode=mode)
            print(f"{mode:13s} @{mbps:6d}: first_token={r.first_token_ms:8.2f} ms kv={r.kv_resident_ms:8.2f} "
                  f"merge={r.merge_point}/{r.n_chunks} race={r.raced_chunk}/{r.race_winner} final={r.final_step_ms:.2f}ms "
                  f"dev={r.device_ttft_ms:.2f}", flush=True)
    lg = rt.logits()
    print("logits finite:", np.isfinite(lg).all(), "top1", lg.argmax())


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    if which in ("tiny", "all"):
        tiny()
    if which in ("8b", "all"):
        llama8b()
