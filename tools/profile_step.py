"""One compute-only 8B step for ncu's launch list (per-kernel device time) and
to compare the kernels' sum with the step's wall time (launch gaps)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(os.environ.get("T", "8192"))
mode = os.environ.get("MODE", "compute_only")
sched = os.environ.get("GEMM_SCHED")
if sched is not None:
    from paper_2410_03065_b200 import native
    native.load_cuda().cake_gemm_set_schedule(int(sched))
C = int(os.environ.get("C", "512"))
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=C, lookahead_layers=int(os.environ.get("LOOKAHEAD", "0")))
tier = rt.build_cache_tier(T, C, 42)
for i in range(int(os.environ.get("REPS", "2"))):
    t0 = time.time()
    r = rt.run(tier, T, C, 42, mbps=float(os.environ.get("MBPS", "64000")), mode=mode)
    print(f"{mode} T={T} C={C}: device {r.device_ttft_ms:.2f} ms, wall {1e3*(time.time()-t0):.1f} ms, "
          f"launches {r.kernel_launches}, merge {r.merge_point}", flush=True)
