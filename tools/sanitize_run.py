"""Small bidirectional runs covering every product kernel (2-SM and cluster
GEMMs at M = 512, the 1-SM GEMM at M <= 128, tcgen05 attention with split-KV,
the first-token chain kernel, scatter/gather, quant8 decode-scatter) for
compute-sanitizer (memcheck / racecheck / synccheck): tools/sanitize.sh."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

for dims, T, C in [((2, 1024, 8, 2, 128, 2048, 32768), 1024, 512), ((2, 256, 4, 4, 64, 1024, 32000), 1000, 256)]:
    rt = GpuRuntime(dims, max_tokens=1024, max_chunk=C)
    tier = rt.build_cache_tier(T, C, 42)
    for mode in ("compute_only", "io_only", "cake"):
        r = rt.run(tier, T, C, 42, mbps=2000, mode=mode)
        print(dims[1], mode, "merge", r.merge_point, "first token", round(r.first_token_ms, 2), flush=True)
    rt.set_codec("quant8")
    q8 = rt.build_cache_tier(T, C, 42)
    r = rt.run(q8, T, C, 42, mbps=2000, mode="io_only")
    print(dims[1], "quant8 io_only", round(r.first_token_ms, 2), flush=True)
    rt.close()
