"""A/B of the attention kernels inside a compute-only 8B tier build (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_03065_b200.runtime import GpuRuntime  # noqa: E402

T = int(os.environ.get("T", "8192"))
rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=512)
rt.set_attention_impl(os.environ.get("IMPL", "tcgen05_2tile"))
rt.build_cache_tier(T, 512, 42)
