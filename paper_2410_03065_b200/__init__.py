"""B200-native bidirectional KV-cache generator (Cake, arXiv 2410.03065 hot path).

The product is native: libcake.so (C++ cake:: runtime, drop-in for the
reference's scheduler/loader API) over libcake_cuda.so (sm_100a kernels).
This package is the thin Python handle on its C ABI.
"""
from .cake import BandwidthTrace, Cake, ChunkStore, CostModel, RunPlan, RunReport  # noqa: F401
from .native import LIB_DIR, load  # noqa: F401

__all__ = ["BandwidthTrace", "Cake", "ChunkStore", "CostModel", "RunPlan", "RunReport", "GpuRuntime", "PRESETS"]


def __getattr__(name):
    if name in ("GpuRuntime", "PRESETS"):
        from . import runtime

        return getattr(runtime, name)
    raise AttributeError(name)
