"""The C-ABI libraries load and export every symbol their headers declare (CPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2410_03065_b200", "_lib")


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"CAKE_API\s+[\w\s\*]+?\b(cake_\w+)\s*\(", text)))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(LIB, lib)], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


@pytest.mark.parametrize("header,lib", [("cake_cuda.h", "libcake_cuda.so"), ("cake_c.h", "libcake.so")])
def test_every_declared_symbol_is_exported(header, lib):
    names = declared(header)
    assert len(names) > 10
    missing = [n for n in names if n not in exported(lib)]
    assert not missing, f"{lib} lacks {missing}"


def test_libraries_load_without_gpu():
    ctypes.CDLL(os.path.join(LIB, "libcake_cuda.so"))
    ctypes.CDLL(os.path.join(LIB, "libcake.so"))


def test_kernels_are_sm100a_tcgen05():
    """The shipped CUDA layer is sm_100a code with tcgen05 MMA + TMA (SASS evidence)."""
    sass = subprocess.run(["cuobjdump", "-sass", os.path.join(LIB, "libcake_cuda.so")], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "LDTM" in sass  # tcgen05.ld (TMEM -> registers)


def test_gpu_entry_fails_loudly_without_device():
    """No CPU fallback: asking for the GPU runtime without a device raises."""
    from paper_2410_03065_b200.runtime import GpuRuntime
    from paper_2410_03065_b200.native import CakeError

    from conftest import have_gpu

    if have_gpu():
        pytest.skip("GPU present")
    with pytest.raises(CakeError):
        GpuRuntime("tiny", max_tokens=256, max_chunk=256)
