"""The reference's OWN unit suites (proj/tests/test_{model,codec,store,transfer,
compute,scheduler}.cpp, compiled unmodified with oracle/doctest_shim) pass against
both the reference library and the B200 library (oracle/Makefile unit_ref/unit_b200).
This is the drop-in check for the C++ API: same headers, same behaviour."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref")


def _run(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=600, cwd=os.path.join(ROOT, "oracle"))
    return p


def test_reference_suites_pass_on_reference():
    p = _run("unit_ref")
    assert p.returncode == 0, p.stderr[-4000:]
    assert "0 failed" in p.stdout


def test_reference_suites_pass_on_b200_library():
    p = _run("unit_b200")
    assert p.returncode == 0, p.stderr[-4000:]
    assert "| 0 failed | assertions" in p.stdout, p.stdout
