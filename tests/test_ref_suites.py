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


@pytest.mark.parametrize("name", ["acceptance_ref", "acceptance_b200"])
def test_reference_acceptance_main(name):
    """proj/tests/acceptance.cpp:498-527 — the reference's 10 acceptance criteria
    (near-optimality, exactly-once under jitter, dominance, merge trend, collapse,
    live throttle fidelity, scheduler overhead, codec equivalence, store
    integrity, reproducibility), against the reference and against libcake.so."""
    p = _run(name)
    failed = [l for l in p.stdout.splitlines() if l.startswith("criterion") and "FAIL" in l]
    if p.returncode != 0 and failed and all(l.startswith("criterion 6 ") for l in failed):
        # criterion 6 is a wall-clock throttle audit; a descheduled container
        # thread (both attempts of a rate) is noise, not a throttle bug: one rerun.
        p = _run(name)
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-3000:])
    assert "acceptance: all criteria passed" in p.stdout, p.stdout[-3000:]


def test_reference_suites_pass_on_b200_library():
    p = _run("unit_b200")
    assert p.returncode == 0, p.stderr[-4000:]
    assert "| 0 failed | assertions" in p.stdout, p.stdout
