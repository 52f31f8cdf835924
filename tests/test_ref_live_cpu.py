"""The un-extrapolated CPU baseline of BASELINE config 1 (oracle/ref_live_cpu.cpp):
the reference's own live run (claim table, throttled file-tier loader, store,
scheduler: proj/src/*.cpp compiled unmodified) with its compute sleep
(proj/src/compute.cpp:48-49) replaced by the CPU forward of llama_ref.c.
Every chunk is covered exactly once in every mode, and the first token is the
same whichever side produced the tail (the loaded bytes are the oracle's own KV)."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "ref_live_cpu")


def _run(mode, tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/ref_live_cpu not built (needs /root/reference at build time)")
    p = subprocess.run([BIN, "2048", "256", "800", "4", str(tmp_path / mode), mode], capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr
    return json.loads(p.stdout)


def test_config1_live_cpu_modes(tmp_path):
    import llama_oracle
    from paper_2410_03065_b200.cake import Cake

    out = {m: _run(m, tmp_path) for m in ("cake", "compute_only", "io_only")}
    for m, r in out.items():
        assert r["chunks_reported"] == r["n_chunks"] == 8, m
    assert out["compute_only"]["merge_point"] == 8 and not out["compute_only"]["recomputed_last"]
    assert out["io_only"]["merge_point"] == 0 and out["io_only"]["recomputed_last"]
    assert len({r["top1"] for r in out.values()}) == 1
    # the oracle computed directly gives the same first token
    T, C = 2048, 256
    toks = Cake().token_stream(42, T).astype(np.int32)
    ref = llama_oracle.LlamaRef((2, 256, 4, 4, 64, 1024, 32000), T)
    for s in range(0, T, C):
        ref.prefill_chunk(toks[s:s + C], s)
    want = ref.final_logits(C - 1)
    assert int(want.argmax()) == out["compute_only"]["top1"]
    assert abs(float(want.max()) - out["compute_only"]["logit_top1"]) < 1e-4
