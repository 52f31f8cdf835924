"""Golden vectors for the quant8 tier codec, produced by the REFERENCE library
(oracle/_ref/libcake_ref.so, built from /root/reference/proj/src/codec.cpp).

Run here (where /root/reference exists):  python tests/golden/make_q8_golden.py
Writes tests/golden/q8_golden.json: fp16 payloads with the reference's
encoding and decoding (hex). The GPU box never needs the reference.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2410_03065_b200 import native  # noqa: E402
from paper_2410_03065_b200.cake import Cake  # noqa: E402


def cases():
    rng = np.random.default_rng(2410)
    yield "uniform_pm1", rng.uniform(-1, 1, 1024).astype(np.float16)
    yield "kv_like", (rng.standard_normal(2048) * 2.5).astype(np.float16)
    yield "constant", np.full(512, 0.3125, dtype=np.float16)  # proj/tests/test_codec.cpp:103
    yield "single", np.array([-7.25], dtype=np.float16)
    yield "two_levels", np.array([0.0, 1.0] * 64, dtype=np.float16)
    yield "halfway", (np.arange(511, dtype=np.float32) / 510.0).astype(np.float16)  # hits .5 levels
    yield "wide", np.concatenate([rng.uniform(-60000, 60000, 256), [65504.0, -65504.0]]).astype(np.float16)
    yield "tiny", (rng.standard_normal(300) * 1e-4).astype(np.float16)


def main():
    ref = Cake(native.load(native.REF_LIB))
    out = []
    for name, v in cases():
        payload = v.tobytes()
        enc = ref.codec_encode("quant8", payload)
        dec = ref.codec_decode("quant8", enc, len(payload))
        out.append({"name": name, "payload": payload.hex(), "encoded": enc.hex(), "decoded": dec.hex()})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "q8_golden.json")
    with open(path, "w") as f:
        json.dump({"source": "oracle/_ref/libcake_ref.so (reference proj/src/codec.cpp:114-162)", "cases": out}, f)
    print(f"wrote {path}: {len(out)} cases")


if __name__ == "__main__":
    main()
