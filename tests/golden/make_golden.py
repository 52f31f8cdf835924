"""Regenerate tests/golden/ref_golden.json by running the REFERENCE library
(oracle/_ref/libcake_ref.so, compiled from /root/reference/proj/src) on seeded
inputs. Hand-copied known-answer values from the reference's own tests are in
KNOWN below with their file:line. Run: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_2410_03065_b200 import native  # noqa: E402
from paper_2410_03065_b200.cake import BandwidthTrace, Cake, CostModel, RunPlan  # noqa: E402

# Known answers quoted from the reference's unit tests.
KNOWN = {
    "kv_bytes": [  # proj/tests/test_model.cpp:38-45 (7B: 32 L x 4096 x fp16; 13B: 40 L x 5120)
        {"args": [32, 4096, 2, 2, 0], "want": 524288},
        {"args": [40, 5120, 2, 2, 0], "want": 819200},
        {"args": [32, 4096, 2, 2, 1000], "want": 1000},
    ],
    "compute_latency": [  # proj/tests/test_model.cpp:98-108  CostModel{10, 0.01, 512}
        {"args": [10.0, 0.01, 512, 0, 512, 1.0], "want": 10000},
        {"args": [10.0, 0.01, 512, 1024, 512, 1.0], "want": 20240},
        {"args": [10.0, 0.01, 512, 1024, 512, 0.5], "want": 40480},
        {"args": [10.0, 0.01, 512, 1024, 512, 0.1], "want": 202400},
        {"args": [10.0, 0.01, 512, 0, 256, 1.0], "want": 5000},
        {"args": [10.0, 0.01, 512, 512, 512, 1.0], "want": 15120},  # proj/tests/test_compute.cpp:10-16
    ],
    "fetch_latency": [  # proj/tests/test_model.cpp:132-149
        {"trace": [[0, 2000]], "nbytes": 268435456, "start": 0, "want": 1073742},
        {"trace": [[0, 10000]], "nbytes": 268435456, "start": 0, "want": 214749},
        {"trace": [[0, 5000]], "nbytes": 0, "start": 0, "want": 0},
        {"trace": [[0, 1000], [1000000, 4000]], "nbytes": 140625000, "start": 0, "want": 1031250},
        {"trace": [[0, 1000], [1000000, 4000]], "nbytes": 140625000, "start": 1000000, "want": 281250},
    ],
    "oracle_best_split": [  # proj/tests/test_scheduler.cpp:123-142
        {"c": [10000, 20000, 30000, 40000], "f": [25000] * 4, "want": [2, 50000]},
        {"c": [10000, 20000, 30000, 40000], "f": [0] * 4, "want": [0, 0]},
        {"c": [10000], "f": [25000], "want": [1, 10000]},
    ],
    # proj/tests/test_scheduler.cpp:93-121 worked example: compute 10/20/30/40 ms, fetch 25 ms each
    "worked_example": {"bytes": [6400000] * 4, "cost": [10.0, 10.0 / 512.0, 512], "mbps": 2048,
                       "cake": {"ttft": 50000, "merge": 2}, "io_only": {"ttft": 100000, "merge": 0},
                       "compute_only": {"ttft": 100000, "merge": 4}},
    # proj/tests/test_compute.cpp:18-27: 64 chunks of the {10, 0.01, 512} law
    "closed_form_64": 10961920,
}


def random_instance(rng):  # shape of proj/tests/test_scheduler.cpp:44-71
    n = 1 + rng.randrange(64)
    chunk = 1 + rng.randrange(1024)
    per_token = 1000 + rng.randrange(1000000)
    counts = [chunk] * n
    if rng.randrange(3) == 0:
        counts[-1] = 1 + rng.randrange(chunk)
    starts = [sum(counts[:i]) for i in range(n)]
    bytes_ = [per_token * c for c in counts]
    cost = [0.1 + rng.randrange(500) / 10.0, rng.randrange(50) / 1000.0, chunk]
    mbps = float(100 + rng.randrange(39900))
    power = rng.choice([0.1, 0.25, 0.5, 0.75, 0.9, 1.0])
    return {"starts": starts, "counts": counts, "bytes": bytes_, "cost": cost, "mbps": mbps, "power": power}


def main():
    ref = Cake(native.load(native.REF_LIB))
    rng = random.Random(20241003)
    out = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref/libcake_ref.so (reference built from source)",
           "known": KNOWN, "fetch": [], "sim": [], "hash": {}, "codec": []}
    for _ in range(120):
        segs = 1 + rng.randrange(4)
        t, pts = 0, []
        frac = rng.randrange(4) == 0
        for _ in range(segs):
            rate = 100 + rng.randrange(20000) + (0.37 if frac else 0.0)
            pts.append([t, rate])
            t += 10000 + rng.randrange(2000000)
        nbytes = 1 + rng.randrange(500000000)
        start = rng.randrange(3000000)
        out["fetch"].append({"trace": pts, "nbytes": nbytes, "start": start,
                             "want": ref.fetch_latency(BandwidthTrace([tuple(p) for p in pts]), nbytes, start)})
    for _ in range(150):
        inst = random_instance(rng)
        plan = RunPlan(inst["starts"], inst["counts"], inst["bytes"], inst["bytes"])
        cost = CostModel(*inst["cost"])
        budget = max(512, inst["cost"][2])
        res = {}
        for mode in ("cake", "compute_only", "io_only"):
            r = ref.run_sim_planned(plan, cost, BandwidthTrace.constant(inst["mbps"]), mode, inst["power"],
                                    token_budget=budget)
            res[mode] = {"ttft": r.ttft_us, "merge": r.merge_point,
                         "rows": [[c.index, c.side, c.start_us, c.finish_us] for c in r.chunks]}
        inst["want"] = res
        out["sim"].append(inst)
    toks = ref.token_stream(42, 64)
    out["hash"]["token_stream_42_64"] = [int(x) for x in toks]
    k0 = ref.chain_hash(None, toks[:32])
    k1 = ref.chain_hash(k0, toks[32:])
    out["hash"]["chain"] = [k0.hex(), k1.hex()]
    out["hash"]["synth_payload_sha256"] = hashlib.sha256(ref.synth_payload(42, 3, 4098)).hexdigest()
    for codec in ("identity", "quant8", "factor:8.6"):
        p = ref.synth_payload(7, 1, 20000)
        enc = ref.codec_encode(codec, p)
        dec = ref.codec_decode(codec, enc, len(p))
        out["codec"].append({"codec": codec, "seed": 7, "index": 1, "n": 20000,
                             "enc_sha256": hashlib.sha256(enc).hexdigest(), "enc_len": len(enc),
                             "dec_sha256": hashlib.sha256(dec).hexdigest()})
    with open(os.path.join(HERE, "ref_golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "ref_golden.json"))


if __name__ == "__main__":
    main()
