#!/usr/bin/env python3
"""Headline benchmark: TTFT of one Llama-3-8B-shaped prompt (32K tokens, 512-token
chunks) whose saved prefix KV sits in a pinned host-DRAM cache tier behind an
emulated 8 GB/s link, filled bidirectionally on one B200 (compute forward from
token 0, loads backward from the tail, runtime merge point, race-to-finish
boundary), plus the GPU compute-only and I/O-only modes of the same request.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

A "step" is one full acquisition: request arrival -> first-token logits in host
memory. Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TTFT ms at 32K ctx (Llama-3-8B shape) vs compute-only/IO-only; chunks/s"


def workload_config(T, C, mbps, world):
    """The `config` object of both arms' JSON lines (same workload)."""
    return {"workload": f"llama3-8b-shape T={T} chunk={C} tier=pinned-DRAM link={mbps}mbps "
                        f"({mbps / 8000:g} GB/s) bidirectional+race", "model": "llama-3-8b-shape", "seq_len": T,
            "chunk": C, "link_mbps": mbps,
            "parallelism": f"tp{world} (KV-head sharded, peer-memory reductions)" if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (16 GB weights, 4 GiB KV tier) — no flush"}


DIMS_8B = (32, 4096, 32, 8, 128, 14336, 128256)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops_sustained"], p["bf16_tflops"], p["hbm_gbs"], "measured"
    except Exception:
        return 1400.0, 1590.0, 6650.0, "fallback"


# ------------------------------------------------------------------ roofline model
def chunk_flops(dims, start, count):
    L, H, nh, nkv, hd, ffn, V = dims
    linear = 2 * L * ((nh + 2 * nkv) * hd * H + H * nh * hd + 3 * ffn * H)
    attn = 4 * nh * hd * L * (count * start + count * (count + 1) / 2)
    return linear * count + attn


def ttft_roofline_ms(dims, T, C, mbps, peak_tflops, hbm_gbs, pcie_gbs=50.0, tp=1):
    """oracle_best_split (reference proj/src/scheduler.cpp:71-87) over ideal per-chunk
    times: compute at the sustained bf16 peak, loads at min(emulated link, PCIe),
    plus the memory-bound first-token step. TP: every rank computes 1/tp of each
    chunk and loads 1/tp of its KV over its own link (collectives taken as free)."""
    from paper_2410_03065_b200.cake import Cake

    L, H, nh, nkv, hd, ffn, V = dims
    kv_tok = 2 * L * nkv * hd * 2
    link = min(mbps * 1e6 / 8, pcie_gbs * 1e9)
    starts = list(range(0, T, C))
    c_us = [int(chunk_flops(dims, s, min(C, T - s)) / tp / (peak_tflops * 1e12) * 1e6) for s in starts]
    f_us = [int(min(C, T - s) * kv_tok / tp / link * 1e6) for s in starts]
    k, t = Cake().oracle_best_split(c_us, f_us)
    final_bytes = (2 * L * (nh * hd * H + H * nh * hd + 3 * ffn * H) + T * kv_tok) / tp + 2 * V * H
    final_ms = final_bytes / (hbm_gbs * 1e9) * 1e3
    return {"bidir_ms": t / 1e3 + final_ms, "k_star": k, "n_chunks": len(starts),
            "compute_only_ms": sum(c_us) / 1e3 + final_ms, "io_only_ms": sum(f_us) / 1e3 + final_ms}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU baseline
def cpu_baseline(T, C, mbps, budget_s=20.0):
    """The reference's scheduler (oracle/_ref, the reference library built from source)
    driving a CPU fp32 Llama forward (oracle/llama_ref.c) on this host's cores.
    Sample: one 8B-shaped layer of a 512-token chunk at prefix 0 and at prefix T/2,
    plus one last-token layer over the T-token cache; the per-chunk law is fitted
    from the two chunk samples, scaled to 32 layers, and the reference's own
    simulator (run_sim_planned) places the merge point at the emulated bandwidth."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np

    import llama_oracle
    from paper_2410_03065_b200 import native
    from paper_2410_03065_b200.cake import BandwidthTrace, Cake, CostModel, RunPlan

    cores = os.cpu_count() or 1
    L, H, nh, nkv, hd, ffn, V = DIMS_8B
    one = (1, H, nh, nkv, hd, ffn, V)
    mid = (T // 2) // C * C
    ref = llama_oracle.LlamaRef(one, mid + C, seed=1234, threads=cores, cache_weight_bytes=8 << 30)
    toks = np.arange(C, dtype=np.int32) % 32000
    t0 = time.time()
    ref.prefill_chunk(toks, 0)
    t_first = time.time() - t0
    t0 = time.time()
    ref.prefill_chunk(toks, mid)  # prefix KV content is irrelevant to the timing
    t_mid = time.time() - t0
    alpha_ms = L * t_first * 1e3
    beta_ms = L * max(0.0, t_mid - t_first) * 1e3 / mid
    # last-token step: one q-only row over a mid-length cache, x32 layers (+ LM head bytes at DRAM speed)
    t0 = time.time()
    ref.prefill_chunk(toks[:1], mid + C - 1)
    t_dec = (time.time() - t0) * (T / (mid + C))
    final_ms = L * t_dec * 1e3
    del ref
    lib = Cake(native.load(native.REF_LIB)) if os.path.exists(native.REF_LIB) else Cake()
    kind = "reference" if os.path.exists(native.REF_LIB) else "port"
    kv_tok = 2 * L * nkv * hd * 2
    n = -(-T // C)
    starts = [i * C for i in range(n)]
    counts = [min(C, T - s) for s in starts]
    b = [c * kv_tok for c in counts]
    plan = RunPlan(starts, counts, b, b)
    cost = CostModel(alpha_ms, beta_ms, C)
    rep = lib.run_sim_planned(plan, cost, BandwidthTrace.constant(mbps), "cake")
    comp = lib.run_sim_planned(plan, cost, BandwidthTrace.constant(mbps), "compute_only")
    return {
        "value": rep.ttft_us / 1e3 + final_ms, "unit": "ms", "cores": cores, "kind": kind,
        "sample": f"8B-shaped layer x 512-token chunk at prefix 0 ({t_first:.2f}s) and {mid} ({t_mid:.2f}s), "
                  f"last-token layer ({t_dec:.2f}s); x{L} layers, reference run_sim_planned at {mbps} mbps "
                  f"(extrapolated, merge {rep.merge_point}/{n})",
        "compute_only_ms": comp.ttft_us / 1e3 + final_ms,
        "sample_seconds": t_first + t_mid + t_dec,
    }


def config1_live_cpu(mbps=800.0, modes=("cake", "compute_only", "io_only")):
    """BASELINE config 1 served for real on the host cores, nothing extrapolated:
    the reference's own live run (oracle/_ref/ref_live_cpu: its scheduler, loader and
    store sources) with its compute sleep replaced by the CPU forward (llama_ref.c)."""
    import tempfile

    exe = os.path.join(ROOT, "oracle", "_ref", "ref_live_cpu")
    if not os.path.exists(exe):
        return None
    threads = max(1, (os.cpu_count() or 2) - 2)  # two cores stay with the loader's reader and pacer
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for mode in modes:
            p = subprocess.run([exe, "2048", "256", str(mbps), str(threads), os.path.join(d, mode), mode],
                               capture_output=True, text=True, timeout=600)
            if p.returncode != 0:
                return {"error": p.stderr[-300:]}
            out[mode] = json.loads(p.stdout)
    return out


def config1_gpu(mbps=800.0, reps=5):
    """The same config-1 request on the GPU path (tiny preset, file-free pinned tier)."""
    from paper_2410_03065_b200.runtime import GpuRuntime

    rt = GpuRuntime("tiny", max_tokens=2048, max_chunk=256)
    try:
        tier = rt.build_cache_tier(2048, 256, 42)
        out = {}
        for mode in ("cake", "compute_only", "io_only"):
            rs = [rt.run(tier, 2048, 256, 42, mbps=mbps, mode=mode) for _ in range(reps + 1)][1:]
            best = min(rs, key=lambda r: r.first_token_ms)
            out[mode] = {"first_token_ms": best.first_token_ms, "device_ttft_ms": best.device_ttft_ms,
                         "ttft_ms": best.kv_resident_ms, "merge_point": best.merge_point,
                         "top1": int(rt.logits().argmax()) if mode == "io_only" else None}
        tier.close()
        return out
    finally:
        rt.close()


# ------------------------------------------------------------------ arms
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def reference_arm(args):
    rank, local, world = dist_env()
    if rank != 0:
        return
    vals, last = [], None
    for _ in range(args.warmup):
        cpu_baseline(args.tokens, args.chunk, args.mbps)
    t0 = time.time()
    for _ in range(args.steps):
        last = cpu_baseline(args.tokens, args.chunk, args.mbps)
        vals.append(last["value"])
    wall = (time.time() - t0) / max(1, args.steps)
    v = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(args.tokens, args.chunk, args.mbps, 1),
                           parallelism=f"host CPU, {last['cores']} threads (reference scheduler + CPU Llama forward)"),
            "cpu_baseline": dict({k: last[k] for k in ("value", "unit", "cores", "kind", "sample")},
                                 config1_live=config1_live_cpu()),
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def b200_arm(args):
    rank, local, world = dist_env()
    dist = None
    tp_kw = {}
    if world > 1:
        import ctypes
        import uuid

        import torch
        import torch.distributed as td

        from paper_2410_03065_b200 import native as N

        if args.share_device:  # functional check of the multi-process path on one GPU
            local = 0
        torch.cuda.set_device(local)
        if args.share_device:
            td.init_process_group("gloo")
        else:
            td.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist = td
        # ONE request, KV-head-sharded over the group; coordinator
        # name from rank 0. The per-layer reductions run over peer memory
        # (tp_peer.cuh, CUDA IPC handles all-gathered below) or, with
        # --tp-reduce nccl, the baseline ncclAllReduce on the model's own
        # communicator (torch's group only does barriers / the max below).
        cl = N.load_cuda()
        uid = (ctypes.c_uint8 * 128)()
        if args.tp_reduce == "nccl" and rank == 0 and cl.cake_nccl_unique_id(uid) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        obj = [bytes(uid), f"/cake_tp_{uuid.uuid4().hex[:16]}"]
        td.broadcast_object_list(obj, src=0)
        tp_kw = dict(tp_rank=rank, tp_size=world, tp_shm=obj[1])
        if args.tp_reduce == "nccl":
            ctypes.memmove(uid, obj[0], 128)
            comm = ctypes.c_void_p()
            cl.cake_cuda_set_device(local)
            if cl.cake_nccl_init(ctypes.byref(comm), uid, world, rank) != 0:
                raise RuntimeError("ncclCommInitRank failed")
            tp_kw["nccl_comm"] = comm.value
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C, mbps = args.tokens, args.chunk, args.mbps
    seed = 42  # every TP rank serves the same prompt
    rt = GpuRuntime("llama3_8b", max_tokens=T, max_chunk=C, device=local, **tp_kw)
    if world > 1 and args.tp_reduce == "peer":
        handles = [None] * world
        dist.all_gather_object(handles, rt.tp_peer_handles())
        rt.tp_peer_open(handles)
    rt.calibrate(T, C, seed)
    tier = rt.build_cache_tier(T, C, seed)

    def one(mode="cake"):
        t0 = time.perf_counter()
        r = rt.run(tier, T, C, seed, mbps=mbps, mode=mode, race=not args.no_race)
        return r, (time.perf_counter() - t0) * 1e3

    base_c = min((one("compute_only")[0] for _ in range(2)), key=lambda r: r.first_token_ms)
    base_io = min((one("io_only")[0] for _ in range(2)), key=lambda r: r.first_token_ms)
    # warm-up 1 is fully event-bracketed: the per-kernel breakdown ("kernels") and
    # the choice of the dominant kernel class
    rt.set_profiling("all")
    one()
    breakdown = rt.kernel_stats(reset=True)
    rt.set_profiling(None)
    dom_name = max(breakdown, key=lambda k: breakdown[k]["ms"])
    for _ in range(args.warmup - 1):
        one()
    rt.kernel_stats(reset=True)

    def barrier():
        if dist:
            import torch

            torch.cuda.synchronize()
            dist.barrier()

    # timed steps: no event brackets (every programmatic-launch chain intact)
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    res, walls = [], []
    for _ in range(args.steps):
        r, w = one()
        res.append(r)
        walls.append(w)
    barrier()
    clk = clocks.stop()
    stats = None
    if args.profile:
        # roofline steps, right after the timed region on the same warm state: every
        # launch of the dominant class is bracketed by CUDA events on its own stream
        rt.kernel_stats(reset=True)
        rt.set_profiling([dom_name], stride=1)
        for _ in range(max(1, min(args.steps, 3))):
            one()
        stats = rt.kernel_stats(reset=True)
        rt.set_profiling(None, stride=1)

    dev = statistics.mean(r.device_ttft_ms for r in res)
    e2e = statistics.mean(r.first_token_ms for r in res)
    wall = statistics.mean(walls)
    if dist:
        import torch

        t = torch.tensor([dev, e2e, wall], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev, e2e, wall = t.tolist()
    if rank != 0:
        return
    peak_s, peak_b, hbm, peak_kind = load_peaks()
    roof = ttft_roofline_ms(DIMS_8B, T, C, mbps, peak_s, hbm, tp=world)
    last = res[-1]
    # dominant kernel class, timed live in the timed region (CUDA events bracketing
    # each of its launches on its own stream); its share from the bracketed warm-up
    total = sum(v["ms"] for v in breakdown.values()) or 1.0
    d = stats[dom_name] if stats and stats[dom_name]["launches"] else breakdown[dom_name]
    tensor_bound = is_tensor_bound(d)
    if tensor_bound:
        achieved = d["flops"] / (d["ms"] / 1e3) / 1e12
        rl = {"bound": "tensor", "achieved": achieved, "peak": peak_s, "unit": "TFLOP/s", "frac": achieved / peak_s}
    else:
        achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9
        rl = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm}
    rl.update({"kernel": dom_name, "share_of_kernel_time": breakdown[dom_name]["ms"] / total,
               "launches": d["launches"],
               "per_launch_ms": d["ms"] / max(1, d["launches"]),
               "peak_kind": f"{peak_kind} bf16 sustained" if tensor_bound else f"{peak_kind} hbm",
               "traffic": traffic_from_profiles(dom_name)})
    kernels = {k: class_roofline(v, peak_s, hbm) for k, v in breakdown.items() if v["launches"]}
    line = {
        "metric": METRIC, "value": dev, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init Llama-3-8B-shape weights, seeded prompt)",
        "config": workload_config(T, C, mbps, world),
        "ttft_compute_only_ms": base_c.device_ttft_ms, "ttft_io_only_ms": base_io.device_ttft_ms,
        "ttft_vs_min_baseline": dev / min(base_c.device_ttft_ms, base_io.device_ttft_ms),
        "chunks_per_s": last.n_chunks / (dev / 1e3), "merge_point": last.merge_point, "n_chunks": last.n_chunks,
        "raced_chunk": last.raced_chunk, "race_winner": last.race_winner, "kv_resident_ms": last.kv_resident_ms,
        "final_step_ms": last.final_step_ms,
        "ttft_roofline": {"bidir_ms": roof["bidir_ms"], "k_star": roof["k_star"],
                          "compute_only_ms": roof["compute_only_ms"], "io_only_ms": roof["io_only_ms"],
                          "frac": roof["bidir_ms"] / dev},
        "e2e": {"value": e2e, "unit": "ms", "h2d_bytes_per_step": last.h2d_bytes,
                "d2h_bytes_per_step": last.d2h_bytes},
        "gpu_launches": last.kernel_launches,
        "roofline": rl, "kernels_bracketed_warmup_step": kernels, "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:
        try:
            line["cpu_baseline"] = {k: v for k, v in cpu_baseline(T, C, mbps).items()
                                    if k in ("value", "unit", "cores", "kind", "sample")}
            # BASELINE config 1 end to end on both: the reference's live loop on the host
            # cores (no extrapolation) next to the GPU path, same prompt and link
            line["config1"] = {"workload": "tiny 2-layer d=256 4-head, T=2048 chunk=256, tier behind 800 mbps",
                               "cpu_live": config1_live_cpu(), "gpu": config1_gpu()}
        except Exception as e:  # reported, never fatal to the GPU line
            line["cpu_baseline"] = {"value": None, "unit": "ms", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"failed: {e}"}
    print(json.dumps(line), flush=True)


def is_tensor_bound(v):
    """Arithmetic intensity above the B200 ridge (~200 FLOP/B): tensor-pipe bound."""
    return v["flops"] > 0 and v["flops"] / max(v["bytes"], 1) > 300


def class_roofline(v, peak_tflops, hbm_gbs):
    """Per-class line of the bracketed warm-up step: time, launches, achieved rate
    against the roof that bounds the class (bf16 sustained or HBM)."""
    ms = v["ms"]
    out = {"ms_per_step": ms, "launches_per_step": v["launches"],
           "tflops": (v["flops"] / (ms / 1e3) / 1e12) if ms > 0 and v["flops"] > 0 else None,
           "gbs": (v["bytes"] / (ms / 1e3) / 1e9) if ms > 0 else None}
    if ms > 0 and (v["flops"] > 0 or v["bytes"] > 0):
        if is_tensor_bound(v):
            out.update(bound="tensor", frac=out["tflops"] / peak_tflops)
        else:
            out.update(bound="hbm", frac=out["gbs"] / hbm_gbs)
    return out


def traffic_from_profiles(kernel):
    """dram bytes per launch for `kernel` from the committed ncu summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--chunk", type=int, default=512)
    ap.add_argument("--mbps", type=float, default=64000.0)
    ap.add_argument("--no-race", action="store_true")
    ap.add_argument("--no-profile", dest="profile", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tp-reduce", default="peer", choices=["peer", "nccl"],
                    help="TP reductions: one peer-memory kernel (product) or ncclAllReduce (baseline)")
    ap.add_argument("--share-device", action="store_true",
                    help="every rank on GPU 0 (functional check of the multi-process path on one GPU)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch our own ranks when not started by torchrun
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.run(cmd).returncode)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
