"""Head-sharded tensor parallelism, verified on one B200.

Two TP ranks (tp_size=2) are separate models on the same device driven by
cake_prefill_group: per half-layer each rank runs its column-parallel QKV /
gate-up and row-parallel O / down shards, and the ranks' partial sums are added
in rank order where the multi-GPU path calls ncclAllReduce. Each rank's KV-head
shard must match the corresponding heads of the unsharded model, and the
first-token logits must match, within the bf16 tolerance of tests/test_gpu_parity.py.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (2, 1024, 8, 4, 128, 2048, 32000)  # GQA 2:1, 2 KV heads per rank at TP=2


def rel(a, b):
    return float(np.abs(a - b).max() / (np.abs(b).max() + 1e-12))


def test_tp2_matches_unsharded():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import llama_oracle
    from paper_2410_03065_b200 import native
    from paper_2410_03065_b200.cake import Cake
    from paper_2410_03065_b200.runtime import GpuRuntime

    T, C, seed = 1024, 512, 11
    cu = native.load_cuda()
    full = GpuRuntime(DIMS, max_tokens=T, max_chunk=C)
    tier = full.build_cache_tier(T, C, seed)
    full.run(tier, T, C, seed, mbps=1000, mode="compute_only")
    want_logits = full.logits()
    ranks = [GpuRuntime(DIMS, max_tokens=T, max_chunk=C, tp_rank=r, tp_size=2) for r in range(2)]
    models = (ctypes.c_void_p * 2)(*[rt.n.lib.cake_gpu_model(rt.h) for rt in ranks])
    toks = torch.tensor(Cake().token_stream(seed, T).astype(np.int32), device="cuda")
    bt = torch.arange(T // 64, dtype=torch.int32, device="cuda")
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for s in range(0, T, C):
        st = cu.cake_prefill_group(models, 2, toks[s:].data_ptr(), s, C, bt.data_ptr(), stream)
        assert st == 0
    torch.cuda.synchronize()
    L, H, nh, nkv, hd, ffn, V = DIMS
    half = nkv // 2
    for s in range(0, T, C):
        ref = llama_oracle.bf16_to_f32(np.frombuffer(full.read_chunk(s, C), dtype=np.uint16)).reshape(L, 2, nkv, C, hd)
        for r, rt in enumerate(ranks):
            nbytes = cu.cake_kv_chunk_bytes(models[r], C)
            buf = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
            assert cu.cake_kv_gather(models[r], buf.data_ptr(), s, C, bt.data_ptr(), stream) == 0
            torch.cuda.synchronize()
            got = llama_oracle.bf16_to_f32(buf.cpu().numpy().view(np.uint16)).reshape(L, 2, half, C, hd)
            assert rel(got, ref[:, :, r * half:(r + 1) * half]) <= 2e-2, (s, r)
    logits = torch.empty(V, dtype=torch.float32, device="cuda")
    assert cu.cake_final_logits(models[0], T, toks[T - 1:].data_ptr(), 0, C - 1, bt.data_ptr(), logits.data_ptr(),
                                stream) == 0
    torch.cuda.synchronize()
    got_logits = logits.cpu().numpy()
    assert rel(got_logits, want_logits) <= 2e-2
    assert want_logits[int(got_logits.argmax())] >= want_logits.max() - 2e-2 * np.abs(want_logits).max()
