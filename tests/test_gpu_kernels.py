"""sm_100a kernels through the C ABI (libcake_cuda.so), on a B200.

GEMM: tcgen05/TMEM/TMA kernel vs a plain torch fp32 matmul of the same bf16
operands (tolerance: fp32 accumulation-order noise, ~1e-3 relative).
KV scatter/gather: bit-exact permutation between the cache-tier chunk format
and the paged pool, through arbitrary block tables.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_03065_b200 import native

    return native.load_cuda()


def _stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _err(cu):
    buf = ctypes.create_string_buffer(1024)
    cu.cake_cuda_last_error(buf, 1024)
    return buf.value.decode()


@pytest.mark.parametrize("M,N,K,bn", [(128, 256, 64, 256), (1, 128, 4096, 128), (77, 512, 1024, 128),
                                      (512, 6144, 4096, 256), (300, 4096, 14336, 128), (640, 28672, 4096, 256)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_gemm_matches_torch(cu, M, N, K, bn, epi):
    import torch

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    ref = a.float() @ b.float().t()
    if epi == 0:
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    elif epi == 1:
        c = torch.empty(M, N, device="cuda", dtype=torch.float32)
    else:
        c = torch.full((M, N), 0.5, device="cuda", dtype=torch.float32)
    st = cu.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, epi, bn, _stream())
    assert st == 0, _err(cu)
    torch.cuda.synchronize()
    got = c.float() - (0.5 if epi == 2 else 0.0)
    scale = ref.abs().max().item()
    tol = 1e-2 * scale if epi == 0 else 2e-4 * scale  # bf16 output rounding / fp32 order noise
    assert (got - ref).abs().max().item() <= tol


@pytest.mark.parametrize("M,N,K,bn", [(512, 4096, 4096, 128), (512, 6144, 4096, 192), (384, 4096, 14336, 128),
                                      (1024, 4096, 1024, 128), (200, 1024, 512, 128)])
@pytest.mark.parametrize("schedule", [0, 256, 512])
def test_gemm_pair_clusters_match_torch(cu, M, N, K, bn, schedule):
    """Schedule 0: the A-sharing pair clusters (gemm2c, 2 pairs), 512: 4 pairs,
    256: unclustered pairs (gemm2) — against torch, every epilogue."""
    import torch

    assert cu.cake_gemm_set_schedule(schedule) == 0
    try:
        for epi in (0, 1, 2):
            if bn == 192 and epi != 0:
                continue
            g = torch.Generator(device="cuda").manual_seed(M + N + K + epi)
            a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
            b = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
            ref = a.float() @ b.float().t()
            c = (torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi == 0 else
                 torch.full((M, N), 0.5, device="cuda", dtype=torch.float32))
            st = cu.cake_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, epi, bn, _stream())
            assert st == 0, _err(cu)
            torch.cuda.synchronize()
            got = c.float() - (0.5 if epi == 2 else 0.0)
            scale = ref.abs().max().item()
            tol = 1e-2 * scale if epi == 0 else 2e-4 * scale
            assert (got - ref).abs().max().item() <= tol, (epi, (got - ref).abs().max().item())
    finally:
        cu.cake_gemm_set_schedule(0)


def test_gemm_rejects_bad_shapes(cu):
    st = cu.cake_gemm(None, None, None, 128, 100, 64, 0, 128, None)
    assert st != 0 and "bad shape" in _err(cu)


@pytest.fixture(scope="module")
def tiny_rt():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_03065_b200.runtime import GpuRuntime

    return GpuRuntime((2, 256, 4, 2, 128, 1024, 32000), max_tokens=1024, max_chunk=256)


def test_kv_scatter_gather_bit_exact(cu, tiny_rt):
    """random bytes -> staging -> scatter (permuted block table) -> gather == input."""
    import torch

    from paper_2410_03065_b200 import native

    model = tiny_rt.n.lib.cake_gpu_model(tiny_rt.h)
    n_pages = 1024 // 64
    perm = torch.tensor(np.random.default_rng(0).permutation(n_pages).astype(np.int32), device="cuda")
    for start, length in [(0, 256), (256, 192), (512, 64), (768, 256)]:
        nbytes = cu.cake_kv_chunk_bytes(model, length)
        src = torch.randint(-(2 ** 15), 2 ** 15, (nbytes // 2,), dtype=torch.int16, device="cuda")
        st = cu.cake_kv_scatter(model, src.data_ptr(), start, length, perm.data_ptr(), 0, nbytes, _stream())
        assert st == 0, _err(cu)
        back = torch.zeros_like(src)
        st = cu.cake_kv_gather(model, back.data_ptr(), start, length, perm.data_ptr(), _stream())
        assert st == 0, _err(cu)
        torch.cuda.synchronize()
        assert torch.equal(src, back)
    # partial byte ranges compose (per-slice scatter)
    nbytes = cu.cake_kv_chunk_bytes(model, 256)
    src = torch.randint(-(2 ** 15), 2 ** 15, (nbytes // 2,), dtype=torch.int16, device="cuda")
    cut = (nbytes // 3) // 16 * 16
    assert cu.cake_kv_scatter(model, src.data_ptr(), 0, 256, perm.data_ptr(), 0, cut, _stream()) == 0
    assert cu.cake_kv_scatter(model, src.data_ptr(), 0, 256, perm.data_ptr(), cut, nbytes, _stream()) == 0
    back = torch.zeros_like(src)
    assert cu.cake_kv_gather(model, back.data_ptr(), 0, 256, perm.data_ptr(), _stream()) == 0
    torch.cuda.synchronize()
    assert torch.equal(src, back)
    assert native  # keep import used


def test_kv_scatter_rejects_misaligned(cu, tiny_rt):
    model = tiny_rt.n.lib.cake_gpu_model(tiny_rt.h)
    assert cu.cake_kv_scatter(model, None, 32, 64, None, 0, 16, None) != 0  # not page aligned
    assert cu.cake_kv_scatter(model, None, 0, 64, None, 0, 10, None) != 0  # not 16-B aligned


ATTN_MODELS = {
    # name: dims (L, H, n_heads, n_kv, hd, ffn, vocab) — GQA 4:1 at hd 128 and 64, and 8:1
    "gqa4_hd128": (1, 1024, 8, 2, 128, 1024, 32000),
    "gqa4_hd64": (1, 512, 8, 2, 64, 1024, 32000),
    "gqa8_hd128": (1, 2048, 16, 2, 128, 1024, 32000),
}
# (chunk_start, chunk_len): prefill chunks at several prefixes (odd and even 128-key block counts, a
# ragged tail), and single-token rows at an unaligned position (split-KV + the combine)
ATTN_CASES = [(0, 512), (512, 512), (1536, 512), (2048, 200), (0, 37), (3583, 1), (1000, 1)]


@pytest.mark.parametrize("scores", ["flat", "growing"])
@pytest.mark.parametrize("impl", ["tcgen05", "tcgen05_1tile", "mma_sync"])
@pytest.mark.parametrize("name", list(ATTN_MODELS))
def test_attention_kernel_matches_torch(cu, name, impl, scores):
    """The attention kernels alone (cake_attention_debug) against a plain fp32 attention of the same
    bf16 inputs: random K/V scattered into the paged pool through a permuted block table, random Q,
    causal over the prefix. "growing" scales the keys up along the sequence, so rows move their
    running max block after block at different times (the online-softmax rescale of O in TMEM runs
    for some rows of a warp and not others: the case that once hung the tcgen05 kernels).
    Tolerance: RMS-normalised error <= 2^-7 (bf16 P and output)."""
    import torch

    from paper_2410_03065_b200.runtime import GpuRuntime

    dims = ATTN_MODELS[name]
    L, H, nq, nkv, hd = dims[:5]
    T = 4096
    rt = GpuRuntime(dims, max_tokens=T, max_chunk=512)
    rt.set_attention_impl(impl)
    model = rt.n.lib.cake_gpu_model(rt.h)
    g = torch.Generator(device="cuda").manual_seed(7)
    n_pages = T // 64
    perm = torch.tensor(np.random.default_rng(1).permutation(n_pages).astype(np.int32), device="cuda")
    # KV of every position in the tier's chunk layout [layer][K|V][kv head][token][hd], 512 tokens a chunk
    kv = torch.randn(T, L, 2, nkv, hd, device="cuda", generator=g) * 2.0
    if scores == "growing":
        kv[:, :, 0] *= torch.linspace(0.5, 4.0, T, device="cuda")[:, None, None, None]
    kv = kv.to(torch.bfloat16)
    for s0 in range(0, T, 512):
        staging = kv[s0:s0 + 512].permute(1, 2, 3, 0, 4).contiguous()
        nbytes = cu.cake_kv_chunk_bytes(model, 512)
        assert staging.numel() * 2 == nbytes
        assert cu.cake_kv_scatter(model, staging.data_ptr(), s0, 512, perm.data_ptr(), 0, nbytes, _stream()) == 0, \
            _err(cu)
    G = nq // nkv
    for start, length in ATTN_CASES:
        q = (torch.randn(length, nq, hd, device="cuda", generator=g) * 2.0).to(torch.bfloat16)
        out = torch.empty_like(q)
        assert cu.cake_attention_debug(model, q.data_ptr(), start, length, 0, perm.data_ptr(), out.data_ptr(),
                                       _stream()) == 0, _err(cu)
        torch.cuda.synchronize()
        end = start + length
        k = kv[:end, 0, 0].float()  # [keys, nkv, hd]
        v = kv[:end, 0, 1].float()
        qf = q.float()
        kh = k.repeat_interleave(G, dim=1)  # q head h reads kv head h // G
        vh = v.repeat_interleave(G, dim=1)
        scores = torch.einsum("thd,khd->htk", qf, kh) / hd ** 0.5
        pos = torch.arange(start, end, device="cuda")[:, None]
        keys = torch.arange(end, device="cuda")[None, :]
        scores = scores.masked_fill((keys > pos)[None], float("-inf"))
        ref = torch.einsum("htk,khd->thd", torch.softmax(scores, dim=-1), vh)
        got = out.float()
        assert torch.isfinite(got).all(), (name, impl, start, length)
        err = float(torch.sqrt(torch.mean((got - ref) ** 2)) / torch.sqrt(torch.mean(ref ** 2)))
        assert err <= 2.0 ** -7, (name, impl, start, length, err)
    rt.close()
