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
