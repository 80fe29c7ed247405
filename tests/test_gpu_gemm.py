"""tcgen05 GEMM: numerics against an fp64 torch reference, and batch invariance (bitwise).

The reduction order inside one tcgen05.mma (K=16) is hardware-defined, so the GEMM is checked
against fp64 within a bound derived from the magnitudes; everything that decides bits on our side
(K order, tile shape, sub-tile position) is checked bitwise across batch sizes and permutations.
"""
import pytest

pytestmark = pytest.mark.gpu


def _gemm(W, X, n_out=None):
    import torch
    from paper_2602_00182_b200._lib import lib, check

    n_out = W.shape[0] if n_out is None else n_out
    Y = torch.full((X.shape[0], n_out), float("nan"), dtype=torch.float32, device=W.device)
    check(lib.detgpu_k_gemm(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, W.shape[1], X.shape[0], n_out, None))
    torch.cuda.synchronize()
    return Y


def _rand_bf16(shape, gen, scale=1.0):
    import torch

    return (torch.rand(shape, generator=gen, dtype=torch.float32) * 2 - 1).mul(scale).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("n_out,K,ncols", [(128, 64, 1), (256, 256, 8), (384, 512, 64), (512, 1024, 100),
                                            (256, 4096, 256), (128, 768, 300), (1024, 256, 513)])
def test_gemm_matches_fp64(n_out, K, ncols):
    import torch

    g = torch.Generator().manual_seed(n_out * 7 + K + ncols)
    W = _rand_bf16((n_out, K), g)
    X = _rand_bf16((ncols, K), g)
    Y = _gemm(W, X)
    ref = X.double() @ W.double().T
    bound = (X.double().abs() @ W.double().abs().T) * (K * 2.0 ** -23) + 1e-30
    err = (Y.double() - ref).abs()
    assert torch.isfinite(Y).all()
    assert (err <= bound).all(), f"max err {err.max().item()} bound {bound.min().item()}"


@pytest.mark.parametrize("n_out,K,ncols,scale", [(128, 64, 3, 1.0), (256, 4096, 17, 0.02), (128, 14336, 5, 0.01),
                                                  (384, 256, 70, 30.0)])
def test_gemm_bit_exact_with_b200_profile(n_out, K, ncols, scale):
    """Every output equals the oracle's b200 accumulation profile bit for bit."""
    import numpy as np
    import torch

    from oracle import oracle as O

    g = torch.Generator().manual_seed(K + ncols)
    W = _rand_bf16((n_out, K), g, scale)
    X = _rand_bf16((ncols, K), g)
    Y = _gemm(W, X)
    Wn = W.view(torch.int16).cpu().numpy().view(np.uint16)
    Xn = X.view(torch.int16).cpu().numpy().view(np.uint16)
    ref = O.gemm(Wn, Xn)
    assert (Y.cpu().numpy().view(np.uint32) == ref.view(np.uint32)).all()


def test_batch_invariance_bitwise():
    import torch

    g = torch.Generator().manual_seed(1234)
    W = _rand_bf16((512, 1024), g, 0.05)
    X = _rand_bf16((300, 1024), g)
    full = _gemm(W, X)
    for n in (1, 2, 7, 63, 64, 65, 128, 129, 255, 256, 257):
        part = _gemm(W, X[:n].contiguous())
        assert torch.equal(part.view(torch.int32), full[:n].view(torch.int32)), f"ncols={n}"
    perm = torch.randperm(300, generator=g)
    permuted = _gemm(W, X[perm.cuda()].contiguous())
    assert torch.equal(permuted.view(torch.int32), full[perm.cuda()].view(torch.int32))
    # single column at every sub-tile position of a 256-wide tile
    col = X[5:6]
    for pos in (0, 1, 31, 63, 64, 127, 200, 255):
        Xp = X[:256].clone()
        Xp[pos] = col[0]
        Yp = _gemm(W, Xp)
        assert torch.equal(Yp[pos].view(torch.int32), full[5].view(torch.int32)), f"pos={pos}"


def test_repeat_bitwise():
    import torch

    g = torch.Generator().manual_seed(99)
    W = _rand_bf16((1024, 4096), g, 0.02)
    X = _rand_bf16((16, 4096), g)
    first = _gemm(W, X)
    for _ in range(20):
        assert torch.equal(_gemm(W, X).view(torch.int32), first.view(torch.int32))


def test_wide_mma_form_is_bit_identical():
    """One N = nb*64 tcgen05.mma per K step (the engine's form) gives the same column bits as nb
    separate N = 64 instructions."""
    import torch
    from paper_2602_00182_b200._lib import check, lib

    g = torch.Generator().manual_seed(5)
    for n_out, K, ncols in [(256, 512, 256), (512, 4096, 200), (384, 256, 70)]:
        W = _rand_bf16((n_out, K), g, 0.05)
        X = _rand_bf16((ncols, K), g)
        Y1 = torch.empty(ncols, n_out, device="cuda")
        Y2 = torch.empty(ncols, n_out, device="cuda")
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y1.data_ptr(), n_out, K, ncols, n_out, 0, None))
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y2.data_ptr(), n_out, K, ncols, n_out, -1, None))
        torch.cuda.synchronize()
        assert torch.equal(Y1.view(torch.int32), Y2.view(torch.int32))


def test_cta_pair_gemm_bit_identical():
    """The CTA-pair form (gemm_pair_kernel: tcgen05.mma.cta_group::2, M = 256, each CTA holding its
    128 weight rows and half of the 128 activation columns) against the one-CTA form, S = 1..8 (up
    to 16-CTA clusters): every output bit equal."""
    import torch
    from paper_2602_00182_b200._lib import lib, check

    g = torch.Generator().manual_seed(5)
    for n_out, K, ncols, S in [(256, 256, 65, 1), (256, 512, 128, 2), (512, 1024, 200, 2), (512, 4096, 256, 4),
                               (768, 2048, 300, 5), (256, 4096, 129, 8), (1024, 1024, 512, 3)]:
        W = _rand_bf16((n_out, K), g, 0.05)
        X = _rand_bf16((ncols, K), g)
        Y1 = torch.full((ncols, n_out), float("nan"), device="cuda")
        Y2 = Y1.clone()
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y1.data_ptr(), n_out, K, ncols, n_out, S, None))
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y2.data_ptr(), n_out, K, ncols, n_out, 200 + S, None))
        torch.cuda.synchronize()
        assert torch.equal(Y1.view(torch.int32), Y2.view(torch.int32)), (n_out, K, ncols, S)


def test_persistent_gemm_bit_identical():
    """The persistent many-column form (gemm_persist_kernel: clusters of S CTAs walking (tile, 128-
    column) units with double-buffered TMEM accumulators and mbarrier hand-offs over DSMEM) against
    the one-unit-per-cluster form: every output bit equal, S = 2..8, ragged column counts, several
    units per cluster (the accumulator buffers and the partial tile reused)."""
    import torch
    from paper_2602_00182_b200._lib import lib, check

    g = torch.Generator().manual_seed(9)
    for n_out, K, ncols, S in [(256, 512, 65, 2), (512, 1024, 200, 2), (2048, 1024, 1000, 2), (768, 2048, 300, 5),
                               (4096, 4096, 512, 8), (1024, 1024, 129, 3), (6144, 4096, 256, 5), (4096, 14336, 384, 8),
                               (28672, 4096, 130, 2)]:
        W = _rand_bf16((n_out, K), g, 0.05)
        X = _rand_bf16((ncols, K), g)
        Y1 = torch.full((ncols, n_out), float("nan"), device="cuda")
        Y2 = Y1.clone()
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y1.data_ptr(), n_out, K, ncols, n_out, S, None))
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y2.data_ptr(), n_out, K, ncols, n_out, 300 + S, None))
        torch.cuda.synchronize()
        assert torch.equal(Y1.view(torch.int32), Y2.view(torch.int32)), (n_out, K, ncols, S)
