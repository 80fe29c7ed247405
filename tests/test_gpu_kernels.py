"""Kernel-level parity: every non-GEMM kernel is BIT-EXACT with the CPU oracle on the same inputs.

(The GEMM's in-instruction accumulation order is hardware-defined: see test_gpu_gemm.py.)
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2602_00182_b200._lib import check, lib

    return lib, check


def _u16_to_bf16_tensor(a):
    import torch

    return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).cuda()


def _bf16_tensor_to_u16(t):
    import torch

    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def test_expf_bit_exact_with_libm():
    import torch

    lib, check = _lib()
    bits = np.arange(0, 2**32, 251, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x) & (x >= -104.0) & (x <= 88.72)]
    x = np.concatenate([x, np.array([0.0, -0.0, -1e-38, -87.33654, -88.0, -103.97, -104.0, -1e4, float("-inf"),
                                     88.72, 89.0, 1e4, float("inf"), float("nan")], dtype=np.float32)])
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty_like(xt)
    check(lib.detgpu_k_expf(xt.data_ptr(), yt.data_ptr(), xt.numel(), None))
    y = yt.cpu().numpy()
    ref = O.libm_expf(x)
    same = (y.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(y) & np.isnan(ref))
    assert same.all(), x[~same][:5]


@pytest.mark.parametrize("n", [1, 3, 32, 100, 128, 129, 1000, 4096, 14336, 128256, 131072])
def test_tree_sum_bit_exact(n):
    import torch

    lib, check = _lib()
    rng = np.random.default_rng(n)
    rows = 4
    x = (rng.standard_normal((rows, n)) * np.exp2(rng.integers(-8, 8, (rows, n)))).astype(np.float32)
    x[0, ::5] = -0.0
    xt = torch.from_numpy(x).cuda()
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    check(lib.detgpu_k_tree_sum(xt.data_ptr(), out.data_ptr(), rows, n, None))
    got = out.cpu().numpy()
    for r in range(rows):
        assert got[r].view(np.uint32) == O.tree_reduce(x[r]).view(np.uint32), r


@pytest.mark.parametrize("d", [256, 4096])
def test_rmsnorm_bit_exact(d):
    import torch

    lib, check = _lib()
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((7, d)) * 3).astype(np.float32)
    gamma = O.gen_tensor(123, 1, d, 0, True)[0]
    out = torch.empty((7, d), dtype=torch.bfloat16, device="cuda")
    xt, gt = torch.from_numpy(x).cuda(), _u16_to_bf16_tensor(gamma)   # keep both alive across the call
    check(lib.detgpu_k_rmsnorm(xt.data_ptr(), gt.data_ptr(), out.data_ptr(), 7, d, 1e-5, None))
    torch.cuda.synchronize()
    assert (_bf16_tensor_to_u16(out) == O.rmsnorm(x, gamma)).all()


@pytest.mark.parametrize("rows,cols,scale,gamma,mul,add", [(33, 256, -4, False, 1, 0), (1, 4096, 0, True, 1, 0),
                                                            (64, 128, -7, False, 2, 1)])
def test_weight_generation_bit_exact(rows, cols, scale, gamma, mul, add):
    import torch

    lib, check = _lib()
    seed = 0x1234567890ABCDEF
    dst = torch.zeros((rows * mul + add, cols), dtype=torch.bfloat16, device="cuda")
    check(lib.detgpu_k_init_tensor(dst.data_ptr(), seed, rows, cols, scale, int(gamma), mul, add, None))
    torch.cuda.synchronize()
    got = _bf16_tensor_to_u16(dst)[add::mul][:rows]
    assert (got == O.gen_tensor(seed, rows, cols, scale, gamma)).all()


@pytest.mark.parametrize("hd,hq,hkv,ctxs", [(64, 4, 2, [1, 5, 128, 129, 300]), (128, 32, 8, [1, 200, 257, 640])])
def test_attention_bit_exact(hd, hq, hkv, ctxs):
    """Paged decode attention (fixed 128-position chunks) vs the oracle, one query per column."""
    import torch

    lib, check = _lib()
    rng = np.random.default_rng(hd + len(ctxs))
    page, ncols = 64, len(ctxs)
    max_ctx = max(ctxs)
    pps = (max_ctx + page - 1) // page
    total_pages = pps * ncols
    # shuffled page table to exercise the indirection
    perm = rng.permutation(total_pages).astype(np.int32)
    table = perm.reshape(ncols, pps)
    def bf(shape):
        return np.frombuffer(np.array(rng.standard_normal(shape), dtype=np.float32).tobytes(), dtype=np.uint32)\
            .reshape(shape).__rshift__(16).astype(np.uint16)
    kpool = bf((total_pages, hkv, page, hd))
    vpool = bf((total_pages, hkv, page, hd))
    q = bf((ncols, hq * hd))
    pos = np.array([c - 1 for c in ctxs], dtype=np.int32)
    req = np.arange(ncols, dtype=np.int32)
    out = torch.zeros((ncols, hq * hd), dtype=torch.bfloat16, device="cuda")
    tens = [_u16_to_bf16_tensor(a) for a in (q, kpool, vpool)]
    tt = torch.from_numpy(table.copy()).cuda()
    pt = torch.from_numpy(pos).cuda()
    rt = torch.from_numpy(req).cuda()
    check(lib.detgpu_k_attention(tens[0].data_ptr(), tens[1].data_ptr(), tens[2].data_ptr(), tt.data_ptr(),
                                 pt.data_ptr(), rt.data_ptr(), out.data_ptr(), ncols, hq, hkv, hd, page, pps, None))
    torch.cuda.synchronize()
    got = _bf16_tensor_to_u16(out)
    G = hq // hkv
    for c, ctx in enumerate(ctxs):
        for h in range(hq):
            kvh = h // G
            k = np.stack([kpool[table[c, p // page], kvh, p % page] for p in range(ctx)])
            v = np.stack([vpool[table[c, p // page], kvh, p % page] for p in range(ctx)])
            ref = O.attention_head(q[c, h * hd:(h + 1) * hd], k, v)
            assert (got[c, h * hd:(h + 1) * hd] == ref).all(), (c, h, ctx)


def _sample(logits, policies, seeds):
    import ctypes as C
    import torch
    from paper_2602_00182_b200._lib import Policy

    lib, check = _lib()
    rows, V = logits.shape
    lt = torch.from_numpy(np.ascontiguousarray(logits)).cuda()
    st = np.stack([O.Prng(s).s for s in seeds]).astype(np.uint64)
    stt = torch.from_numpy(st.view(np.int64).copy()).cuda()
    tok = torch.zeros(rows, dtype=torch.int32, device="cuda")
    probs = torch.zeros((rows, V), dtype=torch.float32, device="cuda")
    status = torch.zeros(rows, dtype=torch.int32, device="cuda")
    pols = (Policy * rows)(*[Policy(k, kk is not None, pp is not None, 0, kk or 0, pp or 0.0, 1)
                             for (k, kk, pp) in policies])
    check(lib.detgpu_k_sample(lt.data_ptr(), rows, V, pols, stt.data_ptr(), tok.data_ptr(), probs.data_ptr(),
                              status.data_ptr(), None))
    return (tok.cpu().numpy(), probs.cpu().numpy(), stt.cpu().numpy().view(np.uint64), status.cpu().numpy())


@pytest.mark.parametrize("V", [32, 4096, 128256])
def test_softmax_decode_bit_exact(V):
    rng = np.random.default_rng(V)
    policies = [(0, None, None), (1, 1, None), (1, 4, None), (1, 40, None), (1, 2000, None), (2, None, 0.9),
                (2, None, 0.5), (2, None, 1.0), (0, None, None), (2, None, 0.999)]
    rows = len(policies)
    scale = np.array([9.0, 9.0, 3.0, 1.0, 0.3, 9.0, 2.0, 0.5, 0.001, 0.05])[:, None]
    logits = (rng.standard_normal((rows, V)) * scale).astype(np.float32)
    logits[0, 7] = logits[0].max() + 0.0  # exact tie at the max: smallest index wins
    logits[0, 3] = logits[0, 7]
    seeds = [11 + i for i in range(rows)]
    tok, probs, state, status = _sample(logits, policies, seeds)
    assert (status == 0).all()
    for r, (kind, k, p) in enumerate(policies):
        ref_p = O.softmax(logits[r])
        assert (probs[r].view(np.uint32) == ref_p.view(np.uint32)).all(), r
        g = O.Prng(seeds[r])
        draw = g.next_unit_f32()
        assert (state[r] == g.s).all(), "one generator step per token"
        assert tok[r] == O.decode_with_draw(ref_p, kind, k=k, p=p, r=draw), (r, kind, k, p)
    assert tok[0] == 3


@pytest.mark.parametrize("V", [4096, 128256])
def test_sampler_nonfinite_is_reported(V):
    logits = np.zeros((2, V), dtype=np.float32)
    logits[1, 17] = np.nan
    tok, probs, state, status = _sample(logits, [(0, None, None), (0, None, None)], [1, 2])
    assert status[0] == 0 and status[1] != 0
