import sys, torch
sys.path.insert(0, '.')
from paper_2602_00182_b200._lib import lib, check
ok = True
for n_out, K, ncols in [(256, 512, 256), (512, 4096, 200), (1024, 1024, 130), (6144, 4096, 256), (128, 14336, 512), (384, 256, 70)]:
    g = torch.Generator().manual_seed(n_out + ncols)
    W = (torch.rand(n_out, K, generator=g) * 2 - 1).mul(0.05).to(torch.bfloat16).cuda()
    X = (torch.rand(ncols, K, generator=g) * 2 - 1).to(torch.bfloat16).cuda()
    Y1 = torch.empty(ncols, n_out, device='cuda'); Y2 = torch.empty(ncols, n_out, device='cuda')
    check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y1.data_ptr(), n_out, K, ncols, n_out, 0, None))
    check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y2.data_ptr(), n_out, K, ncols, n_out, -1, None))
    torch.cuda.synchronize()
    eq = torch.equal(Y1.view(torch.int32), Y2.view(torch.int32))
    print(n_out, K, ncols, "bit-identical" if eq else "DIFFERENT", flush=True)
    ok &= eq
    # speed
    for mode in (0, -1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y1.data_ptr(), n_out, K, ncols, n_out, mode, None))
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        print("   mode", "wide" if mode else "n64", round(us, 1), "us", round(2 * n_out * K * ncols / us / 1e6, 1), "TFLOP/s")
print("ALL_EQUAL" if ok else "MISMATCH")
