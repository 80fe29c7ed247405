"""Scan the fixed K-segment count S for the 8B decode GEMM shapes (speed only; S changes numerics)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200._lib import check, lib  # noqa: E402

SHAPES = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (128256, 4096)]


def timeit(W, X, Y, n_out, K, ncols, S, n=20):
    for _ in range(3):
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, S, None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, S, None))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n


for n_out, K in SHAPES:
    W = torch.randn(n_out, K, device="cuda").mul(0.01).to(torch.bfloat16)
    X = torch.randn(256, K, device="cuda").to(torch.bfloat16)
    Y = torch.empty(256, n_out, device="cuda")
    for ncols in (1, 64):
        res = {}
        for S in (1, 2, 3, 4, 5, 6, 7, 8):
            if S > K // 64 or (n_out // 128) * S > 2400:
                continue
            res[S] = round(timeit(W, X, Y, n_out, K, ncols, S), 2)
        print(json.dumps({"n_out": n_out, "K": K, "ncols": ncols, "us_by_S": res,
                          "GBs_best": round(n_out * K * 2 / min(res.values()) / 1e3, 1)}), flush=True)
