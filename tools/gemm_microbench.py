"""Time the tcgen05 GEMM (detgpu_k_gemm, row-major weights) over decode shapes with CUDA events.

  python tools/gemm_microbench.py
Prints one JSON line per shape: n_out, K, ncols, ksplit, us per launch, weight GB/s.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200._lib import check, lib  # noqa: E402

SHAPES = [
    (6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (128256, 4096),   # 8B decode GEMMs
    (18944, 256), (18944, 1024), (18944, 4096),                                  # 148 tiles, S=1
    (4096, 1024), (128 * 37, 4096), (128 * 74, 4096),
]


def ksplit(n_out, k):
    tiles, nkb = n_out // 128, k // 64
    s = max(1, min(8, 148 // max(tiles, 1)))
    return min(s, nkb)


def main():
    ncols_list = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "64"])]
    for n_out, K in SHAPES:
        W = torch.randn(n_out, K, device="cuda").mul(0.01).to(torch.bfloat16)
        for ncols in ncols_list:
            X = torch.randn(max(ncols, 64), K, device="cuda").to(torch.bfloat16)
            Y = torch.empty(max(ncols, 64), n_out, device="cuda")
            for _ in range(3):
                check(lib.detgpu_k_gemm(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, None))
            torch.cuda.synchronize()
            n = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                check(lib.detgpu_k_gemm(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, None))
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1000 / n
            print(json.dumps({"n_out": n_out, "K": K, "ncols": ncols, "ksplit": ksplit(n_out, K),
                              "us": round(us, 2), "weight_GBs": round(n_out * K * 2 / us / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
