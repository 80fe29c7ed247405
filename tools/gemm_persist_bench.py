"""A/B: many-column GEMM, one-unit-per-cluster (gemm_tc_kernel) vs persistent (gemm_persist_kernel).
  python tools/gemm_persist_bench.py
Prints one JSON line per (shape, columns): us per launch and TFLOP/s of both forms."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200._lib import check, lib  # noqa: E402

SHAPES = [(6144, 4096, "qkv"), (4096, 4096, "o"), (28672, 4096, "gate_up"), (4096, 14336, "down")]


def run(W, X, Y, n_out, K, ncols, code, n=20):
    for _ in range(3):
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, code, None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, code, None))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n


for n_out, K, name in SHAPES:
    W = torch.randn(n_out, K, device="cuda").mul(0.01).to(torch.bfloat16)
    for ncols in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["128", "256", "512"])]:
        X = torch.randn(ncols, K, device="cuda").to(torch.bfloat16)
        Y = torch.empty(ncols, n_out, device="cuda")
        a = run(W, X, Y, n_out, K, ncols, 0)
        b = run(W, X, Y, n_out, K, ncols, 300)
        fl = 2.0 * n_out * K * ncols
        print(json.dumps({"gemm": name, "ncols": ncols, "us_cluster": round(a, 2), "us_persist": round(b, 2),
                          "TFs_cluster": round(fl / a / 1e6, 1), "TFs_persist": round(fl / b / 1e6, 1)}), flush=True)
