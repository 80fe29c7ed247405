"""Time the tcgen05 GEMM at the 8B prefill shapes (wide-N MMA form, K-split rule of the engine).

  python tools/gemm_prefill_bench.py [ncols,...]
One JSON line per (shape, ncols): us per launch, TFLOP/s, fraction of MEASURED_PEAKS bf16.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200._lib import check, lib  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def main():
    ncols_list = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["128", "512", "2048"])]
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    for name, (n_out, K) in SHAPES.items():
        W = torch.randn(n_out, K, device="cuda").mul(0.01).to(torch.bfloat16)
        for ncols in ncols_list:
            X = torch.randn(ncols, K, device="cuda").to(torch.bfloat16)
            Y = torch.empty(ncols, n_out, device="cuda")
            for _ in range(3):
                check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, -1,
                                              None))
            torch.cuda.synchronize()
            n = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                check(lib.detgpu_k_gemm_split(W.data_ptr(), X.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, -1,
                                              None))
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1000 / n
            tf = 2.0 * n_out * K * ncols / (us * 1e-6) / 1e12
            print(json.dumps({"gemm": name, "n_out": n_out, "K": K, "ncols": ncols, "us": round(us, 2),
                              "tflops": round(tf, 1), "frac_bf16_peak": round(tf / peaks["bf16_tflops"], 3)}))


if __name__ == "__main__":
    main()
