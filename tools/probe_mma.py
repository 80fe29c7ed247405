"""Probe the tcgen05 kind::f16 (bf16 x bf16 -> f32) accumulation semantics through detgpu_k_gemm.

Generates crafted W/X with a fixed seed, runs the engine's GEMM, saves inputs and outputs to
gpurun_out/mma_probe.npz for offline model fitting (tools/fit_mma.py)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200._lib import check, lib  # noqa: E402


def bf16_bits(rng, shape, emin, emax, zero_frac=0.0):
    sign = rng.integers(0, 2, shape).astype(np.uint32) << 31
    exp = (rng.integers(emin, emax + 1, shape) + 127).astype(np.uint32) << 23
    man = rng.integers(0, 128, shape).astype(np.uint32) << 16
    f = (sign | exp | man).view(np.float32)
    if zero_frac > 0:
        f[rng.random(shape) < zero_frac] = 0.0
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def run(W16, X16):
    n_out, K = W16.shape
    ncols = X16.shape[0]
    Wt = torch.from_numpy(W16.view(np.int16).copy()).view(torch.bfloat16).cuda()
    Xt = torch.from_numpy(X16.view(np.int16).copy()).view(torch.bfloat16).cuda()
    Y = torch.zeros((ncols, n_out), dtype=torch.float32, device="cuda")
    check(lib.detgpu_k_gemm(Wt.data_ptr(), Xt.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, None))
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def main():
    rng = np.random.default_rng(20261018)
    out = {}
    cases = {
        # name: (n_out, K, ncols, active_K, emin, emax, xones)
        "k16_spread": (256, 64, 128, 16, -24, 24, False),
        "k16_narrow": (256, 64, 128, 16, -3, 3, False),
        "k16_ones": (256, 64, 128, 16, -24, 24, True),
        "k8_spread": (256, 64, 128, 8, -24, 24, False),
        "k32_spread": (256, 64, 128, 32, -24, 24, False),
        "k64_spread": (256, 64, 128, 64, -24, 24, False),
        "k64_narrow": (256, 64, 128, 64, -4, 4, False),
        "k256_spread": (128, 256, 128, 256, -16, 16, False),
        "k4096_normal": (128, 4096, 64, 4096, -6, 2, False),
    }
    for name, (n_out, K, ncols, act, emin, emax, xones) in cases.items():
        W = bf16_bits(rng, (n_out, K), emin, emax)
        X = bf16_bits(rng, (ncols, K), emin, emax)
        W[:, act:] = 0
        X[:, act:] = 0
        if xones:
            X[:, :act] = 0x3F80
        Y = run(W, X)
        out[name + "_W"], out[name + "_X"], out[name + "_Y"] = W, X, Y
        print(name, Y.shape, float(np.abs(Y).max()))
    Path("gpurun_out").mkdir(exist_ok=True)
    np.savez_compressed("gpurun_out/mma_probe.npz", **out)


if __name__ == "__main__":
    main()
