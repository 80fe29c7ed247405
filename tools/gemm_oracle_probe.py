"""GPU GEMM (the engine's shape rule for S) vs the oracle's b200 profile at the 8B decode shapes, with
engine-like magnitudes (weights ~U(-1,1)*2^-6, activations ~N(0,1) bf16). Prints mismatch counts.
  python tools/gemm_oracle_probe.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import oracle as O  # noqa: E402
from paper_2602_00182_b200._lib import check, lib  # noqa: E402

O.lib().orc_set_threads(16)
g = torch.Generator().manual_seed(3)
for n_out, K in [(6144, 4096), (4096, 4096), (4096, 14336), (28672, 4096)]:
    for ncols in (1, 12):
        W = ((torch.rand(n_out, K, generator=g) * 2 - 1) * 2 ** -6).to(torch.bfloat16)
        X = torch.randn(ncols, K, generator=g).to(torch.bfloat16)
        Wd, Xd = W.cuda(), X.cuda()
        Y = torch.empty(ncols, n_out, device="cuda")
        check(lib.detgpu_k_gemm(Wd.data_ptr(), Xd.data_ptr(), Y.data_ptr(), n_out, K, ncols, n_out, None))
        torch.cuda.synchronize()
        ref = O.gemm(W.view(torch.int16).numpy().view(np.uint16), X.view(torch.int16).numpy().view(np.uint16))
        y = Y.cpu().numpy()
        bad = (y.view(np.uint32) != ref.view(np.uint32))
        d = np.abs(y - ref)
        print(f"n_out {n_out} K {K} ncols {ncols}: mismatches {int(bad.sum())} / {bad.size}, max |d| {d.max():.3e}",
              flush=True)
