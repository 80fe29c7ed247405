"""Checker workload: small engines that drive every hand-synchronised kernel path once, checked
against the CPU oracle, then the out-of-bounds-write canaries of every engine buffer
(detgpu_debug_check_canaries). compute-sanitizer is closed on the GPU pool (it left GPUs needing a
reset); this is the substitute, run by tests/test_gpu_engine.py::test_no_out_of_bounds_writes_canaries.

  python tools/sanitize_run.py [--part all|tiny|mid|cont]

Paths covered:
  * tcgen05 GEMM, decode push-combine (st.async into the owner's receive buffer) and prefill
    DSMEM pull-combine -- every engine GEMM;
  * cluster attention (<= 8 columns) incl. the separate receive buffer (<= 2 columns) and the
    workspace + global-ticket combine (> 16 chunks: llama-mid, 1,100-token context);
  * streamed attention (> 8 columns, TMA ring, shared-memory completion counters, global tickets);
  * the 32-CTA sampler (greedy / top-k / nucleus, last-CTA fold);
  * continuous batching (admission between graph-replayed decode steps);
  * fused and unfused RMSNorm.
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2602_00182_b200.detcore import DecodePolicy, Engine  # noqa: E402


def _prompt(seed, n, V):
    g = O.Prng(seed ^ 0xABCD)
    return [g.next_below(V) for _ in range(n)]


def check(eng, orc, prompts, pols, seeds, **kw):
    toks, logits, hashes = eng.generate(prompts, pols, seeds, **kw)
    for i, (p, pol, s) in enumerate(zip(prompts, pols, seeds)):
        ot, ol = orc.generate(p, kind=int(pol.kind), k=pol.k, p=pol.p, max_tokens=pol.max_tokens, seed=s)
        assert toks[i].tolist() == ot.tolist(), f"request {i}: tokens differ from the oracle"
        assert (logits[i].view(np.uint32) == ol.view(np.uint32)).all(), f"request {i}: logits differ"
    return hashes


_KEEP = []


def close_all():
    for e in _KEEP:
        e.close()
    _KEEP.clear()


def part_tiny(keep=False):
    eng = Engine("llama-tiny:san", "b200", max_batch=16, max_context=320)
    orc = O.Llama("llama-tiny:san")
    V = eng.vocab
    # batch 1: cluster attention (sep. receive buffer), fused RMSNorm, push-combine GEMMs, sampler
    check(eng, orc, [_prompt(1, 12, V)], [DecodePolicy.greedy(3)], [1])
    # batch 2..8 fused paths with every policy
    pols = [DecodePolicy.greedy(3), DecodePolicy.top_k(40, 3), DecodePolicy.nucleus(0.9, 3)]
    check(eng, orc, [_prompt(2 + i, 5 + 9 * i, V) for i in range(3)], pols, [7, 8, 9])
    # > 8 columns: streamed attention, unfused RMSNorm; ragged contexts crossing chunk / page edges
    n = 12
    pr = [_prompt(20 + i, 3 + (i * 23) % 140, V) for i in range(n)]
    check(eng, orc, pr, [pols[i % 3] for i in range(n)], list(range(100, 100 + n)))
    _KEEP.append(eng) if keep else eng.close()


def part_cont(keep=False):
    eng = Engine("llama-tiny:san", "b200", max_batch=4, max_context=256)
    orc = O.Llama("llama-tiny:san")
    V = eng.vocab
    n = 7
    pr = [_prompt(40 + i, 4 + 17 * i, V) for i in range(n)]
    pols = [DecodePolicy.greedy(2 + (i * 3) % 5) for i in range(n)]
    check(eng, orc, pr, pols, list(range(n)), batch_size=4, continuous=True)
    _KEEP.append(eng) if keep else eng.close()


def part_mid(keep=False):
    eng = Engine("llama-mid:san", "b200", max_batch=2, max_context=1200)
    orc = O.Llama("llama-mid:san")
    V = eng.vocab
    # 1,100-token context: > 16 chunks -> workspace + ticket combine in decode attention; prefill
    # on the many-column GEMM / query-block attention paths
    check(eng, orc, [_prompt(5, 1100, V)], [DecodePolicy.greedy(2)], [3])
    _KEEP.append(eng) if keep else eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="all", choices=["all", "tiny", "mid", "cont"])
    a = ap.parse_args()
    parts = {"tiny": part_tiny, "cont": part_cont, "mid": part_mid}
    import ctypes as C

    from paper_2602_00182_b200 import _lib as L

    for name, fn in parts.items():
        if a.part in ("all", name):
            t0 = time.time()
            fn(keep=True)
            print(f"sanitize_run part {name}: ok, bytes equal the oracle ({time.time() - t0:.0f} s)", flush=True)
    n, bad = C.c_uint64(), C.c_uint64()
    L.check(L.lib.detgpu_debug_check_canaries(C.byref(n), C.byref(bad)))
    print(f"canaries: {n.value} buffers checked, {bad.value} overwritten", flush=True)
    close_all()


if __name__ == "__main__":
    main()
