"""Golden output of the CPU oracle for bench.py's OWN workload (test infrastructure).

  python tests/golden/make_llama8b_bench_golden.py [--only greedy|nucleus]   # ~30-60 min per case, 8 cores

BASELINE.json configs[1] is "Llama-3-8B-shape random-init bf16 greedy decode, batch 1, prompt
512 / gen 256"; bench.py measures it on model "llama3-8b:bench" with request 0 of
paper_2602_00182_b200.replicas (synthetic_prompt(0, 512, V), request_seed(0)). This script runs
that exact request through the oracle (oracle/oracle.cpp, the b200 accumulation profile; the
prompt is prefilled with multi-column GEMMs, bit-identical to per-token products) and records
  * the 256 greedy tokens, the out_hash (SHA-256 of the reference-layout canonical bytes:
    tokens + 256 x 128,256 f32 logits, detcore.cpp:73-84 / receipts.cpp:120) and the receipt v2
    digest;
  * SHA-256 of every step's logits row (so a mismatch names the first divergent step) and raw
    logit bits of a few steps;
and the same for a nucleus p = 0.9 request (request 1: synthetic_prompt(1, 512, V),
request_seed(1), 256 tokens) -- BASELINE.json configs[3]'s policy at the 8B shape.
tests/test_gpu_llama8b.py checks the GPU engine against this file at batch 1, inside a batch of
256 distinct requests, and across 1,000 replays; bench.py reports receipt_probe_matches_oracle.
"""
import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_2602_00182_b200 import replicas  # noqa: E402

MODEL = "llama3-8b:bench"
PROMPT, GEN = 512, 256
OUT = Path(__file__).parent / "llama8b_bench_oracle.json"


def case(m, name, idx, kind, p):
    pr = replicas.synthetic_prompt(idx, PROMPT, m.V)
    seed = replicas.request_seed(idx)
    t0 = time.time()
    toks, lg = m.generate(pr, kind=kind, p=p, max_tokens=GEN, seed=seed)
    dt = time.time() - t0
    bits = lg.view(np.uint32)
    return {"name": name, "request_index": idx, "kind": kind, "p": p, "seed": seed, "prompt_len": PROMPT,
            "max_tokens": GEN, "prompt_sha256": hashlib.sha256(pr.astype("<u4").tobytes()).hexdigest(),
            "tokens": toks.tolist(), "out_hash": O.out_hash(toks, lg).hex(),
            "out_hash_v2": O.hash_canonical_v2(toks, lg).hex(),
            "step_logits_sha256": [hashlib.sha256(lg[t].astype("<f4").tobytes()).hexdigest() for t in range(GEN)],
            "logit_bits": {str(t): [int(x) for x in bits[t, :8]] + [int(x) for x in bits[t, -8:]]
                           for t in (0, 1, 127, GEN - 1)},
            "oracle_seconds": round(dt, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["greedy", "nucleus"], default=None)
    a = ap.parse_args()
    O.lib().orc_set_threads(os.cpu_count() or 1)
    t0 = time.time()
    m = O.Llama(MODEL)
    print(f"weights {time.time() - t0:.0f} s", flush=True)
    data = json.loads(OUT.read_text()) if OUT.exists() else {"model": MODEL, "cases": []}
    have = {c["name"]: c for c in data["cases"]}
    for name, idx, kind, p in (("greedy", 0, 0, None), ("nucleus", 1, 2, 0.9)):
        if a.only and a.only != name:
            continue
        c = case(m, name, idx, kind, p)
        have[name] = c
        print(name, c["tokens"][:16], c["out_hash"], f"{c['oracle_seconds']} s", flush=True)
        data = {"model": MODEL, "generated_by": "tests/golden/make_llama8b_bench_golden.py (CPU oracle, b200 "
                                               "accumulation profile)",
                "cases": [have[k] for k in ("greedy", "nucleus") if k in have]}
        OUT.write_text(json.dumps(data, indent=1) + "\n")


if __name__ == "__main__":
    main()
