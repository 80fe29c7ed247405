"""Golden output of the CPU oracle at the Llama-3-8B shape (test infrastructure).

  python tests/golden/make_llama8b_golden.py     # ~10 min on 8 host cores

Runs the oracle (oracle/oracle.cpp, the b200 accumulation profile) on 8B-shape requests —
model "llama3-8b:golden", a 12-token synthetic prompt with greedy and nucleus (p = 0.9) decodes of 4
tokens, and a 70-token prompt (two 64-position attention chunks) with a greedy decode of 2 tokens —
and writes the tokens, the out_hash (SHA-256 of the reference-layout canonical bytes, tokens and f32
logits) and a few raw logit bits to llama8b_oracle.json. tests/test_gpu_engine.py checks the
GPU engine against it, so the 8B path is pinned to the oracle bit for bit without running the
oracle on the GPU box.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_2602_00182_b200 import replicas  # noqa: E402

MODEL = "llama3-8b:golden"


def main():
    import os

    O.lib().orc_set_threads(os.cpu_count() or 1)
    t0 = time.time()
    m = O.Llama(MODEL)
    prompt = replicas.synthetic_prompt(0, 12, m.V)
    cases = []
    for kind, p, seed, plen, T in ((0, None, 1, 12, 4), (2, 0.9, replicas.request_seed(0), 12, 4), (0, None, 5, 70, 2)):
        pr = replicas.synthetic_prompt(0 if plen == 12 else 1, plen, m.V)
        toks, logits = m.generate(pr, kind=kind, p=p, max_tokens=T, seed=seed)
        cases.append({"kind": kind, "p": p, "seed": seed, "max_tokens": T, "prompt": pr.tolist(), "tokens": toks.tolist(),
                      "out_hash": O.out_hash(toks, logits).hex(),
                      "logit_bits_step0_first8": [int(x) for x in logits[0, :8].view(np.uint32)],
                      "logit_bits_last_step_last8": [int(x) for x in logits[T - 1, -8:].view(np.uint32)]})
        print(cases[-1]["tokens"], cases[-1]["out_hash"], f"{time.time() - t0:.0f} s", flush=True)
    out = {"model": MODEL, "prompt": prompt.tolist(), "cases": cases,
           "generated_by": "tests/golden/make_llama8b_golden.py (CPU oracle, b200 accumulation profile)"}
    (Path(__file__).parent / "llama8b_oracle.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
