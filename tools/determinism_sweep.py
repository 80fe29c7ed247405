"""Receipt determinism sweeps (BASELINE.json configs 3 and 4) on one GPU.

  python tools/determinism_sweep.py [--model llama3-8b:sweep] [--prompts 64] [--prompt-len 64] [--gen 32]
                                    [--replays 1000] [--out profiles/determinism_r1.json]

* batch sweep: the same distinct prompts (greedy and nucleus, per-request seeds) decoded at batch
  sizes 1, 8, 64, 256 (and in reversed order): every request's out_hash must be identical.
* replay: one nucleus-sampled request (p = 0.9) replayed `--replays` times as copies spread over
  batches of 250 plus sequential single replays: all out_hashes identical.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import replicas  # noqa: E402
from paper_2602_00182_b200.detcore import DecodePolicy, Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b:sweep")
    ap.add_argument("--prompts", type=int, default=64)
    ap.add_argument("--prompt-len", type=int, default=64)
    ap.add_argument("--gen", type=int, default=32)
    ap.add_argument("--replays", type=int, default=1000)
    ap.add_argument("--singles", type=int, default=16)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    eng = Engine(a.model, "b200", max_batch=256, max_context=a.prompt_len + a.gen + 1)
    V = eng.vocab
    prompts = [replicas.synthetic_prompt(i, a.prompt_len, V) for i in range(a.prompts)]
    pols = [DecodePolicy.greedy(a.gen) if i % 2 == 0 else DecodePolicy.nucleus(0.9, a.gen) for i in range(a.prompts)]
    seeds = [replicas.request_seed(i) for i in range(a.prompts)]
    res = {"model": a.model, "prompts": a.prompts, "prompt_len": a.prompt_len, "gen": a.gen}
    t0 = time.time()
    ref = None
    sweep = {}
    for bs in (256, 64, 8, 1):
        n = a.prompts if bs > 1 else min(a.singles, a.prompts)
        _, _, h = eng.generate(prompts[:n], pols[:n], seeds[:n], batch_size=bs, want_logits=False)
        if ref is None:
            ref = h
        sweep[bs] = sum(x == y for x, y in zip(h, ref[:n])) / n
    rev = list(range(a.prompts))[::-1]
    _, _, hr = eng.generate([prompts[i] for i in rev], [pols[i] for i in rev], [seeds[i] for i in rev], batch_size=64,
                            want_logits=False)
    sweep["reversed_64"] = sum(hr[rev.index(i)] == ref[i] for i in range(a.prompts)) / a.prompts
    res["batch_sweep_match_rate"] = sweep
    # replay: copies of one nucleus request
    p0, pol0, s0 = prompts[1], DecodePolicy.nucleus(0.9, a.gen), seeds[1]
    _, _, hrep = eng.generate([p0] * a.replays, [pol0] * a.replays, [s0] * a.replays, batch_size=250, want_logits=False)
    singles = [eng.generate([p0], [pol0], [s0], batch_size=1, want_logits=False)[2][0] for _ in range(a.singles)]
    allh = hrep + singles
    res["replays"] = len(allh)
    res["replay_match_rate"] = sum(h == allh[0] for h in allh) / len(allh)
    res["replay_equals_sweep"] = allh[0] == ref[1]
    res["distinct_tokens_example"] = int(len(set(eng.generate([p0], [pol0], [s0])[0][0].tolist())))
    res["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(res))
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
