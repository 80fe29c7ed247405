"""Prefill timing at 8B shape: one request (or a batch) of `--prompt` tokens, max_tokens 1."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import replicas  # noqa: E402
from paper_2602_00182_b200.detcore import DecodePolicy, Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prompt", type=int, default=512)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--opt", action="append", default=[], help="engine option name=value (detgpu_set_option)")
a = ap.parse_args()
eng = Engine("llama3-8b:bench", "b200", max_batch=max(a.batch, 1), max_context=a.prompt + 2)
for o in a.opt:
    k, v = o.split("=")
    eng.set_option(k, int(v))
prompts = [replicas.synthetic_prompt(i, a.prompt, eng.vocab) for i in range(a.batch)]
res = []
for r in range(a.reps + 1):
    eng.generate(prompts, [DecodePolicy.greedy(1)] * a.batch, [1] * a.batch, device_only=True)
    if r:
        res.append(eng.last_stats.prefill_ms)
toks = a.prompt * a.batch
print(json.dumps({"opts": a.opt, "prompt": a.prompt, "batch": a.batch, "prefill_ms": res,
                  "prefill_tok_s": toks / (min(res) / 1000), "tflops": 2 * 8.03e9 * toks / (min(res) / 1000) / 1e12}))
