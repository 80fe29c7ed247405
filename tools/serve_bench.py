"""Continuous vs static batching on a mixed-length request set (8B shape, receipts on).

  python tools/serve_bench.py [--requests 32] [--slots 8] [--prompt 128]
Generated tokens per second of the whole set, and whether every out_hash matches between modes.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import replicas  # noqa: E402
from paper_2602_00182_b200.detcore import DecodePolicy, Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--requests", type=int, default=32)
ap.add_argument("--slots", type=int, default=8)
ap.add_argument("--prompt", type=int, default=128)
ap.add_argument("--v2", action="store_true")
a = ap.parse_args()
eng = Engine("llama3-8b:serve", "b200", max_batch=a.slots, max_context=a.prompt + 257)
V = eng.vocab
prompts = [replicas.synthetic_prompt(i, a.prompt, V) for i in range(a.requests)]
gens = [16 + (i * 97) % 241 for i in range(a.requests)]   # 16 .. 256, mixed
pols = [DecodePolicy.greedy(g) if i % 2 else DecodePolicy.nucleus(0.9, g) for i, g in enumerate(gens)]
seeds = [replicas.request_seed(i) for i in range(a.requests)]
res = {"requests": a.requests, "slots": a.slots, "tokens": sum(gens), "receipt": "v2" if a.v2 else "v1"}
hashes = {}
for mode in ("static", "continuous", "static", "continuous"):
    t0 = time.perf_counter()
    _, _, h = eng.generate(prompts, pols, seeds, batch_size=a.slots, want_logits=False, receipt_v2=a.v2,
                           continuous=mode == "continuous")
    dt = time.perf_counter() - t0
    res[f"{mode}_tok_s"] = round(sum(gens) / dt, 1)
    hashes.setdefault(mode, h)
res["receipts_equal"] = hashes["static"] == hashes["continuous"]
print(json.dumps(res))
