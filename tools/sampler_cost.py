"""Decode-step cost of the sampling policies at the 8B shape (nucleus cost):
greedy vs top-k 50 vs nucleus p=0.9, batch 1 / 64 / 256, prompt 128, 64 generated tokens.
  python tools/sampler_cost.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import replicas  # noqa: E402
from paper_2602_00182_b200.detcore import DecodePolicy, Engine  # noqa: E402

eng = Engine("llama3-8b:bench", "b200", max_batch=256, max_context=256)
V = eng.vocab
for b in (1, 64, 256):
    prompts = [replicas.synthetic_prompt(i, 128, V) for i in range(b)]
    seeds = [replicas.request_seed(i) for i in range(b)]
    r = {"batch": b}
    for name, pol in (("greedy", DecodePolicy.greedy(64)), ("top_k50", DecodePolicy.top_k(50, 64)),
                      ("nucleus0.9", DecodePolicy.nucleus(0.9, 64))):
        eng.generate(prompts, [pol] * b, seeds, batch_size=b, device_only=True)
        eng.generate(prompts, [pol] * b, seeds, batch_size=b, device_only=True)
        st = eng.last_stats
        r[name + "_ms_per_step"] = round(st.decode_ms / max(1, st.decode_steps), 3)
    print(json.dumps(r), flush=True)
