"""Where the end-to-end time of the bench's e2e leg goes (8B shape, batch-1 requests).

  python tools/e2e_breakdown.py [--n 3] [--prompt 512] [--gen 256]

Times, for the same n requests: device-only (no D2H, no hash), static groups with the v1 receipt,
continuous batching with the v1 receipt (the bench's e2e leg), and receipt v2; prints each call's
wall time and the engine's stats (prefill / decode / D2H / hash ms, bytes).
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import replicas  # noqa: E402
from paper_2602_00182_b200.detcore import DecodePolicy, Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3)
    ap.add_argument("--prompt", type=int, default=512)
    ap.add_argument("--gen", type=int, default=256)
    a = ap.parse_args()
    eng = Engine("llama3-8b:bench", "b200", max_batch=1, max_context=a.prompt + a.gen)
    prompts = [replicas.synthetic_prompt(0, a.prompt, eng.vocab)] * a.n
    pols = [DecodePolicy.greedy(a.gen)] * a.n
    seeds = [replicas.request_seed(0)] * a.n
    cases = {
        "device_only": dict(device_only=True),
        "static_v1": dict(want_logits=False, want_hash=True),
        "continuous_v1": dict(want_logits=False, want_hash=True, continuous=True),
        "continuous_v1_logits": dict(want_logits=True, want_hash=True, continuous=True),
        "static_v2": dict(want_logits=False, want_hash=True, receipt_v2=True),
    }
    eng.generate(prompts[:1], pols[:1], seeds[:1], device_only=True)   # warm-up (graphs, pools)
    for name, kw in cases.items():
        for rep in range(2):
            t0 = time.perf_counter()
            eng.generate(prompts, pols, seeds, batch_size=1, **kw)
            wall = (time.perf_counter() - t0) * 1e3
            st = eng.last_stats
            if rep:
                print(json.dumps({"case": name, "n": a.n, "wall_ms": round(wall, 1),
                                  "tok_s": round(a.n * a.gen / wall * 1e3, 1), "prefill_ms": round(st.prefill_ms, 1),
                                  "decode_ms": round(st.decode_ms, 1), "d2h_ms": round(st.d2h_ms, 1),
                                  "hash_ms": round(st.hash_ms, 1), "d2h_bytes": st.d2h_bytes}), flush=True)


if __name__ == "__main__":
    main()
