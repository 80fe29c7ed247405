"""A/B of the persistent many-column GEMM inside the engine (detgpu_set_option "gemm_persist"):
decode-step graph time at batch 64/128/256 (context 640) and the 512-token prefill.
  python tools/persist_ab.py"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import _lib as L, replicas  # noqa: E402
from paper_2602_00182_b200.detcore import DecodePolicy, Engine  # noqa: E402

eng = Engine("llama3-8b:bench", "b200", max_batch=256, max_context=768)
pr = [replicas.synthetic_prompt(0, 512, eng.vocab)]
out = {}
for mode in (0, 1, 2):
    eng.set_option("gemm_persist", mode)
    r = {}
    for b in (64, 128, 256):
        ms = C.c_float()
        L.check(L.lib.detgpu_profile_graph(eng.h, b, 640, 0, 10, C.byref(ms)), eng.h)
        r[f"b{b}_ms"] = round(ms.value, 3)
    pf = []
    hs = set()
    for _ in range(4):
        _, _, h = eng.generate(pr, [DecodePolicy.greedy(2)], [1], want_logits=False)
        pf.append(eng.last_stats.prefill_ms)
        hs.add(h[0])
    r["prefill512_ms"] = round(min(pf[1:]), 3)
    r["hash"] = next(iter(hs)).hex()[:16] if len(hs) == 1 else "MISMATCH"
    out[f"persist{mode}"] = r
    print(json.dumps({f"persist{mode}": r}), flush=True)
