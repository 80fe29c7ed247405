"""Decode-step graph time vs the L2 weight-warming schedule (detgpu_set_option l2pf_*).

  python tools/l2pf_scan.py [batch] [ctx]
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import _lib as L  # noqa: E402
from paper_2602_00182_b200.detcore import Engine  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 640
eng = Engine("llama3-8b:bench", "b200", max_batch=max(batch, 1), max_context=768)
cases = [(0, 64), (1, 64), (16, 64), (2, 16), (2, 32), (2, 64), (4, 16), (4, 32), (8, 16), (8, 64), (1 | 2, 32),
         (1 | 2 | 4 | 8, 16), (1 | 2 | 4 | 8, 32), (1 | 2 | 8, 32), (1 | 8, 64), (0, 64)]
out = []
for mask, cap in cases:
    eng.set_option("l2pf_mask", mask)
    eng.set_option("l2pf_cap_mb", cap)
    ms = C.c_float()
    L.check(L.lib.detgpu_profile_graph(eng.h, batch, ctx, 0, 30, C.byref(ms)), eng.h)
    out.append({"mask": mask, "cap_mb": cap, "ms": round(ms.value, 4)})
    print(json.dumps(out[-1]), flush=True)
