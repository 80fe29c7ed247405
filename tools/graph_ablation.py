"""Decode-step graph ablation (timing only): which kernel classes cost what inside the PDL pipeline."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import _lib as L  # noqa: E402
from paper_2602_00182_b200.detcore import Engine  # noqa: E402

QKV, ATTN, O, GU, DOWN = 1, 2, 3, 4, 5
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1
eng = Engine("llama3-8b:bench", "b200", max_batch=max(batch, 1), max_context=768)
cases = {"full": 0, "no_norm": 1, "no_attn": 1 << ATTN, "no_qkv": 1 << QKV, "no_o": 1 << O, "no_gate_up": 1 << GU,
         "no_down": 1 << DOWN, "only_gemm_gu_down": (1 << ATTN) | (1 << QKV) | (1 << O),
         "only_attn": (1 << QKV) | (1 << O) | (1 << GU) | (1 << DOWN), "nothing": (1 << ATTN) | (1 << QKV) | (1 << O) | (1 << GU) | (1 << DOWN)}
out = {}
for name, mask in cases.items():
    ms = C.c_float()
    L.check(L.lib.detgpu_profile_graph(eng.h, batch, 640, mask, 20, C.byref(ms)), eng.h)
    out[name] = round(ms.value, 4)
print(json.dumps({"batch": batch, "ms_per_step": out}))
