"""Decode-step graph time vs scheduling options (detgpu_set_option: l2pf_*, self_pf_kb, max_nsub).

  python tools/l2pf_scan.py [batch] [ctx] [--cases JSON]
Each case is a dict of options; unspecified options are reset to their defaults first.
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import _lib as L  # noqa: E402
from paper_2602_00182_b200.detcore import Engine  # noqa: E402

DEFAULTS = {"l2pf_mask": 2, "l2pf_cap_mb": 16, "self_pf_kb": 4, "attn_cluster_max_cols": 8, "max_nsub": 0,
            "attn_stream_min_cols": 8, "fuse_max_cols": 8, "attn_sep_recv_max_cols": 2, "self_pf_kb_qkv": -1,
            "self_pf_kb_o": 0,
            "self_pf_kb_gate_up": -1, "self_pf_kb_down": 0, "self_pf_kb_lm_head": -1,
            "gemm_pair": 0, "gemm_persist": 0, "attn_stream_prefill": 1}   # engine defaults
ap = argparse.ArgumentParser()
ap.add_argument("batch", nargs="?", type=int, default=1)
ap.add_argument("ctx", nargs="?", type=int, default=640)
ap.add_argument("--cases", default=None)
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
cases = json.loads(a.cases) if a.cases else [
    {}, {"self_pf_kb": 0, "l2pf_mask": 0}, {"self_pf_kb": 4}, {"self_pf_kb": 16}, {"l2pf_mask": 0},
    {"l2pf_cap_mb": 32}, {}]
eng = Engine("llama3-8b:bench", "b200", max_batch=max(a.batch, 1), max_context=768)
for case in cases:
    opts = dict(DEFAULTS, **case)
    for k, v in opts.items():
        try:
            eng.set_option(k, v)
        except ValueError:   # an older library without this option (A/B runs via DETGPU_LIB)
            if k in case:
                raise
    ms = C.c_float()
    L.check(L.lib.detgpu_profile_graph(eng.h, a.batch, a.ctx, 0, a.reps, C.byref(ms)), eng.h)
    print(json.dumps({"batch": a.batch, "case": case, "ms": round(ms.value, 4)}), flush=True)
