"""One un-graphed decode step of the 8B-shape engine (for ncu). Prints per-class event timings.

  python tools/profile_step.py [--model llama3-8b:bench] [--batch 1] [--ctx 640] [--reps 1]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2602_00182_b200 import _lib as L  # noqa: E402
from paper_2602_00182_b200.detcore import Engine  # noqa: E402

NAMES = ["norm", "qkv_gemm", "attention", "o_gemm", "gate_up_gemm", "down_gemm", "lm_head_gemm", "sample"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b:bench")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ctx", type=int, default=640)
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    eng = Engine(a.model, "b200", max_batch=a.batch, max_context=max(a.ctx, 768))
    ms = (C.c_float * 8)()
    cnt = (C.c_uint32 * 8)()
    L.check(L.lib.detgpu_profile_decode_step(eng.h, a.batch, a.ctx, a.reps, ms, cnt), eng.h)
    print(json.dumps({"batch": a.batch, "ctx": a.ctx, "ms": {NAMES[i]: ms[i] for i in range(8)},
                      "launches": {NAMES[i]: cnt[i] for i in range(8)}}))


if __name__ == "__main__":
    main()
