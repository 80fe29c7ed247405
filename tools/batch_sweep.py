"""Decode-step time and HBM roofline fraction vs batch size at the 8B shape (one GPU).

  python tools/batch_sweep.py [--batches 1,8,32,64,128,256] [--ctx 640] [--reps 20] [--out F]

Per batch: the CUDA-graph decode step time (detgpu_profile_graph, every column at context `ctx`),
the step's algorithmic bytes (weights once + per column KV read/write, embedding
row, f32 logits write) and the per-class times of one un-graphed step (detgpu_profile_decode_step),
with the attention class's achieved KV-read bandwidth (32 layers x ctx x 4 KiB per column).
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
PEAK = 6551.4   # MEASURED_PEAKS.json HBM GB/s


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b:bench")
    ap.add_argument("--batches", default="1,8,32,64,128,256")
    ap.add_argument("--ctx", type=int, default=640)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    bs = [int(x) for x in a.batches.split(",")]
    eng = Engine(a.model, "b200", max_batch=max(bs), max_context=max(a.ctx + 1, 768))
    info = eng.info
    d, Lr, hq, hkv, hd, F, V = (info.d_model, info.n_layers, info.n_heads, info.n_kv_heads, info.head_dim, info.ffn,
                                info.vocab)
    weights = 2.0 * (Lr * (d * (hq + 2 * hkv) * hd + hq * hd * d + 3 * d * F + 2 * d) + d + V * d)
    kv_pos = Lr * 2 * hkv * hd * 2
    rows = []
    for b in bs:
        ms = C.c_float()
        L.check(L.lib.detgpu_profile_graph(eng.h, b, a.ctx, 0, a.reps, C.byref(ms)), eng.h)
        cms = (C.c_float * 8)()
        cnt = (C.c_uint32 * 8)()
        L.check(L.lib.detgpu_profile_decode_step(eng.h, b, a.ctx, 3, cms, cnt), eng.h)
        step_b = weights + b * (kv_pos * a.ctx + kv_pos + 2 * d + 4 * V)
        attn_b = b * kv_pos * a.ctx
        cls = {NAMES[k]: round(float(cms[k]), 4) for k in range(8)}
        row = {"batch": b, "ctx": a.ctx, "graph_step_ms": round(ms.value, 4), "tok_s": round(b / ms.value * 1e3, 1),
               "step_GB": round(step_b / 1e9, 3), "step_frac": round(step_b / (ms.value / 1e3) / 1e9 / PEAK, 4),
               "attention_GBs": round(attn_b / (cls["attention"] / 1e3) / 1e9, 1) if cls["attention"] > 0 else None,
               "per_class_ms": cls}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1) + "\n")


if __name__ == "__main__":
    main()
