"""Per-CTA timeline of one captured decode step (detgpu_set_option "trace").

  python tools/trace_step.py [batch] [ctx] [--layers N] [--json out.json]

For every kernel launch of the last traced step: first CTA start, first/last dependency release
(griddepcontrol.wait returning), last CTA end (µs from the step's first CTA), plus the
release->end span and the gap from the previous launch's end to this launch's first release
(the PDL hand-off). Timing instrumentation only.
"""
import argparse
import ctypes as C
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import _lib as L  # noqa: E402
from paper_2602_00182_b200.detcore import Engine  # noqa: E402

NAMES = {1: "qkv", 2: "attn", 3: "o", 4: "gate_up", 5: "down", 6: "lm_head"}
REC = np.dtype([("tag", "<u4"), ("sm", "<u4"), ("t", "<u8", (15,))])
END = 14
PHASES = {"gemm": ["wait", "b_setup", "mainloop", "tmem->partial", "cluster_sync1", "dsmem_ld", "epilogue",
                   "cluster_sync2", "ab:ld_ml", "ab:max_exp", "ab:Lchain", "ab:bar", "ab:round0", "exit"],
          "attn": ["wait", "kv_load", "scores", "softmax", "pv", "", "", "", "", "", "", "", "", "exit"]}

ap = argparse.ArgumentParser()
ap.add_argument("batch", nargs="?", type=int, default=1)
ap.add_argument("ctx", nargs="?", type=int, default=640)
ap.add_argument("--layers", type=int, default=3)
ap.add_argument("--l2pf", type=int, default=None)
ap.add_argument("--json", default=None)
ap.add_argument("--raw", default=None, help="save the last step's records (.npy)")
ap.add_argument("--cap", type=int, default=1 << 20, help="trace buffer capacity (records)")
a = ap.parse_args()

eng = Engine("llama3-8b:bench", "b200", max_batch=max(a.batch, 1), max_context=768)
if a.l2pf is not None:
    eng.set_option("l2pf_mask", a.l2pf)
eng.set_option("trace", a.cap)
ms = C.c_float()
L.check(L.lib.detgpu_profile_graph(eng.h, a.batch, a.ctx, 0, 1, C.byref(ms)), eng.h)   # 3 warm-up + 1
buf = np.zeros(a.cap, dtype=REC)
n = C.c_uint32()
L.check(L.lib.detgpu_trace_read(eng.h, buf.ctypes.data, len(buf), C.byref(n)), eng.h)
r = buf[: n.value]
r = r[np.argsort(r["t"][:, 0], kind="stable")]
r = r[len(r) * 3 // 4:]   # the last of the four identical steps
t_base = int(r["t"][:, 0].min())
if a.raw:
    np.save(a.raw, r)
# k-th occurrence of (class, CTA) -> launch k of that class
occ = defaultdict(int)
launch = defaultdict(list)
for x in r:
    cls, cta = int(x["tag"]) >> 24, int(x["tag"]) & 0xFFFFFF
    k = occ[(cls, cta)]
    occ[(cls, cta)] += 1
    launch[(cls, k)].append(x)
rows = []
for (cls, k), xs in launch.items():
    xs = np.array(xs, dtype=REC)
    t = xs["t"].astype(np.int64)
    rel = t[:, 1][t[:, 1] > 0]
    # phase j = mark j - the latest earlier mark (median/p90/max over CTAs), µs
    ph = []
    for j in range(1, END + 1):
        d = []
        for row in t:   # chronological: the latest other mark not after this one
            prev = [v for i2, v in enumerate(row) if i2 != j and i2 != END and 0 < v <= row[j]]
            if row[j] > 0 and prev:
                d.append(row[j] - max(prev))
        ph.append(f"{np.median(d) / 1e3:.2f}/{np.percentile(d, 90) / 1e3:.2f}/{np.max(d) / 1e3:.2f}" if d else None)
    live = t[:, 1] > 0
    rows.append({"kernel": NAMES.get(cls, str(cls)), "layer": k, "ctas": len(xs),
                 "start": (int(t[:, 0].min()) - t_base) / 1e3,
                 "release_first": (int(rel.min()) - t_base) / 1e3 if len(rel) else None,
                 "release_last": (int(rel.max()) - t_base) / 1e3 if len(rel) else None,
                 "end": (int(t[:, END].max()) - t_base) / 1e3,
                 "cta_median_us": float(np.median((t[:, END] - np.maximum(t[:, 1], t[:, 0]))[live] if live.any() else 0)) / 1e3,
                 "phases": {k: v for k, v in zip(PHASES["attn" if cls == 2 else "gemm"], ph) if k and v},
                 "sms": int(len(np.unique(xs["sm"])))})
rows.sort(key=lambda z: z["end"])
prev_end = None
for z in rows:
    z["span"] = round(z["end"] - (z["release_first"] if z["release_first"] is not None else z["start"]), 2)
    z["handoff"] = round(z["release_first"] - prev_end, 2) if (prev_end is not None and z["release_first"]) else None
    prev_end = z["end"]
step_us = rows[-1]["end"]
print(f"graph ms/step {ms.value:.4f}; traced step {step_us:.1f} us over {len(rows)} launches")
hdr = ["kernel", "layer", "ctas", "sms", "start", "release_first", "release_last", "end", "span", "handoff", "cta_median_us"]
print(" ".join(f"{h:>12}" for h in hdr))
for z in rows:
    if z["layer"] < a.layers or z["kernel"] == "lm_head":
        print(" ".join(f"{(round(z[h], 2) if isinstance(z[h], float) else z[h])!s:>12}" for h in hdr))
        print(" " * 14 + "phase us median/p90/max: " + ", ".join(f"{k}={v}" for k, v in z["phases"].items()))
agg = defaultdict(lambda: [0.0, 0.0, 0])
for z in rows:
    agg[z["kernel"]][0] += z["span"]
    agg[z["kernel"]][1] += z["handoff"] or 0.0
    agg[z["kernel"]][2] += 1
print("per class: total span us / total hand-off us / launches")
for k, v in agg.items():
    print(f"  {k:>8} {v[0]:9.1f} {v[1]:9.1f} {v[2]:4d}")
if a.json:
    Path(a.json).write_text(json.dumps({"batch": a.batch, "ctx": a.ctx, "graph_ms": ms.value, "launches": rows}, indent=1))
