"""Per-CTA timeline of a captured decode-step graph (measurement only; never changes a bit).

The engine's kernels record, per CTA, globaltimer stamps of start, dependency release
(griddepcontrol.wait returning) and end when the "trace" option is on (detgpu_set_option,
detgpu_trace_read). From one traced CUDA-graph step this module derives each launch's
span INSIDE the PDL pipeline: first dependency release of any CTA -> last CTA end. That is the
time the launch occupies the step as it is really run (bench.py's roofline uses it next to the
un-graphed per-launch CUDA-event time).
"""
from __future__ import annotations

import ctypes as C
from collections import defaultdict

import numpy as np

from . import _lib as L

CLASS = {1: "qkv_gemm", 2: "attention", 3: "o_gemm", 4: "gate_up_gemm", 5: "down_gemm", 6: "lm_head_gemm"}
REC = np.dtype([("tag", "<u4"), ("sm", "<u4"), ("t", "<u8", (15,))])
END = 14


def read_launches(records: np.ndarray, steps: int):
    """Group the last of `steps` identical traced steps into launches: list of dicts with
    kernel class, occurrence index, CTA count, start / first release / end (ns, absolute)."""
    r = records[np.argsort(records["t"][:, 0], kind="stable")]
    r = r[len(r) * (steps - 1) // steps:]
    occ = defaultdict(int)
    groups = defaultdict(list)
    for x in r:
        cls, cta = int(x["tag"]) >> 24, int(x["tag"]) & 0xFFFFFF
        k = occ[(cls, cta)]
        occ[(cls, cta)] += 1
        groups[(cls, k)].append(x)
    out = []
    for (cls, k), xs in groups.items():
        t = np.array([x["t"] for x in xs], dtype=np.int64)
        rel = t[:, 1][t[:, 1] > 0]
        out.append({"kernel": CLASS.get(cls, str(cls)), "index": k, "ctas": len(xs), "start": int(t[:, 0].min()),
                    "release": int(rel.min()) if len(rel) else int(t[:, 0].min()), "end": int(t[:, END].max())})
    out.sort(key=lambda z: z["end"])
    return out


def graph_step_spans(eng, batch: int, ctx: int, cap: int = 1 << 20):
    """Trace one CUDA-graph decode step (batch columns at context ctx) of `eng` and return
    ({class: [span_us of each launch]}, graph ms/step, traced step us). Turns tracing off after."""
    eng.set_option("trace", cap)
    try:
        ms = C.c_float()
        L.check(L.lib.detgpu_profile_graph(eng.h, batch, ctx, 0, 1, C.byref(ms)), eng.h)   # 3 warm-up + 1 step
        buf = np.zeros(cap, dtype=REC)
        n = C.c_uint32()
        L.check(L.lib.detgpu_trace_read(eng.h, buf.ctypes.data, len(buf), C.byref(n)), eng.h)
    finally:
        eng.set_option("trace", 0)
    launches = read_launches(buf[: n.value], 4)
    spans = defaultdict(list)
    for z in launches:
        spans[z["kernel"]].append((z["end"] - z["release"]) / 1e3)
    t0 = min(z["start"] for z in launches)
    return dict(spans), float(ms.value), (max(z["end"] for z in launches) - t0) / 1e3
