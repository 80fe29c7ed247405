"""Stress: repeated CUDA-graph decode steps at batch 1/8/64/256 (the bench's decode_batch_sweep)
on one engine; prints the batch at which a launch error first appears. Diagnostic only.

  python tools/stress_sweep.py [iters] [--opt name=value ...]
"""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_00182_b200 import _lib as L  # noqa: E402
from paper_2602_00182_b200.detcore import Engine  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
opts = [a.split("=") for a in sys.argv[2:] if "=" in a]
batches = [int(x) for x in next((a[2:] for a in sys.argv if a.startswith("b=")), "1,8,64,256").split(",")]
eng = Engine("llama3-8b:bench", "b200", max_batch=256, max_context=768)
for k, v in opts:
    if k != "b":
        eng.set_option(k, int(v))
t0 = time.time()
for it in range(iters):
    for b in batches:
        ms = C.c_float()
        rc = L.lib.detgpu_profile_graph(eng.h, b, 640, 0, 10, C.byref(ms))
        if rc != 0:
            print(f"FAIL iter {it} batch {b}: {L.lib.detgpu_last_error(eng.h).decode()}", flush=True)
            sys.exit(3)
print(f"ok {iters} iters {time.time() - t0:.1f} s", flush=True)
