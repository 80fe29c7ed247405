python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
python tools/trace_step.py 1 640 --layers 1 2>&1 | head -16
python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2602_00182_b200 import _lib as L
from paper_2602_00182_b200.detcore import Engine
for b in (1, 8, 64):
    eng = Engine("llama3-8b:bench", "b200", max_batch=max(b, 1), max_context=768)
    for fuse in (0, 1):
        eng.set_option("attn_fuse", fuse)
        ms = C.c_float()
        L.check(L.lib.detgpu_profile_graph(eng.h, b, 640, 0, 30, C.byref(ms)), eng.h)
        print("batch", b, "attn_fuse", fuse, "ms", round(ms.value, 4), flush=True)
    eng.close()
PY
