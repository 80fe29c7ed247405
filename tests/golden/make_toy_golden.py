"""Generate tests/golden/toy_reference.json from the REFERENCE ITSELF.

Runs the unmodified reference detcore (proj/src/detcore.cpp, bytes.cpp, codec.cpp compiled from
/root/reference by `make -C oracle ref` into oracle/_ref/libref.so) on:
  * the SURVEY.md §8(c) cases (model-a, container-a, drv-1, prompt 1 5 9 13 2, seed 42),
  * the test_receipts.cpp:21-30 fixture,
  * 48 randomized tuples in the style of test_detcore.cpp:21-34 (sample_exec),
and records tokens, logits (f32 bits), canonical length, out_hash and req_hash. Run here (it needs
/root/reference); the JSON is committed and travels to the GPU box.
"""
from __future__ import annotations

import hashlib
import json
import struct
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402


def run(model_id, digest, arch, driver, kind, k, p, max_tokens, seed, prompt):
    R = O.ref()
    pr = np.ascontiguousarray(prompt, dtype=np.uint32)
    toks = np.zeros(max(max_tokens, 1), dtype=np.uint32)
    logits = np.zeros((max(max_tokens, 1), 32), dtype=np.float32)
    clen = np.zeros(1, dtype=np.uint64)
    oh = np.zeros(32, dtype=np.uint8)
    rh = np.zeros(32, dtype=np.uint8)
    dg = np.frombuffer(digest, dtype=np.uint8).copy()
    rc = R.ref_infer(model_id.encode(), dg.ctypes.data, arch.encode(), driver.encode(), kind, k is not None, k or 0,
                     p is not None, 0.0 if p is None else p, max_tokens, seed, pr.ctypes.data if pr.size else None,
                     pr.size, toks.ctypes.data, clen.ctypes.data, oh.ctypes.data, rh.ctypes.data, logits.ctypes.data)
    case = dict(model_id=model_id, digest=digest.hex(), arch=arch, driver=driver, kind=kind, k=k, p=p,
                max_tokens=max_tokens, seed=seed, prompt=[int(x) for x in prompt], rc=int(rc))
    if rc == 0:
        case.update(tokens=[int(x) for x in toks[:max_tokens]], canonical_len=int(clen[0]), out_hash=oh.tobytes().hex(),
                    req_hash=rh.tobytes().hex(),
                    logits_bits=[[int(b) for b in row.view(np.uint32)] for row in logits[:max_tokens]])
    return case


def main():
    cases = []
    digest_a = hashlib.sha256(b"container-a").digest()
    base = dict(model_id="model-a", digest=digest_a, driver="drv-1", seed=42, prompt=[1, 5, 9, 13, 2])
    for arch, kind, k, p, T in [("archA", 1, 4, None, 4), ("archA", 0, None, None, 64), ("archB", 0, None, None, 64),
                                ("archA", 2, None, 0.9, 64), ("archA", 1, 4, None, 64), ("archB", 2, None, 0.5, 32),
                                ("archB", 1, 7, None, 16), ("archA", 0, None, None, 0), ("archA", 2, None, 1.0, 8)]:
        cases.append(run(base["model_id"], digest_a, arch, "drv-1", kind, k, p, T, 42, base["prompt"]))
    cases.append(run("model-a", digest_a, "archA", "drv-1", 0, None, None, 64, 1, base["prompt"]))
    cases.append(run("model-a", digest_a, "archZ", "drv-1", 0, None, None, 4, 1, base["prompt"]))  # rc=1
    cases.append(run("model-a", digest_a, "archA", "drv-1", 0, None, None, 4, 1, [1, 40]))  # OOV, rc=1
    # randomized tuples, test_detcore.cpp:21-34 style
    rng = O.Prng(2024)
    digest_c = hashlib.sha256(b"container").digest()
    for trial in range(48):
        seed = rng.next_u64()
        plen = 2 + rng.next_below(8)
        T = 1 + rng.next_below(24)
        pr = O.Prng(seed ^ 0xABCD)
        prompt = [pr.next_below(32) for _ in range(plen)]
        kind = trial % 3
        k = [None, 1 + trial % 6, None][kind]
        p = [None, None, [0.3, 0.5, 0.9, 1.0][trial % 4]][kind]
        cases.append(run(f"model-{seed % 5}", digest_c, "archA" if trial % 2 == 0 else "archB", "drv-1", kind, k, p,
                         T, seed, prompt))
    out = ROOT / "tests" / "golden" / "toy_reference.json"
    out.write_text(json.dumps({"generator": "tests/golden/make_toy_golden.py",
                               "reference": "proj/src/detcore.cpp infer() + codec.cpp encode_execution_tuple",
                               "cases": cases}, indent=0))
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    main()
