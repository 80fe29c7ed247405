"""Golden vectors for receipt v2 from the REFERENCE's own DA Merkle code (proj/src/da.cpp
leaf_hash / merkle_root, compiled from /root/reference by `make -C oracle ref`).

  python tests/golden/make_receipt_v2_golden.py   ->  tests/golden/receipt_v2.json

Logits are generated from a splitmix64 counter (exactly reproducible, finite f32 in +-[1, 2));
per step: the 4 KiB leaves are hashed with ref_leaf_hash and folded with ref_merkle_root. The v2
envelope (tag, T, tokens, (V, root) x T) is then SHA-256'd here (FIPS 180-4, hashlib).
"""
import ctypes as C
import hashlib
import json
import struct
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

M64 = (1 << 64) - 1


def splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def logits(seed, T, V):
    n = T * V
    idx = np.arange(n, dtype=np.uint64) + np.uint64(seed)
    with np.errstate(over="ignore"):
        x = idx + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    bits = ((x & np.uint64(0x007FFFFF)) | np.uint64(0x3F800000) | ((x >> np.uint64(32)) & np.uint64(0x80000000)))
    return bits.astype(np.uint32).view(np.float32).reshape(T, V)


def main():
    R = O.ref()
    cases = []
    for seed, T, V in [(1, 3, 1), (2, 2, 5), (3, 2, 1024), (4, 2, 1025), (5, 3, 4096), (6, 1, 32771),
                       (7, 4, 4096 * 3), (8, 2, 128256), (9, 0, 4096)]:
        lg = logits(seed, T, V)
        tokens = [(t * 7 + seed) % V for t in range(T)]
        roots = []
        for t in range(T):
            b = lg[t].astype("<f4").tobytes()
            leaves = []
            for i in range(0, len(b), O.V2_LEAF_BYTES):
                chunk = np.frombuffer(b[i:i + O.V2_LEAF_BYTES], dtype=np.uint8).copy()
                out = np.zeros(32, np.uint8)
                R.ref_leaf_hash(chunk.ctypes.data, chunk.size, out.ctypes.data)
                leaves.append(out)
            lh = np.concatenate(leaves) if leaves else np.zeros(32, np.uint8)
            root = np.zeros(32, np.uint8)
            R.ref_merkle_root(lh.ctypes.data, len(leaves), root.ctypes.data)
            roots.append(root.tobytes())
        env = [O.V2_TAG, struct.pack("<I", T), np.asarray(tokens, "<u4").tobytes(), struct.pack("<I", T)]
        for r in roots:
            env += [struct.pack("<I", V), r]
        cases.append({"seed": seed, "T": T, "V": V, "tokens": tokens, "roots": [r.hex() for r in roots],
                      "out_hash_v2": hashlib.sha256(b"".join(env)).hexdigest()})
    e = np.zeros(32, np.uint8)
    R.ref_merkle_root(e.ctypes.data, 0, e.ctypes.data)
    doc = {"generator": "tests/golden/make_receipt_v2_golden.py (reference da.cpp via oracle/_ref)",
           "leaf_bytes": O.V2_LEAF_BYTES, "empty_root": e.tobytes().hex(), "cases": cases}
    (ROOT / "tests/golden/receipt_v2.json").write_text(json.dumps(doc, indent=1) + "\n")
    print(f"{len(cases)} cases")


if __name__ == "__main__":
    main()
