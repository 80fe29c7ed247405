"""Golden vectors for the receipt formats from the REFERENCE's own receipts.cpp / codec.cpp /
sign.cpp / sha256.cpp (compiled from /root/reference by `make -C oracle ref-receipts`, libsodium
from PyNaCl, nlohmann json):  python tests/golden/make_receipts_golden.py
-> tests/golden/receipts_reference.json (body / wire / JSON / signature / verify verdicts,
policy display strings). Canonical output bytes come from the CPU oracle's ToyModel."""
import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

R = C.CDLL(str(ROOT / "oracle" / "_ref" / "libref_receipts.so"))
vp, sz, u32, u64, i32, f32 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64, C.c_int, C.c_float
R.refr_make.restype = i32
R.refr_make.argtypes = [C.c_char_p, vp, C.c_char_p, C.c_char_p, i32, i32, u32, i32, f32, u32, u64, vp, u32, vp, sz, vp,
                        C.c_char_p, C.c_char_p, u32, u64, vp, sz, i32, vp, C.POINTER(sz), vp, C.POINTER(sz),
                        C.c_char_p, C.POINTER(sz), vp]
R.refr_verify.restype = i32
R.refr_verify.argtypes = [vp, sz, vp, C.c_char_p, sz]
R.refr_json_to_wire.restype = sz
R.refr_json_to_wire.argtypes = [C.c_char_p, vp, sz]
R.refr_policy_to_string.restype = sz
R.refr_policy_to_string.argtypes = [i32, i32, u32, i32, f32, u32, C.c_char_p, sz]
R.refr_policy_from_string.restype = i32
R.refr_policy_from_string.argtypes = [C.c_char_p] + [C.POINTER(i32), C.POINTER(i32), C.POINTER(u32), C.POINTER(i32),
                                                    C.POINTER(f32), C.POINTER(u32)]

KINDS = {"greedy": 0, "top_k": 1, "nucleus": 2}


def make(case, sign_seed):
    kind = KINDS[case["policy"][0]]
    k, p, mt = case["policy"][1], case["policy"][2], case["policy"][3]
    toks, logits = O.toy_infer(case["model_id"], case["arch"] if case["arch"] in ("archA", "archB") else "archA",
                               case["prompt"], kind, k, p, mt, case["seed"])
    canon = np.frombuffer(O.encode_canonical(toks, logits), np.uint8).copy()
    digest = np.frombuffer(hashlib.sha256(case["container"].encode()).digest(), np.uint8).copy()
    pr = np.asarray(case["prompt"], np.uint32)
    q = np.frombuffer(bytes.fromhex(case["att_quote"]) if case["att_quote"] is not None else b"\0", np.uint8).copy()
    bn, wn, jn = sz(0), sz(0), sz(0)
    pk = np.zeros(32, np.uint8)
    args = lambda b, w, j: (case["model_id"].encode(), digest.ctypes.data, case["arch"].encode(), case["driver"].encode(),
                            kind, k is not None, k or 0, p is not None, 0.0 if p is None else p, mt, case["seed"],
                            pr.ctypes.data, pr.size, canon.ctypes.data, canon.size, sign_seed.ctypes.data,
                            case["chain_id"].encode(), case["da_pointer"].encode(), case["key_epoch"],
                            case["timestamp"], q.ctypes.data, len(bytes.fromhex(case["att_quote"] or "")),
                            case["att_quote"] is not None, b, C.byref(bn), w, C.byref(wn), j, C.byref(jn),
                            pk.ctypes.data)
    R.refr_make(*args(None, None, None))
    body, wire = np.zeros(bn.value, np.uint8), np.zeros(wn.value, np.uint8)
    js = C.create_string_buffer(jn.value)
    R.refr_make(*args(body.ctypes.data, wire.ctypes.data, js))
    return canon.tobytes(), body.tobytes(), wire.tobytes(), js.value.decode(), pk.tobytes()


def verify(wire, pk):
    w = np.frombuffer(wire, np.uint8).copy()
    why = C.create_string_buffer(256)
    r = R.refr_verify(w.ctypes.data, w.size, np.frombuffer(pk, np.uint8).copy().ctypes.data, why, 256)
    return r, why.value.decode()


def main():
    sign_seed = np.frombuffer(hashlib.sha256(b"operator-key").digest(), np.uint8).copy()
    base = {"model_id": "model-a", "container": "container-a", "arch": "archA", "driver": "drv-1",
            "prompt": [1, 5, 9, 13, 2], "seed": 42, "chain_id": "chain-1", "da_pointer": "3:7", "key_epoch": 2,
            "timestamp": 1700000000, "att_quote": None, "policy": ["top_k", 4, None, 4]}
    variants = [
        {},
        {"policy": ["greedy", None, None, 8]},
        {"policy": ["nucleus", None, 0.9, 6], "att_quote": "00ff10" * 5},
        {"policy": ["nucleus", None, 0.1, 3], "arch": "archB", "model_id": "modèle-ü", "chain_id": "",
         "da_pointer": "18446744073709551615:0"},
        {"policy": ["top_k", 1, None, 2], "att_quote": "", "key_epoch": 4294967295, "timestamp": 0},
        {"arch": "b200", "policy": ["greedy", None, None, 1]},   # not in the reference's approved set
    ]
    cases = []
    for v in variants:
        case = dict(base, **v)
        canon, body, wire, js, pk = make(case, sign_seed)
        r, why = verify(wire, pk)
        tampered = bytearray(wire)
        tampered[20] ^= 1
        rt, why_t = verify(bytes(tampered), pk)
        back = np.zeros(len(wire) + 16, np.uint8)
        nb = R.refr_json_to_wire(js.encode(), back.ctypes.data, back.size)
        cases.append(dict(case, canonical_sha256=hashlib.sha256(canon).hexdigest(), body=body.hex(), wire=wire.hex(),
                          json=js, pubkey=pk.hex(), verify=[r, why], verify_tampered=[rt, why_t],
                          json_to_wire=back[:nb].tobytes().hex()))
    pols = []
    for name, k, p, mt in [("greedy", None, None, 8), ("top_k", 40, None, 8), ("nucleus", None, 0.9, 8),
                           ("nucleus", None, 0.1, 1), ("nucleus", None, 1.0, 256), ("top_k", 1, 0.5, 2)]:
        buf = C.create_string_buffer(96)
        R.refr_policy_to_string(KINDS[name], k is not None, k or 0, p is not None, 0.0 if p is None else p, mt, buf, 96)
        pols.append({"policy": [name, k, p, mt], "text": buf.value.decode()})
    parses = []
    for text in ["greedy,max_tokens=8", "top_k,k=40,max_tokens=8", "nucleus,p=0.9,max_tokens=8", "greedy",
                 "nucleus,p=1.5,max_tokens=8", "top_k,k=0,max_tokens=1", "greedy,max_tokens=8,", "beam,max_tokens=2",
                 "nucleus,p=0.899999976,max_tokens=3", "top_k,k=4,max_tokens=x", "greedy,max_tokens=8,k=3"]:
        a = [i32(), i32(), u32(), i32(), f32(), u32()]
        ok = R.refr_policy_from_string(text.encode(), *[C.byref(x) for x in a])
        parses.append({"text": text, "ok": ok,
                       "policy": [a[0].value, a[1].value, a[2].value, a[3].value, a[4].value, a[5].value] if ok else None})
    doc = {"generator": "tests/golden/make_receipts_golden.py (reference receipts/codec/sign/sha256 via oracle/_ref)",
           "sign_seed": sign_seed.tobytes().hex(), "receipts": cases, "policy_strings": pols, "policy_parses": parses}
    (ROOT / "tests/golden/receipts_reference.json").write_text(json.dumps(doc, indent=1, ensure_ascii=False) + "\n")
    print(len(cases), "receipts")


if __name__ == "__main__":
    main()
