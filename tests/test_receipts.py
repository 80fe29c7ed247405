"""Receipt formats and the replay verifier, pinned by golden vectors
from the reference's own receipts.cpp / codec.cpp / sign.cpp (tests/golden/make_receipts_golden.py)."""
import hashlib
import json
from pathlib import Path

import pytest

GOLD = json.loads((Path(__file__).parent / "golden" / "receipts_reference.json").read_text())
KIND = {"greedy": 0, "top_k": 1, "nucleus": 2}


def _policy(spec):
    from paper_2602_00182_b200.detcore import DecodeKind, DecodePolicy

    name, k, p, mt = spec
    import numpy as np

    return DecodePolicy(DecodeKind(KIND[name]), k, None if p is None else float(np.float32(p)), mt)


def _exec(c):
    from paper_2602_00182_b200.detcore import ExecutionTuple

    return ExecutionTuple(c["model_id"], hashlib.sha256(c["container"].encode()).digest(), c["arch"], c["driver"],
                          _policy(c["policy"]), c["seed"], c["prompt"])


def _receipt(c):
    from paper_2602_00182_b200 import receipts as R
    from paper_2602_00182_b200.detcore import InferenceOutput, req_hash

    signer = R.Ed25519Signer.from_seed(bytes.fromhex(GOLD["sign_seed"]))
    e = _exec(c)
    out = InferenceOutput(None, None, bytes.fromhex(c["canonical_sha256"]))
    quote = None if c["att_quote"] is None else bytes.fromhex(c["att_quote"])
    rc = R.make_receipt(e, out, signer, c["chain_id"], c["da_pointer"], c["key_epoch"], c["timestamp"], quote)
    assert rc.req_hash == req_hash(e)
    return rc, signer


@pytest.mark.parametrize("i", range(len(GOLD["receipts"])))
def test_receipt_bytes_json_and_signature_match_reference(i):
    from paper_2602_00182_b200 import receipts as R

    c = GOLD["receipts"][i]
    rc, signer = _receipt(c)
    assert signer.public_key().hex() == c["pubkey"]
    assert R.canonical_receipt_body(rc).hex() == c["body"]
    assert R.encode_receipt(rc).hex() == c["wire"]
    assert R.receipt_to_json(rc) == c["json"]
    assert R.decode_receipt(bytes.fromhex(c["wire"])) == rc
    back = R.receipt_from_json(c["json"])
    assert back is not None and R.encode_receipt(back).hex() == c["json_to_wire"] == c["wire"]
    ok, why = R.verify_receipt(rc, signer.public_key())   # the reference's default registry
    assert [int(ok), why] == c["verify"]
    tampered = bytearray(bytes.fromhex(c["wire"]))
    tampered[20] ^= 1
    dec = R.decode_receipt(bytes(tampered))
    if c["verify_tampered"][0] == -1:
        assert dec is None
    else:
        ok, why = R.verify_receipt(dec, signer.public_key())
        assert [int(ok), why] == c["verify_tampered"]


def test_policy_strings_match_reference():
    from paper_2602_00182_b200 import receipts as R

    for p in GOLD["policy_strings"]:
        assert R.policy_to_string(_policy(p["policy"])) == p["text"]
    for p in GOLD["policy_parses"]:
        got = R.policy_from_string(p["text"])
        if not p["ok"]:
            assert got is None, p["text"]
            continue
        kind, has_k, k, has_p, pv, mt = p["policy"]
        assert got is not None and int(got.kind) == kind and (got.k is not None) == bool(has_k)
        assert (got.k or 0) == k and (got.p is not None) == bool(has_p) and got.max_tokens == mt
        if has_p:
            assert got.p == pv


def test_strict_decoders_reject_malleable_encodings():
    from paper_2602_00182_b200 import receipts as R

    c = GOLD["receipts"][0]
    rc, _ = _receipt(c)
    wire = R.encode_receipt(rc)
    assert R.decode_receipt(wire + b"\0") is None
    body = bytearray(R.canonical_receipt_body(rc))
    # has_k flag byte: model_id, chain_id (u32 len + bytes each), digest, arch, driver, kind
    off = 4 + len(rc.model_id.encode()) + 4 + len(rc.chain_id.encode()) + 32 + 4 + len(rc.gpu_arch) + 4 + \
        len(rc.driver_tag) + 1
    body[off] = 2
    w = R.Writer()
    w.blob(bytes(body))
    w.blob(rc.sig)
    assert R.decode_receipt(w.take()) is None
    assert R.receipt_from_json("[]") is None and R.receipt_from_json("{") is None
    bad = json.loads(c["json"])
    bad["req_hash"] = bad["req_hash"][:-2]
    assert R.receipt_from_json(json.dumps(bad)) is None


def test_da_store_inclusion_proofs():
    from oracle import oracle as O
    from paper_2602_00182_b200 import receipts as R

    st = R.MemoryStore()
    ptrs = [st.publish(bytes([i]) * (i + 1)) for i in range(7)]
    st.advance_slot()
    root = st.root_of(0)
    assert root == O.merkle_root([O.merkle_leaf(bytes([i]) * (i + 1)) for i in range(7)])
    for p in ptrs:
        status, blob, proof = st.fetch_with_proof(*R.parse_pointer(p))
        assert status == "ok" and R.verify_inclusion(proof, root)
        proof.leaf = proof.leaf + b"x"
        assert not R.verify_inclusion(proof, root)
    assert st.fetch_with_proof(0, 7)[0] == "not_found" and st.fetch_with_proof(1, 0)[0] == "not_found"
    for bad in ["", "3", "3:", ":3", "a:1", "1:2:3", "-1:0", "1:4294967296"]:
        assert R.parse_pointer(bad) is None


def _pipeline(reexec_hash):
    """An honest receipt published to a DA store (cipher = plaintext blobs; the reference's sealed
    boxes are out of scope) and the auditor's inputs."""
    from paper_2602_00182_b200 import receipts as R
    from paper_2602_00182_b200.detcore import InferenceOutput, encode_execution_tuple

    c = GOLD["receipts"][0]
    e = _exec(c)
    signer = R.Ed25519Signer.from_seed(bytes.fromhex(GOLD["sign_seed"]))
    req = encode_execution_tuple(e)
    out_bytes = b"canonical-output-bytes"
    out = InferenceOutput(None, None, hashlib.sha256(out_bytes).digest())
    st = R.MemoryStore()
    st.publish(b"other")
    rc = R.make_receipt(e, out, signer, "chain-1", "0:1", 3, 99)
    w = R.Writer()
    w.blob(req)
    w.blob(out_bytes)
    cipher = w.take()
    st.publish(R.encode_da_record(cipher, rc))
    st.advance_slot()

    def decrypt(cph, epoch):
        r = R.Reader(cph)
        a, b = r.blob(), r.blob()
        return (a, b) if a is not None and b is not None and r.exhausted() else None

    ka = R.KeyAccess(decrypt, lambda ep: ep == 3)
    return st, R.ResponseMetadata.from_receipt(rc), ka, signer.public_key(), (lambda ex: reexec_hash)


def test_reproduce_and_verify_steps():
    from paper_2602_00182_b200 import receipts as R

    good = hashlib.sha256(b"canonical-output-bytes").digest()
    st, meta, ka, pk, rex = _pipeline(good)
    reg = R.Registry()
    assert R.reproduce_and_verify(st, meta, ka, pk, reg, rex) == R.Verdict(True, "ok")
    st2, meta2, ka2, pk2, rex2 = _pipeline(b"\1" * 32)
    assert R.reproduce_and_verify(st2, meta2, ka2, pk2, reg, rex2).detail == "output-hash"
    assert R.reproduce_and_verify(st, meta, R.KeyAccess(ka.decrypt, lambda ep: False), pk, reg, rex).detail == \
        "epoch-validity"
    assert R.reproduce_and_verify(st, meta, R.KeyAccess(lambda c, e: None, ka.epoch_valid), pk, reg, rex).detail == \
        "decrypt"
    st.withhold(meta.da_link)
    assert R.reproduce_and_verify(st, meta, ka, pk, reg, rex).detail == "da-availability"
    _, meta3, _, _, _ = _pipeline(good)
    meta3.determinism_seed += 1
    assert R.reproduce_and_verify(st2, meta3, ka, pk, reg, rex).detail == "metadata-consistency"
    st4, meta4, ka4, pk4, rex4 = _pipeline(good)
    assert R.reproduce_and_verify(st4, meta4, ka4, b"\0" * 32, reg, rex4).detail == "receipt-verify: signature invalid"


@pytest.mark.gpu
def test_replay_verifier_on_the_gpu_engine():
    """The auditor re-executes the recorded tuple on the GPU engine (toy archA and tiny Llama)."""
    from paper_2602_00182_b200 import receipts as R
    from paper_2602_00182_b200.detcore import DecodePolicy, ExecutionTuple, encode_execution_tuple, infer

    for e in [ExecutionTuple("model-a", bytes(32), "archA", "drv-1", DecodePolicy.top_k(4, 4), 42, [1, 5, 9, 13, 2]),
              ExecutionTuple("llama-tiny:verify", bytes(32), "b200", "drv-1", DecodePolicy.nucleus(0.9, 16), 7,
                             list(range(3, 30)))]:
        out = infer(e)
        req = encode_execution_tuple(e)
        assert R.verify_replay(req, out.out_hash) == R.Verdict(True, "ok")
        assert R.verify_replay(req, bytes(32)).detail == "output-hash"
        signer = R.Ed25519Signer.from_seed(b"\7" * 32)
        rc = R.make_receipt(e, out, signer, "c", "0:0", 1, 5)
        st = R.MemoryStore()
        w = R.Writer()
        w.blob(req)
        w.blob(out.canonical_bytes)
        st.publish(R.encode_da_record(w.take(), rc))
        st.advance_slot()
        def decrypt(cipher, epoch):
            r = R.Reader(cipher)
            return r.blob(), r.blob()

        ka = R.KeyAccess(decrypt, lambda ep: True)
        assert R.reproduce_and_verify(st, R.ResponseMetadata.from_receipt(rc), ka, signer.public_key()) == \
            R.Verdict(True, "ok")
        if e.arch == "archA":   # the reference fixture's out_hash (test_receipts.cpp:21-30)
            assert out.out_hash.hex() == "0e9a353b8c5e90e25da31269140f95b3c678864efc731b914363133397e61560"
