"""The C-ABI library: loads, exports every symbol include/detgpu.h declares, and its host-side receipt
functions (SHA-256, canonical layout, ExecutionTuple codec) agree with the oracle. No GPU needed."""
import hashlib
import random
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "detgpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(detgpu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2602_00182_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing, missing
    assert b"sm_100a" in _lib.lib.detgpu_version()


def test_arch_registry():
    from paper_2602_00182_b200 import _lib

    for a in (b"archA", b"archB", b"b200"):
        assert _lib.lib.detgpu_arch_supported(a)
    assert not _lib.lib.detgpu_arch_supported(b"archZ")


def test_sha256_vectors_and_random():
    from paper_2602_00182_b200.detcore import sha256

    assert sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    rng = random.Random(7)
    for n in [1, 55, 56, 57, 63, 64, 65, 119, 120, 127, 128, 1000, 65537]:
        blob = bytes(rng.getrandbits(8) for _ in range(n))
        assert sha256(blob) == hashlib.sha256(blob).digest(), n


def test_canonical_encoding_matches_oracle_and_streaming_hash():
    from paper_2602_00182_b200 import _lib
    from paper_2602_00182_b200.detcore import decode_canonical_output, encode_canonical_output

    rng = np.random.default_rng(3)
    for T, V in [(0, 32), (1, 32), (5, 32), (3, 4096), (2, 128256)]:
        toks = rng.integers(0, V, T).astype(np.uint32)
        logits = rng.standard_normal((T, V)).astype(np.float32)
        mine = encode_canonical_output(toks, logits)
        assert mine == O.encode_canonical(toks, logits)
        out = np.zeros(32, dtype=np.uint8)
        lg = logits if T else np.zeros(1, np.float32)
        _lib.lib.detgpu_hash_canonical(toks.ctypes.data if T else None, T, lg.ctypes.data, V, out.ctypes.data)
        assert out.tobytes() == hashlib.sha256(mine).digest()
        dec = decode_canonical_output(mine)
        assert dec is not None and dec[0] == toks.tolist()
        assert decode_canonical_output(mine + b"\0") is None
        if len(mine) > 8:
            assert decode_canonical_output(mine[:-1]) is None


def _random_exec(rng):
    from paper_2602_00182_b200.detcore import DecodePolicy, ExecutionTuple

    kind = rng.randrange(3)
    pol = [DecodePolicy.greedy(rng.randrange(300)), DecodePolicy.top_k(rng.randrange(1, 50), rng.randrange(300)),
           DecodePolicy.nucleus(rng.choice([0.1, 0.5, 0.9, 1.0]), rng.randrange(300))][kind]
    return ExecutionTuple(model_id=rng.choice(["llama-tiny:a", "llama3-8b", "model-a", ""]),
                          container_digest=bytes(rng.getrandbits(8) for _ in range(32)),
                          arch=rng.choice(["b200", "archA", "archB"]), driver_tag=rng.choice(["drv-1", "x"]),
                          decode_policy=pol, seed=rng.getrandbits(64),
                          prompt=[rng.randrange(128256) for _ in range(rng.randrange(20))])


def test_exec_tuple_codec_matches_oracle_and_round_trips():
    from paper_2602_00182_b200.detcore import decode_execution_tuple, encode_execution_tuple

    rng = random.Random(11)
    for _ in range(300):
        e = _random_exec(rng)
        b = encode_execution_tuple(e)
        p = e.decode_policy
        assert b == O.encode_exec_tuple(e.model_id, e.container_digest, e.arch, e.driver_tag, int(p.kind), p.k, p.p,
                                        p.max_tokens, e.seed, e.prompt)
        d = decode_execution_tuple(b)
        assert d is not None and encode_execution_tuple(d) == b
        assert d.prompt == list(e.prompt) and d.seed == e.seed and d.decode_policy == e.decode_policy


def test_exec_tuple_strict_decoder_rejects_every_bit_flip_that_changes_meaning():
    """Reference decode_policy accepts has_k/has_p bytes other than 0/1 and ignores payloads of absent
    fields (codec.cpp:76-91), so test_receipts.cpp:79-102 fails on it. Here every
    single-bit mutation either fails to decode or re-encodes to the mutated bytes."""
    from paper_2602_00182_b200.detcore import decode_execution_tuple, encode_execution_tuple

    rng = random.Random(5)
    for _ in range(20):
        b = bytearray(encode_execution_tuple(_random_exec(rng)))
        for bit in range(len(b) * 8):
            m = bytearray(b)
            m[bit // 8] ^= 1 << (bit % 8)
            d = decode_execution_tuple(bytes(m))
            if d is not None:
                assert encode_execution_tuple(d) == bytes(m)
    assert decode_execution_tuple(encode_execution_tuple(_random_exec(rng)) + b"\0") is None
    assert decode_execution_tuple(b"") is None


def test_policy_validation_strings():
    from paper_2602_00182_b200.detcore import DecodeKind, DecodePolicy

    assert DecodePolicy(DecodeKind.top_k).validate() == "top_k policy requires k"
    assert DecodePolicy(DecodeKind.nucleus, p=1.5).validate() == "nucleus p must be in (0,1]"
    assert DecodePolicy(DecodeKind.greedy, k=2, max_tokens=4).validate() == "greedy policy must not carry k or p"
    assert DecodePolicy.top_k(40, 8).validate() == ""
