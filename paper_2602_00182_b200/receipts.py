"""Receipts and the replay verifier over the GPU engine.

Host-side formats of the reference (proj/src/receipts.cpp, codec.cpp, da.cpp), byte-identical on
well-formed input and pinned by golden vectors from the reference's own sources
(tests/golden/receipts_reference.json):

* ``canonical_receipt_body`` / ``encode_receipt`` / ``decode_receipt`` / DA records
  (receipts.cpp:12-105): big-endian fixed-width integers, u32-length-prefixed strings and blobs;
* ``receipt_to_json`` / ``receipt_from_json`` (receipts.cpp:223-275): same keys, order and
  ``dump(2)`` layout; hashes / signature hex, att_quote base64;
* ``policy_to_string`` / ``policy_from_string`` (codec.cpp:123-190), parsed with the C library's
  ``strtoul`` / ``strtof`` like the reference;
* ``make_receipt`` / ``verify_receipt`` (receipts.cpp:107-149), Ed25519 (RFC 8032, deterministic)
  through PyNaCl's libsodium — the reference's own signer library;
* ``reproduce_and_verify`` (receipts.cpp:171-219): the auditor path, re-executing the recorded
  execution tuple on the GPU engine (``detcore.infer``) and comparing output hashes; the verdict
  names the first failing step exactly as the reference does.

Decoders are strict (no trailing bytes, has_k / has_p in {0, 1}, no payload on absent optional
fields): the reference decoders' malleability (codec.cpp:76-91) is not inherited.
"""
from __future__ import annotations

import base64
import ctypes as C
import json
import struct
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Set, Tuple

from . import detcore
from .detcore import DecodeKind, DecodePolicy, ExecutionTuple

_libc = C.CDLL(None)
_libc.strtoul.restype = C.c_ulong
_libc.strtoul.argtypes = [C.c_char_p, C.POINTER(C.c_char_p), C.c_int]
_libc.strtof.restype = C.c_float
_libc.strtof.argtypes = [C.c_char_p, C.POINTER(C.c_char_p)]


# ---------------------------------------------------------------- codec (codec.hpp:16-50)
class Writer:
    def __init__(self):
        self.buf = bytearray()

    def u8(self, v: int):
        self.buf.append(v & 0xFF)

    def u32(self, v: int):
        self.buf += struct.pack(">I", v & 0xFFFFFFFF)

    def u64(self, v: int):
        self.buf += struct.pack(">Q", v & 0xFFFFFFFFFFFFFFFF)

    def f32(self, v: float):
        self.buf += struct.pack(">f", v)

    def str(self, s: str):
        b = s.encode("utf-8", "surrogateescape")
        self.u32(len(b))
        self.buf += b

    def blob(self, b: bytes):
        self.u32(len(b))
        self.buf += b

    def hash(self, h: bytes):
        assert len(h) == 32
        self.buf += h

    def take(self) -> bytes:
        return bytes(self.buf)


class Reader:
    """Every getter returns None past the end (codec.cpp:20-66)."""

    def __init__(self, data: bytes):
        self.d, self.pos = bytes(data), 0

    def _take(self, n: int) -> Optional[bytes]:
        if self.pos + n > len(self.d):
            return None
        b = self.d[self.pos:self.pos + n]
        self.pos += n
        return b

    def u8(self):
        b = self._take(1)
        return None if b is None else b[0]

    def u32(self):
        b = self._take(4)
        return None if b is None else struct.unpack(">I", b)[0]

    def u64(self):
        b = self._take(8)
        return None if b is None else struct.unpack(">Q", b)[0]

    def f32(self):
        b = self._take(4)
        return None if b is None else struct.unpack(">f", b)[0]

    def blob(self):
        n = self.u32()
        return None if n is None else self._take(n)

    def str(self):
        b = self.blob()
        return None if b is None else b.decode("utf-8", "surrogateescape")

    def hash(self):
        return self._take(32)

    def exhausted(self) -> bool:
        return self.pos == len(self.d)


def encode_policy(w: Writer, p: DecodePolicy):   # codec.cpp:67-74
    w.u8(int(p.kind))
    w.u8(1 if p.k is not None else 0)
    w.u32(p.k or 0)
    w.u8(1 if p.p is not None else 0)
    w.f32(0.0 if p.p is None else p.p)
    w.u32(p.max_tokens)


def decode_policy(r: Reader) -> Optional[DecodePolicy]:   # codec.cpp:76-91, strict
    kind, has_k, k, has_p = r.u8(), r.u8(), r.u32(), r.u8()
    pbits = r._take(4)
    mt = r.u32()
    if None in (kind, has_k, k, has_p, pbits, mt) or kind > int(DecodeKind.nucleus):
        return None
    if has_k not in (0, 1) or has_p not in (0, 1) or (not has_k and k != 0) or (not has_p and pbits != b"\0\0\0\0"):
        return None
    return DecodePolicy(DecodeKind(kind), k if has_k else None, struct.unpack(">f", pbits)[0] if has_p else None, mt)


def policy_to_string(p: DecodePolicy) -> str:   # codec.cpp:123-146
    if p.kind == DecodeKind.greedy:
        return f"greedy,max_tokens={p.max_tokens}"
    if p.kind == DecodeKind.top_k:
        return f"top_k,k={p.k or 0},max_tokens={p.max_tokens}"
    return "nucleus,p=%.9g,max_tokens=%u" % (float(struct.unpack("<f", struct.pack("<f", p.p or 0.0))[0]), p.max_tokens)


def policy_from_string(text: str) -> Optional[DecodePolicy]:   # codec.cpp:148-190
    rest = text
    fields: List[str] = []
    while rest:   # next_field: stops at the first empty remainder
        comma = rest.find(",")
        fields.append(rest if comma < 0 else rest[:comma])
        rest = "" if comma < 0 else rest[comma + 1:]
    if not fields:
        return None
    kinds = {"greedy": DecodeKind.greedy, "top_k": DecodeKind.top_k, "nucleus": DecodeKind.nucleus}
    if fields[0] not in kinds:
        return None
    kind, k, p, mt, have_max = kinds[fields[0]], None, None, 0, False
    for f in fields[1:]:
        eq = f.find("=")
        if eq < 0:
            return None
        key, value = f[:eq], f[eq + 1:]
        if not value:
            return None
        raw = value.encode("utf-8", "surrogateescape")
        end = C.c_char_p()
        buf = C.create_string_buffer(raw)
        if key == "k":
            k = _libc.strtoul(buf, C.byref(end), 10) & 0xFFFFFFFF
        elif key == "p":
            p = float(_libc.strtof(buf, C.byref(end)))
        elif key == "max_tokens":
            mt = _libc.strtoul(buf, C.byref(end), 10) & 0xFFFFFFFF
            have_max = True
        else:
            return None
        consumed = C.cast(end, C.c_void_p).value - C.addressof(buf)
        if consumed != len(raw):
            return None
    pol = DecodePolicy(kind, k, p, mt)
    if not have_max or pol.validate():
        return None
    return pol


# ---------------------------------------------------------------- signatures (sign.hpp)
class Ed25519Signer:
    """Ed25519Signer::from_seed (sign.cpp:17-24): deterministic keypair and signatures."""

    def __init__(self, seed: bytes):
        from nacl.signing import SigningKey

        if len(seed) != 32:
            raise ValueError("Ed25519 seed must be 32 bytes")
        self._sk = SigningKey(seed)

    @classmethod
    def from_seed(cls, seed: bytes) -> "Ed25519Signer":
        return cls(seed)

    def sign(self, message: bytes) -> bytes:
        return bytes(self._sk.sign(message).signature)

    def public_key(self) -> bytes:
        return bytes(self._sk.verify_key)


def verify_signature(public_key: bytes, message: bytes, signature: bytes) -> bool:   # sign.cpp:30-38
    from nacl.exceptions import BadSignatureError
    from nacl.signing import VerifyKey

    if len(public_key) != 32 or len(signature) != 64:
        return False
    try:
        VerifyKey(public_key).verify(message, signature)
        return True
    except BadSignatureError:
        return False


# ---------------------------------------------------------------- receipts (receipts.hpp:20-120)
@dataclass
class Registry:
    """Local stand-in for on-chain registration (receipts.hpp:24-31). The reference's default
    approves archA / archB; ``for_engine()`` adds the GPU profile "b200"."""
    archs: detcore.ArchRegistry = field(default_factory=lambda: detcore.ArchRegistry(["archA", "archB"]))
    containers: Set[bytes] = field(default_factory=set)
    models: Set[str] = field(default_factory=set)

    @classmethod
    def for_engine(cls) -> "Registry":
        return cls(archs=detcore.ArchRegistry.defaults())


@dataclass
class Receipt:
    model_id: str = ""
    chain_id: str = ""
    container_digest: bytes = b"\0" * 32
    gpu_arch: str = ""
    driver_tag: str = ""
    decode_policy: DecodePolicy = field(default_factory=lambda: DecodePolicy.greedy(0))
    seed: int = 0
    req_hash: bytes = b"\0" * 32
    out_hash: bytes = b"\0" * 32
    att_quote: Optional[bytes] = None
    timestamp: int = 0
    da_pointer: str = ""
    key_epoch: int = 0
    sig: bytes = b""


def canonical_receipt_body(rc: Receipt) -> bytes:   # receipts.cpp:12-29
    w = Writer()
    w.str(rc.model_id)
    w.str(rc.chain_id)
    w.hash(rc.container_digest)
    w.str(rc.gpu_arch)
    w.str(rc.driver_tag)
    encode_policy(w, rc.decode_policy)
    w.u64(rc.seed)
    w.hash(rc.req_hash)
    w.hash(rc.out_hash)
    w.u8(1 if rc.att_quote is not None else 0)
    if rc.att_quote is not None:
        w.blob(rc.att_quote)
    w.u64(rc.timestamp)
    w.str(rc.da_pointer)
    w.u32(rc.key_epoch)
    return w.take()


def encode_receipt(rc: Receipt) -> bytes:   # receipts.cpp:31-36
    w = Writer()
    w.blob(canonical_receipt_body(rc))
    w.blob(rc.sig)
    return w.take()


def _decode_body(body: bytes) -> Optional[Receipt]:   # receipts.cpp:38-70
    r = Reader(body)
    model_id, chain_id, digest, arch, driver = r.str(), r.str(), r.hash(), r.str(), r.str()
    policy = decode_policy(r)
    seed, req_hash, out_hash, has_quote = r.u64(), r.hash(), r.hash(), r.u8()
    if None in (model_id, chain_id, digest, arch, driver, policy, seed, req_hash, out_hash, has_quote):
        return None
    if has_quote not in (0, 1):
        return None
    quote = None
    if has_quote:
        quote = r.blob()
        if quote is None:
            return None
    timestamp, pointer, epoch = r.u64(), r.str(), r.u32()
    if None in (timestamp, pointer, epoch) or not r.exhausted():
        return None
    return Receipt(model_id, chain_id, digest, arch, driver, policy, seed, req_hash, out_hash, quote, timestamp,
                   pointer, epoch)


def decode_receipt(data: bytes) -> Optional[Receipt]:   # receipts.cpp:72-82
    r = Reader(data)
    body, sig = r.blob(), r.blob()
    if body is None or sig is None or not r.exhausted():
        return None
    rc = _decode_body(body)
    if rc is not None:
        rc.sig = sig
    return rc


def encode_da_record(cipher: bytes, rc: Receipt) -> bytes:   # receipts.cpp:84-89
    w = Writer()
    w.blob(cipher)
    w.blob(encode_receipt(rc))
    return w.take()


def decode_da_record(data: bytes) -> Optional[Tuple[bytes, Receipt]]:   # receipts.cpp:91-100
    r = Reader(data)
    cipher, rb = r.blob(), r.blob()
    if cipher is None or rb is None or not r.exhausted():
        return None
    rc = decode_receipt(rb)
    return None if rc is None else (cipher, rc)


def make_receipt(exec_: ExecutionTuple, out: detcore.InferenceOutput, operator_key: Ed25519Signer, chain_id: str,
                 da_pointer: str, key_epoch: int, timestamp: int, att_quote: Optional[bytes] = None) -> Receipt:
    """receipts.cpp:107-127: req_hash commits to the execution tuple, out_hash to the canonical
    output bytes (the engine's out_hash, computed without materialising them)."""
    rc = Receipt(exec_.model_id, chain_id, exec_.container_digest, exec_.arch, exec_.driver_tag, exec_.decode_policy,
                 exec_.seed, detcore.req_hash(exec_), out.out_hash, att_quote, timestamp, da_pointer, key_epoch)
    rc.sig = operator_key.sign(canonical_receipt_body(rc))
    return rc


def verify_receipt(rc: Receipt, operator_pubkey: bytes, registry: Optional[Registry] = None) -> Tuple[bool, str]:
    """receipts.cpp:133-149: (ok, why) with the reference's failure strings and check order."""
    registry = registry or Registry()
    if not registry.archs.contains(rc.gpu_arch):
        return False, "gpu_arch not in approved set"
    if rc.decode_policy.validate():
        return False, "malformed decode_policy"
    if registry.containers and rc.container_digest not in registry.containers:
        return False, "container_digest not registered"
    if registry.models and rc.model_id not in registry.models:
        return False, "model_id not registered"
    if not verify_signature(operator_pubkey, canonical_receipt_body(rc), rc.sig):
        return False, "signature invalid"
    return True, ""


def receipt_to_json(rc: Receipt) -> str:   # receipts.cpp:223-242 (nlohmann ordered_json, dump(2))
    j = {"model_id": rc.model_id, "chain_id": rc.chain_id, "container_digest": rc.container_digest.hex(),
         "gpu_arch": rc.gpu_arch, "driver_tag": rc.driver_tag, "decode_policy": policy_to_string(rc.decode_policy),
         "seed": rc.seed, "req_hash": rc.req_hash.hex(), "out_hash": rc.out_hash.hex()}
    if rc.att_quote is not None:
        j["att_quote"] = base64.b64encode(rc.att_quote).decode()
    j.update({"sig": rc.sig.hex(), "da_pointer": rc.da_pointer, "epoch": rc.key_epoch, "timestamp": rc.timestamp})
    return json.dumps(j, indent=2, ensure_ascii=False)


def _hex32(s) -> Optional[bytes]:
    b = _hex(s)
    return b if b is not None and len(b) == 32 else None


def _hex(s) -> Optional[bytes]:
    if not isinstance(s, str) or len(s) % 2:
        return None
    try:
        return bytes.fromhex(s) if all(c in "0123456789abcdefABCDEF" for c in s) else None
    except ValueError:
        return None


def _uint(v, bits) -> Optional[int]:
    return v if isinstance(v, int) and not isinstance(v, bool) and 0 <= v < (1 << bits) else None


def receipt_from_json(text: str) -> Optional[Receipt]:   # receipts.cpp:244-275
    try:
        j = json.loads(text)
    except (ValueError, RecursionError):
        return None
    if not isinstance(j, dict):
        return None
    try:
        strs = [j["model_id"], j["chain_id"], j["gpu_arch"], j["driver_tag"], j["da_pointer"]]
        if not all(isinstance(s, str) for s in strs):
            return None
        digest, req, out = _hex32(j["container_digest"]), _hex32(j["req_hash"]), _hex32(j["out_hash"])
        pol = policy_from_string(j["decode_policy"]) if isinstance(j["decode_policy"], str) else None
        seed, epoch = _uint(j["seed"], 64), _uint(j["epoch"], 32)
        ts = _uint(j.get("timestamp", 0), 64)
        sig = _hex(j["sig"])
    except KeyError:
        return None
    if None in (digest, req, out, pol, seed, epoch, ts, sig):
        return None
    quote = None
    if "att_quote" in j:
        if not isinstance(j["att_quote"], str):
            return None
        try:
            quote = base64.b64decode(j["att_quote"], validate=True)
        except ValueError:
            return None
    return Receipt(strs[0], strs[1], digest, strs[2], strs[3], pol, seed, req, out, quote, ts, strs[4], epoch, sig)


# ---------------------------------------------------------------- DA store (da.hpp rules)
@dataclass
class InclusionProof:
    slot_id: int = 0
    root: bytes = b""
    path: List[Tuple[bytes, bool]] = field(default_factory=list)   # (sibling, sibling_is_left), leaf upward
    leaf: bytes = b""


def leaf_hash(blob: bytes) -> bytes:   # da.cpp:27-34
    return detcore.sha256(b"\x00" + blob)


def node_hash(left: bytes, right: bytes) -> bytes:   # da.cpp:36-43
    return detcore.sha256(b"\x01" + left + right)


def merkle_root(hashes: Sequence[bytes]) -> bytes:   # da.cpp:45-61
    level = list(hashes)
    if not level:
        return leaf_hash(b"")
    while len(level) > 1:
        level = [node_hash(level[i], level[i + 1] if i + 1 < len(level) else level[i]) for i in range(0, len(level), 2)]
    return level[0]


def verify_inclusion(proof: InclusionProof, trusted_root: bytes) -> bool:   # da.cpp:63-69
    acc = leaf_hash(proof.leaf)
    for sib, is_left in proof.path:
        acc = node_hash(sib, acc) if is_left else node_hash(acc, sib)
    return acc == trusted_root and proof.root == trusted_root


class MemoryStore:
    """In-memory DA store with the reference's semantics (da.cpp:99-147): publish into the open
    slot, seal with advance_slot, fetch with an inclusion proof; withhold() censors a pointer."""

    def __init__(self):
        self.current_slot = 0
        self.open: List[bytes] = []
        self.sealed: Dict[int, Tuple[List[bytes], List[bytes], bytes]] = {}
        self.censored: Set[Tuple[int, int]] = set()

    def publish(self, blob: bytes) -> str:
        self.open.append(bytes(blob))
        return f"{self.current_slot}:{len(self.open) - 1}"

    def advance_slot(self):
        hashes = [leaf_hash(b) for b in self.open]
        self.sealed[self.current_slot] = (self.open, hashes, merkle_root(hashes))
        self.open = []
        self.current_slot += 1

    def withhold(self, pointer: str):
        self.censored.add(parse_pointer(pointer))

    def root_of(self, slot: int) -> Optional[bytes]:
        return self.sealed[slot][2] if slot in self.sealed else None

    def fetch_with_proof(self, slot: int, index: int):
        if slot not in self.sealed or index >= len(self.sealed[slot][0]):
            return "not_found", b"", None
        if (slot, index) in self.censored:
            return "withheld", b"", None
        leaves, hashes, root = self.sealed[slot]
        path, level, pos = [], list(hashes), index
        while len(level) > 1:   # da.cpp:80-97
            sib = pos + 1 if pos % 2 == 0 else pos - 1
            if sib >= len(level):
                sib = pos
            path.append((level[sib], sib < pos))
            level = [node_hash(level[i], level[i + 1] if i + 1 < len(level) else level[i])
                     for i in range(0, len(level), 2)]
            pos //= 2
        return "ok", leaves[index], InclusionProof(slot, root, path, leaves[index])


def parse_pointer(text: str) -> Optional[Tuple[int, int]]:   # DaPointer::parse, da.cpp:13-25
    colon = text.find(":")
    if colon < 0:
        return None
    a, b = text[:colon], text[colon + 1:]
    if not (a.isdigit() and b.isdigit() and a.isascii() and b.isascii()):
        return None
    slot, idx = int(a), int(b)
    return (slot, idx) if slot < (1 << 64) and idx < (1 << 32) else None


# ---------------------------------------------------------------- auditor path
@dataclass
class ResponseMetadata:   # receipts.hpp:82-90, receipts.cpp:151-167
    system_fingerprint: str
    determinism_seed: int
    receipt: Receipt
    da_link: str

    @classmethod
    def from_receipt(cls, rc: Receipt) -> "ResponseMetadata":
        return cls(f"{rc.container_digest.hex()}:{rc.gpu_arch}:{rc.driver_tag}", rc.seed, rc, rc.da_pointer)

    def consistent(self) -> bool:
        rc = self.receipt
        return (self.system_fingerprint == f"{rc.container_digest.hex()}:{rc.gpu_arch}:{rc.driver_tag}"
                and self.determinism_seed == rc.seed and self.da_link == rc.da_pointer)


@dataclass
class KeyAccess:
    decrypt: Callable[[bytes, int], Optional[Tuple[bytes, bytes]]]
    epoch_valid: Callable[[int], bool]


@dataclass
class Verdict:
    verified: bool
    detail: str


def reproduce_and_verify(store: MemoryStore, meta: ResponseMetadata, key_access: KeyAccess, operator_pubkey: bytes,
                         registry: Optional[Registry] = None,
                         reexecute: Optional[Callable[[ExecutionTuple], bytes]] = None) -> Verdict:
    """receipts.cpp:171-219 with the re-execution routed to the GPU engine: `reexecute(exec)`
    returns the out_hash (default: detcore.infer on the engine for exec.arch)."""
    registry = registry or Registry.for_engine()
    bad = lambda step: Verdict(False, step)   # noqa: E731
    if not meta.consistent():
        return bad("metadata-consistency")
    ptr = parse_pointer(meta.da_link)
    if ptr is None:
        return bad("da-pointer")
    status, blob, proof = store.fetch_with_proof(*ptr)
    if status == "withheld":
        return bad("da-availability")
    if status != "ok":
        return bad("fetch")
    root = store.root_of(ptr[0])
    if root is None or not verify_inclusion(proof, root):
        return bad("inclusion-proof")
    rec = decode_da_record(blob)
    if rec is None:
        return bad("record-decode")
    cipher, rc = rec
    if rc != meta.receipt:
        return bad("receipt-mismatch")
    ok, why = verify_receipt(rc, operator_pubkey, registry)
    if not ok:
        return bad("receipt-verify: " + why)
    if key_access.epoch_valid is None or not key_access.epoch_valid(rc.key_epoch):
        return bad("epoch-validity")
    plain = key_access.decrypt(cipher, rc.key_epoch)
    if plain is None:
        return bad("decrypt")
    req_bytes, out_bytes = plain
    if detcore.sha256(req_bytes) != rc.req_hash:
        return bad("request-hash")
    if detcore.sha256(out_bytes) != rc.out_hash:
        return bad("cipher-binding")
    exec_ = detcore.decode_execution_tuple(req_bytes)
    if exec_ is None:
        return bad("request-decode")
    try:
        got = reexecute(exec_) if reexecute is not None else detcore.infer(exec_, registry.archs).out_hash
    except Exception:   # noqa: BLE001 - the reference maps any throw to this step
        return bad("re-execute")
    if got != rc.out_hash:
        return bad("output-hash")
    return Verdict(True, "ok")


def verify_replay(req_bytes: bytes, out_hash: bytes, registry: Optional[Registry] = None) -> Verdict:
    """The CLI `verify-receipt --exec` core (verinf_cli.cpp:199-233): decode the tuple strictly,
    re-execute on the GPU engine, compare out_hash."""
    registry = registry or Registry.for_engine()
    exec_ = detcore.decode_execution_tuple(req_bytes)
    if exec_ is None:
        return Verdict(False, "request-decode")
    try:
        got = detcore.infer(exec_, registry.archs).out_hash
    except Exception:   # noqa: BLE001
        return Verdict(False, "re-execute")
    return Verdict(got == out_hash, "ok" if got == out_hash else "output-hash")
