"""Reference-shaped API over the C-ABI: the names, argument meaning and error behaviour of
``verinf::detcore`` (reference proj/include/verinf/detcore.hpp:21-163), executed on the B200.

    exec = ExecutionTuple(model_id="llama-tiny:model-a", container_digest=..., arch="b200",
                          driver_tag="drv-1", decode_policy=DecodePolicy.greedy(64), seed=42,
                          prompt=[1, 5, 9, 13, 2])
    out = infer(exec)            # InferenceOutput(tokens, logits_trace, canonical_bytes)
    outs = infer_batch(execs, batch_size=8)

Arch profiles: "archA" / "archB" run the reference ToyModel (bit-exact with the reference's CPU
engine), "b200" runs the Llama-style transformer named by the model_id prefix. Invalid input
raises ValueError, the Python face of the reference's std::invalid_argument.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from . import _lib as L


class DecodeKind(IntEnum):
    greedy = 0
    top_k = 1
    nucleus = 2


@dataclass(frozen=True)
class DecodePolicy:
    """detcore.hpp:52-66."""

    kind: DecodeKind = DecodeKind.greedy
    k: Optional[int] = None
    p: Optional[float] = None
    max_tokens: int = 0

    def __post_init__(self):
        # p is a float32 everywhere it matters (the C-ABI, the codec, req_hash; detcore.hpp:55):
        # round it here so validate() judges the value that is actually used
        if self.p is not None:
            object.__setattr__(self, "p", float(np.float32(self.p)))

    @staticmethod
    def greedy(max_tokens: int) -> "DecodePolicy":
        return DecodePolicy(DecodeKind.greedy, None, None, max_tokens)

    @staticmethod
    def top_k(k: int, max_tokens: int) -> "DecodePolicy":
        return DecodePolicy(DecodeKind.top_k, k, None, max_tokens)

    @staticmethod
    def nucleus(p: float, max_tokens: int) -> "DecodePolicy":
        return DecodePolicy(DecodeKind.nucleus, None, float(np.float32(p)), max_tokens)

    def validate(self) -> str:
        """Empty on success, else the reference's diagnostic (detcore.cpp:52-69)."""
        if self.kind == DecodeKind.greedy:
            return "greedy policy must not carry k or p" if (self.k is not None or self.p is not None) else ""
        if self.kind == DecodeKind.top_k:
            if self.k is None:
                return "top_k policy requires k"
            if self.k == 0:
                return "top_k k must be positive"
            if self.p is not None:
                return "top_k policy must not carry p"
            return ""
        if self.kind == DecodeKind.nucleus:
            if self.p is None:
                return "nucleus policy requires p"
            if not (self.p > 0.0) or self.p > 1.0:
                return "nucleus p must be in (0,1]"
            if self.k is not None:
                return "nucleus policy must not carry k"
            return ""
        return "unknown decode kind"

    def to_c(self) -> L.Policy:
        return L.Policy(int(self.kind), self.k is not None, self.p is not None, 0, self.k or 0,
                        0.0 if self.p is None else self.p, self.max_tokens)


@dataclass
class ExecutionTuple:
    """detcore.hpp:68-77."""

    model_id: str
    container_digest: bytes = bytes(32)
    arch: str = "b200"
    driver_tag: str = "drv-1"
    decode_policy: DecodePolicy = field(default_factory=lambda: DecodePolicy.greedy(0))
    seed: int = 0
    prompt: Sequence[int] = ()


@dataclass
class InferenceOutput:
    """detcore.hpp:79-85 (canonical_bytes is built on first access; out_hash is always present)."""

    tokens: np.ndarray
    logits_trace: Optional[np.ndarray]
    out_hash: bytes
    _canonical: Optional[bytes] = None

    @property
    def canonical_bytes(self) -> bytes:
        if self._canonical is None:
            self._canonical = encode_canonical_output(self.tokens, self.logits_trace)
        return self._canonical


class ReductionOrder(IntEnum):
    canonical_tree = 0
    sequential = 1
    tcgen05_b200 = 2


@dataclass(frozen=True)
class ArchProfile:
    """detcore.hpp:21-30. The order selects the engine: canonical_tree / sequential run the
    reference ToyModel ("archA" / "archB"), tcgen05_b200 the Llama-style transformer ("b200")."""

    name: str
    reduction_order: ReductionOrder = ReductionOrder.canonical_tree

    @property
    def engine_arch(self) -> str:
        return {ReductionOrder.canonical_tree: "archA", ReductionOrder.sequential: "archB"}.get(
            self.reduction_order, "b200")


_KNOWN = {"archA": ReductionOrder.canonical_tree, "archB": ReductionOrder.sequential,
          "b200": ReductionOrder.tcgen05_b200}


class ArchRegistry:
    """Approved profiles (detcore.hpp:34-47, detcore.cpp:12-26, plus the GPU profile "b200").
    Built from names of known profiles and/or ArchProfile objects; add() registers more."""

    _default = None

    def __init__(self, profiles=()):
        self._p = {}
        for x in profiles:
            self.add(x if isinstance(x, ArchProfile) else ArchProfile(x, _KNOWN[x]) if x in _KNOWN else None)

    def add(self, profile: Optional[ArchProfile]) -> None:
        if profile is not None:
            self._p[profile.name] = profile

    @classmethod
    def defaults(cls) -> "ArchRegistry":
        if cls._default is None:
            cls._default = ArchRegistry(["archA", "archB", "b200"])
        return cls._default

    def find(self, name: str) -> Optional[ArchProfile]:
        return self._p.get(name)

    def contains(self, name: str) -> bool:
        p = self._p.get(name)
        return p is not None and bool(L.lib.detgpu_arch_supported(p.engine_arch.encode()))

    def names(self):
        return sorted(self._p)


# ---------------------------------------------------------------- canonical bytes & receipts
def encode_canonical_output(tokens, logits_trace) -> bytes:
    """detcore.cpp:73-84 via the library encoder."""
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    T = int(t.size)
    V = int(logits_trace.shape[1]) if T else 0
    lg = np.ascontiguousarray(logits_trace, dtype=np.float32) if T else np.zeros(1, np.float32)
    n = L.lib.detgpu_canonical_size(T, V)
    out = np.zeros(n, dtype=np.uint8)
    L.lib.detgpu_encode_canonical(t.ctypes.data if T else None, T, lg.ctypes.data, V, out.ctypes.data)
    return out.tobytes()


def decode_canonical_output(data: bytes):
    """Strict inverse of encode_canonical_output (detcore.cpp:86-123): trailing bytes rejected."""
    b = memoryview(data)
    pos = 0

    def u32():
        nonlocal pos
        if pos + 4 > len(b):
            raise ValueError("truncated")
        v = int.from_bytes(b[pos:pos + 4], "little")
        pos += 4
        return v

    try:
        T = u32()
        toks = [u32() for _ in range(T)]
        S = u32()
        rows = []
        for _ in range(S):
            V = u32()
            if pos + 4 * V > len(b):
                raise ValueError("truncated")
            rows.append(np.frombuffer(bytes(b[pos:pos + 4 * V]), dtype="<f4").copy())
            pos += 4 * V
    except ValueError:
        return None
    if pos != len(b):
        return None
    return toks, rows


def sha256(data: bytes) -> bytes:
    buf = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    out = np.zeros(32, dtype=np.uint8)
    L.lib.detgpu_sha256(buf.ctypes.data, len(data), out.ctypes.data)
    return out.tobytes()


def encode_execution_tuple(e: ExecutionTuple) -> bytes:
    """codec.cpp:93-104; req_hash = sha256 of these bytes (receipts.cpp:119)."""
    pr = np.ascontiguousarray(e.prompt, dtype=np.uint32)
    dg = np.frombuffer(bytes(e.container_digest), dtype=np.uint8).copy()
    pol = e.decode_policy.to_c()
    enc = lambda s: s.encode("utf-8", "surrogateescape")  # noqa: E731
    args = (enc(e.model_id), dg.ctypes.data, enc(e.arch), enc(e.driver_tag), C.byref(pol), e.seed,
            pr.ctypes.data if pr.size else None, pr.size)
    n = L.lib.detgpu_encode_exec_tuple(*args, None)
    out = np.zeros(n, dtype=np.uint8)
    L.lib.detgpu_encode_exec_tuple(*args, out.ctypes.data)
    return out.tobytes()


def decode_execution_tuple(data: bytes) -> Optional[ExecutionTuple]:
    """Strict decoder: None for anything that is not exactly encode_execution_tuple(x)."""
    buf = np.frombuffer(data, dtype=np.uint8).copy() if data else np.zeros(1, np.uint8)
    mid, arch, drv = C.create_string_buffer(4096), C.create_string_buffer(4096), C.create_string_buffer(4096)
    dg = np.zeros(32, dtype=np.uint8)
    pol = L.Policy()
    seed = C.c_uint64()
    cap = max(1, len(data) // 4)
    prompt = np.zeros(cap, dtype=np.uint32)
    plen = C.c_uint32()
    rc = L.lib.detgpu_decode_exec_tuple(buf.ctypes.data, len(data), mid, 4096, dg.ctypes.data, arch, 4096, drv, 4096,
                                        C.byref(pol), C.byref(seed), prompt.ctypes.data, cap, C.byref(plen))
    if rc != L.DETGPU_OK:
        return None
    dp = DecodePolicy(DecodeKind(pol.kind), pol.k if pol.has_k else None,
                      float(np.float32(pol.p)) if pol.has_p else None, pol.max_tokens)
    dec = lambda b: b.value.decode("utf-8", "surrogateescape")  # noqa: E731 (std::string is raw bytes)
    return ExecutionTuple(dec(mid), dg.tobytes(), dec(arch), dec(drv), dp, seed.value,
                          prompt[:plen.value].tolist())


def hash_canonical_v2(tokens, logits) -> bytes:
    """Receipt v2 digest on the host (detgpu_hash_canonical_v2): what DETGPU_F_RECEIPT_V2 computes."""
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    T = t.size
    lg = np.ascontiguousarray(logits, dtype=np.float32).reshape(T, -1) if T else np.zeros((0, 1), np.float32)
    out = np.zeros(32, np.uint8)
    L.lib.detgpu_hash_canonical_v2(t.ctypes.data if T else None, T, lg.ctypes.data if T else None, lg.shape[1],
                                   out.ctypes.data)
    return out.tobytes()


def req_hash(e: ExecutionTuple) -> bytes:
    return sha256(encode_execution_tuple(e))


# ---------------------------------------------------------------- engine
class Engine:
    """One engine per (GPU, model_id, arch) = one replica. Calls on one instance are serialised."""

    def __init__(self, model_id: str, arch: str = "b200", max_batch: int = 64, max_context: int = 1024,
                 device: int = 0):
        h = C.c_void_p()
        L.check(L.lib.detgpu_create(device, model_id.encode(), arch.encode(), max_batch, max_context, C.byref(h)))
        self.h = h
        self.model_id, self.arch, self.device = model_id, arch, device
        self.max_batch, self.max_context = max_batch, max_context
        info = L.ModelInfo()
        L.check(L.lib.detgpu_get_model_info(self.h, C.byref(info)), self.h)
        self.info = info
        self.vocab = int(info.vocab)
        self.last_stats = L.Stats()
        # one call at a time per handle (detgpu.h): ctypes releases the GIL during detgpu_generate
        self._lock = threading.Lock()

    def close(self):
        if getattr(self, "h", None):
            L.lib.detgpu_destroy(self.h)
            self.h = None

    __del__ = close

    def set_option(self, name: str, value: int) -> None:
        """Scheduling knob that never changes a result bit (detgpu_set_option)."""
        L.check(L.lib.detgpu_set_option(self.h, name.encode(), int(value)), self.h)

    def generate(self, prompts, policies, seeds, batch_size: Optional[int] = None, want_logits: bool = True,
                 want_hash: bool = True, device_only: bool = False, receipt_v2: bool = False,
                 continuous: bool = False):
        """Returns (tokens list[np.uint32], logits list[np.float32 [T,V]] or None, hashes list[bytes]).
        receipt_v2: hashes are the v2 digest (per-step Merkle roots on the GPU).
        continuous: batch_size decode slots stay busy, requests admitted as slots free (same bytes)."""
        n = len(prompts)
        pr = [np.ascontiguousarray(p, dtype=np.uint32) for p in prompts]
        pr_ptrs = (C.POINTER(C.c_uint32) * n)(*[p.ctypes.data_as(C.POINTER(C.c_uint32)) for p in pr])
        lens = (C.c_uint32 * n)(*[p.size for p in pr])
        pols = (L.Policy * n)(*[p.to_c() for p in policies])
        sd = (C.c_uint64 * n)(*[s & (2**64 - 1) for s in seeds])
        toks = [np.zeros(max(p.max_tokens, 1), dtype=np.uint32) for p in policies]
        tok_ptrs = (C.POINTER(C.c_uint32) * n)(*[t.ctypes.data_as(C.POINTER(C.c_uint32)) for t in toks])
        logits = None
        lg_ptrs = None
        if want_logits and not device_only:
            logits = [np.zeros((p.max_tokens, self.vocab), dtype=np.float32) for p in policies]
            lg_ptrs = (C.POINTER(C.c_float) * n)(*[
                (lg.ctypes.data_as(C.POINTER(C.c_float)) if lg.size else C.POINTER(C.c_float)()) for lg in logits])
        hashes = np.zeros(32 * n, dtype=np.uint8) if (want_hash and not device_only) else None
        stats = L.Stats()
        with self._lock:
            rc = self._generate(n, pr_ptrs, lens, pols, sd, batch_size, tok_ptrs, lg_ptrs, hashes, device_only,
                                receipt_v2, continuous, stats)
        L.check(rc, self.h)
        self.last_stats = stats
        toks = [t[:p.max_tokens] for t, p in zip(toks, policies)]
        hs = [hashes[32 * i:32 * i + 32].tobytes() for i in range(n)] if hashes is not None else None
        return toks, logits, hs

    def _generate(self, n, pr_ptrs, lens, pols, sd, batch_size, tok_ptrs, lg_ptrs, hashes, device_only, receipt_v2,
                  continuous, stats):
        return L.lib.detgpu_generate(self.h, n, pr_ptrs, lens, pols, sd, batch_size or self.max_batch, tok_ptrs, lg_ptrs,
                                   hashes.ctypes.data_as(C.POINTER(C.c_uint8)) if hashes is not None else None,
                                   (L.F_DEVICE_ONLY if device_only else 0) | (L.F_RECEIPT_V2 if receipt_v2 else 0)
                                   | (L.F_CONTINUOUS if continuous else 0),
                                   C.byref(stats))


# One cached engine per (device, model_id, engine arch), sized from the requests: rebuilt with a
# larger context when a request needs it (the reference accepts any length), at most MAX_ENGINES
# kept (least recently used dropped). Engine.generate holds the engine's own lock.
ENGINE_MAX_BATCH = 64
ENGINE_MIN_CONTEXT = 2048
MAX_ENGINES = 4
_engines: dict = {}
_lock = threading.Lock()
_clock = [0]


def _engine_for(model_id: str, engine_arch: str, need_ctx: int, device: int = 0) -> Engine:
    key = (device, model_id, engine_arch)
    with _lock:
        _clock[0] += 1
        ent = _engines.get(key)
        if ent is not None and (engine_arch != "b200" or ent[0].max_context >= need_ctx):
            ent[1] = _clock[0]
            return ent[0]
        ctx = ENGINE_MIN_CONTEXT
        while ctx < need_ctx:
            ctx *= 2
        if ent is None and len(_engines) >= MAX_ENGINES:
            victim = min(_engines, key=lambda k: _engines[k][1])
            del _engines[victim]
        eng = Engine(model_id, engine_arch, max_batch=ENGINE_MAX_BATCH, max_context=ctx if engine_arch == "b200" else 1,
                     device=device)
        _engines[key] = [eng, _clock[0]]
        return eng


def release_engines() -> None:
    """Drop every cached engine (GPU memory is freed once no call is using it)."""
    with _lock:
        _engines.clear()


def infer_batch(execs: Sequence[ExecutionTuple], batch_size: int, registry: Optional[ArchRegistry] = None,
                device: int = 0):
    """detcore.cpp:387-410: per-tuple results are byte-identical to individual infer() calls.
    Every tuple is validated (arch against `registry`, then policy) before any work."""
    registry = registry or ArchRegistry.defaults()
    if batch_size == 0:
        raise ValueError("infer_batch: batch_size must be positive")
    results = [None] * len(execs)
    groups: dict = {}
    for i, e in enumerate(execs):
        prof = registry.find(e.arch)
        if prof is None or not registry.contains(e.arch):
            raise ValueError(f"infer: unknown arch profile '{e.arch}'")
        err = e.decode_policy.validate()
        if err:
            raise ValueError("infer: " + err)
        groups.setdefault((e.model_id, prof.engine_arch), []).append(i)
    for (mid, arch), idx in groups.items():
        need = max(max(len(execs[i].prompt), 1) + execs[i].decode_policy.max_tokens for i in idx)
        eng = _engine_for(mid, arch, need, device)
        toks, logits, hashes = eng.generate([execs[i].prompt for i in idx], [execs[i].decode_policy for i in idx],
                                            [execs[i].seed for i in idx], batch_size=batch_size)
        for j, i in enumerate(idx):
            results[i] = InferenceOutput(toks[j], logits[j], hashes[j])
    return results


def infer(e: ExecutionTuple, registry: Optional[ArchRegistry] = None, device: int = 0) -> InferenceOutput:
    """detcore.cpp:380-385."""
    return infer_batch([e], 1, registry, device)[0]
