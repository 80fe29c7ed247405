"""ctypes binding of the CPU oracle (oracle/build/liboracle.so) and of the compiled reference
(oracle/_ref/libref.so). TEST / MEASUREMENT INFRASTRUCTURE ONLY: imported by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs as the checker.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import struct
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libref.so"

_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_SO))
        vp, sz, u32, u64, i32, i64, f32 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_float
        sig = {
            "orc_set_threads": (None, [i32]), "orc_get_threads": (i32, []),
            "orc_set_gemm_mode": (None, [i32]), "orc_tc_dot": (f32, [vp, vp, i32]),
            "orc_tc_dot_fast": (f32, [vp, vp, i32]), "orc_have_avx2": (i32, []),
            "orc_gemm": (None, [vp, vp, i32, i32, i32, vp]),
            "orc_fnv1a64": (u64, [C.c_char_p]), "orc_mix_seed": (u64, [u64, u64]),
            "orc_prng_seeded": (None, [u64, vp]), "orc_prng_next_u64": (u64, [vp]),
            "orc_prng_next_below": (u64, [vp, u64]), "orc_prng_next_unit_f32": (f32, [vp]),
            "orc_tree_reduce": (f32, [vp, sz]), "orc_seq_reduce": (f32, [vp, sz]),
            "orc_expf": (f32, [f32]), "orc_expf_array": (None, [vp, vp, sz]),
            "orc_libm_expf_array": (None, [vp, vp, sz]),
            "orc_softmax": (i32, [vp, sz, vp]),
            "orc_decode_with_draw": (i64, [vp, sz, i32, i32, u32, i32, f32, f32]),
            "orc_sha256": (None, [vp, sz, vp]),
            "orc_canonical_size": (sz, [u32, u32]),
            "orc_encode_canonical": (None, [vp, u32, vp, u32, vp]),
            "orc_encode_exec_tuple": (sz, [C.c_char_p, vp, C.c_char_p, C.c_char_p, i32, i32, u32, i32, f32, u32,
                                           u64, vp, u32, vp]),
            "orc_toy_infer": (i32, [C.c_char_p, i32, vp, u32, i32, i32, u32, i32, f32, u32, u64, vp, vp]),
            "orc_gen_tensor": (None, [u64, i64, i64, i32, i32, vp]),
            "orc_rmsnorm": (None, [vp, vp, i32, f32, vp]),
            "orc_attention_head": (None, [vp, vp, vp, i32, i32, vp]),
            "orc_rope_table": (None, [C.c_double, i32, i32, vp, vp]),
            "orc_llama_new": (vp, [C.c_char_p]), "orc_llama_free": (None, [vp]),
            "orc_llama_info": (None, [vp, vp]), "orc_llama_tensor_seed": (u64, [vp, i32]),
            "orc_llama_tensor": (vp, [vp, i32, i32]),
            "orc_llama_teacher": (i32, [vp, vp, i32, i32, vp]),
            "orc_llama_generate": (i32, [vp, vp, u32, i32, i32, u32, i32, f32, u32, u64, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def ref():
    """The reference's own detcore/codec compiled from /root/reference sources (may be absent)."""
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise ImportError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        R = C.CDLL(str(REF_SO))
        vp, u32, u64, i32, f32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_float
        R.ref_infer.restype = i32
        R.ref_infer.argtypes = [C.c_char_p, vp, C.c_char_p, C.c_char_p, i32, i32, u32, i32, f32, u32, u64, vp, u32,
                                vp, vp, vp, vp, vp]
        R.ref_infer_batch.restype = i32
        R.ref_infer_batch.argtypes = [C.c_char_p, vp, C.c_char_p, i32, i32, u32, i32, f32, u32, u64, vp, u32, u32,
                                      u32, vp]
        R.ref_bench.restype = C.c_double
        R.ref_bench.argtypes = [C.c_char_p, C.c_char_p, u32, u32, u32, i32, C.POINTER(u64)]
        R.ref_leaf_hash.restype = None
        R.ref_leaf_hash.argtypes = [vp, C.c_size_t, vp]
        R.ref_node_hash.restype = None
        R.ref_node_hash.argtypes = [vp, vp, vp]
        R.ref_merkle_root.restype = None
        R.ref_merkle_root.argtypes = [vp, C.c_size_t, vp]
        _ref = R
    return _ref


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------- thin pythonic helpers
class Prng:
    """xoshiro256++ seeded by splitmix64 (reference prng.hpp)."""

    def __init__(self, seed: int):
        self.s = np.zeros(4, dtype=np.uint64)
        lib().orc_prng_seeded(seed, ptr(self.s))

    def next_u64(self) -> int:
        return int(lib().orc_prng_next_u64(ptr(self.s)))

    def next_below(self, bound: int) -> int:
        return int(lib().orc_prng_next_below(ptr(self.s), bound))

    def next_unit_f32(self) -> float:
        return float(lib().orc_prng_next_unit_f32(ptr(self.s)))


def tree_reduce(v) -> np.float32:
    a = np.ascontiguousarray(v, dtype=np.float32)
    return np.float32(lib().orc_tree_reduce(ptr(a), a.size))


def seq_reduce(v) -> np.float32:
    a = np.ascontiguousarray(v, dtype=np.float32)
    return np.float32(lib().orc_seq_reduce(ptr(a), a.size))


def expf(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(a)
    lib().orc_expf_array(ptr(a), ptr(out), a.size)
    return out


def libm_expf(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(a)
    lib().orc_libm_expf_array(ptr(a), ptr(out), a.size)
    return out


def softmax(logits) -> np.ndarray:
    a = np.ascontiguousarray(logits, dtype=np.float32)
    out = np.empty_like(a)
    if lib().orc_softmax(ptr(a), a.size, ptr(out)) != 0:
        raise ValueError("det_softmax: empty or non-finite input")
    return out


def decode_with_draw(probs, kind: int, k=None, p=None, r: float = 0.0) -> int:
    a = np.ascontiguousarray(probs, dtype=np.float32)
    t = lib().orc_decode_with_draw(ptr(a), a.size, kind, k is not None, k or 0, p is not None,
                                   0.0 if p is None else p, r)
    if t < 0:
        raise ValueError("decode: invalid argument")
    return int(t)


def sha256(data: bytes) -> bytes:
    buf = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, dtype=np.uint8)
    out = np.zeros(32, dtype=np.uint8)
    lib().orc_sha256(ptr(buf), len(data), ptr(out))
    return out.tobytes()


def encode_canonical(tokens, logits) -> bytes:
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    lg = np.ascontiguousarray(logits, dtype=np.float32).reshape(t.size, -1) if t.size else np.zeros((0, 0), np.float32)
    V = lg.shape[1] if t.size else 0
    out = np.zeros(lib().orc_canonical_size(t.size, V), dtype=np.uint8)
    lib().orc_encode_canonical(ptr(t) if t.size else None, t.size, ptr(lg) if t.size else None, V, ptr(out))
    return out.tobytes()


def encode_exec_tuple(model_id: str, digest: bytes, arch: str, driver: str, kind: int, k, p, max_tokens: int,
                      seed: int, prompt) -> bytes:
    pr = np.ascontiguousarray(prompt, dtype=np.uint32)
    dg = np.frombuffer(digest, dtype=np.uint8).copy()
    args = (model_id.encode(), ptr(dg), arch.encode(), driver.encode(), kind, k is not None, k or 0, p is not None,
            0.0 if p is None else p, max_tokens, seed, ptr(pr) if pr.size else None, pr.size)
    n = lib().orc_encode_exec_tuple(*args, None)
    out = np.zeros(n, dtype=np.uint8)
    lib().orc_encode_exec_tuple(*args, ptr(out))
    return out.tobytes()


def toy_infer(model_id: str, arch: str, prompt, kind: int, k=None, p=None, max_tokens: int = 0, seed: int = 0):
    pr = np.ascontiguousarray(prompt, dtype=np.uint32)
    toks = np.zeros(max(max_tokens, 1), dtype=np.uint32)
    logits = np.zeros((max(max_tokens, 1), 32), dtype=np.float32)
    rc = lib().orc_toy_infer(model_id.encode(), {"archA": 0, "archB": 1}.get(arch, 9), ptr(pr) if pr.size else None,
                             pr.size, kind, k is not None, k or 0, p is not None, 0.0 if p is None else p, max_tokens,
                             seed, ptr(toks), ptr(logits))
    if rc != 0:
        raise ValueError(f"toy infer failed ({rc})")
    return toks[:max_tokens].copy(), logits[:max_tokens].copy()


def gemm(W_u16: np.ndarray, X_u16: np.ndarray) -> np.ndarray:
    """Y[c, r] = W[r] . X[c] under the active accumulation profile (default: b200 / tcgen05)."""
    W = np.ascontiguousarray(W_u16, dtype=np.uint16)
    X = np.ascontiguousarray(X_u16, dtype=np.uint16)
    Y = np.zeros((X.shape[0], W.shape[0]), dtype=np.float32)
    lib().orc_gemm(ptr(W), ptr(X), W.shape[0], W.shape[1], X.shape[0], ptr(Y))
    return Y


class gemm_profile:
    """Context manager: 0 = b200 (tcgen05 accumulation), 1 = reference canonical tree (archA-style)."""

    def __init__(self, mode: int):
        self.mode = mode

    def __enter__(self):
        lib().orc_set_gemm_mode(self.mode)

    def __exit__(self, *a):
        lib().orc_set_gemm_mode(0)


def gen_tensor(seed: int, rows: int, cols: int, scale_exp: int, is_gamma: bool) -> np.ndarray:
    out = np.zeros((rows, cols), dtype=np.uint16)
    lib().orc_gen_tensor(seed, rows, cols, scale_exp, int(is_gamma), ptr(out))
    return out


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


def rmsnorm(x: np.ndarray, gamma_u16: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.zeros(x.shape, dtype=np.uint16)
    for r in range(x.shape[0]):
        lib().orc_rmsnorm(ptr(x[r]), ptr(gamma_u16), x.shape[1], eps, ptr(out[r]))
    return out


def attention_head(q_u16, k_u16, v_u16) -> np.ndarray:
    q = np.ascontiguousarray(q_u16, dtype=np.uint16)
    k = np.ascontiguousarray(k_u16, dtype=np.uint16)
    v = np.ascontiguousarray(v_u16, dtype=np.uint16)
    out = np.zeros(q.size, dtype=np.uint16)
    lib().orc_attention_head(ptr(q), ptr(k), ptr(v), k.shape[0], q.size, ptr(out))
    return out


class Llama:
    """CPU oracle of the Llama-style transformer."""

    def __init__(self, model_id: str):
        self.h = lib().orc_llama_new(model_id.encode())
        if not self.h:
            raise ValueError(f"unknown model config for {model_id!r}")
        f = np.zeros(7, dtype=np.int32)
        lib().orc_llama_info(self.h, ptr(f))
        self.L, self.d, self.hq, self.hkv, self.hd, self.F, self.V = (int(x) for x in f)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_llama_free(self.h)
            self.h = None

    def teacher(self, tokens, first_logit_pos: int) -> np.ndarray:
        t = np.ascontiguousarray(tokens, dtype=np.uint32)
        out = np.zeros((t.size - first_logit_pos, self.V), dtype=np.float32)
        if lib().orc_llama_teacher(self.h, ptr(t), t.size, first_logit_pos, ptr(out)) != 0:
            raise ValueError("teacher: token out of vocabulary")
        return out

    def generate(self, prompt, kind: int = 0, k=None, p=None, max_tokens: int = 8, seed: int = 0):
        pr = np.ascontiguousarray(prompt, dtype=np.uint32)
        toks = np.zeros(max(max_tokens, 1), dtype=np.uint32)
        logits = np.zeros((max(max_tokens, 1), self.V), dtype=np.float32)
        rc = lib().orc_llama_generate(self.h, ptr(pr), pr.size, kind, k is not None, k or 0, p is not None,
                                      0.0 if p is None else p, max_tokens, seed, ptr(toks), ptr(logits))
        if rc != 0:
            raise ValueError(f"oracle generate failed ({rc})")
        return toks[:max_tokens].copy(), logits[:max_tokens].copy()


def out_hash(tokens, logits) -> bytes:
    return hashlib.sha256(encode_canonical(tokens, logits)).digest()


# ---- receipt v2 ----
# Per generated step, the Merkle root of the step's f32 logits (little-endian bytes) split into
# 4 KiB leaves, with the reference's DA tree rules (proj/include/verinf/da.hpp:16-20):
#   leaf H(0x00 || blob) (da.cpp:27-34), node H(0x01 || l || r) (da.cpp:36-43),
#   odd level: last hash paired with itself; empty list -> H(0x00) (da.cpp:45-61).
# out_hash_v2 = SHA-256("RCPTv2\0\0" || [u32 T][T tokens][u32 T][(u32 V, root) x T]) (LE, like v1).
V2_LEAF_BYTES = 4096
V2_TAG = b"RCPTv2\x00\x00"


def merkle_leaf(blob: bytes) -> bytes:
    return sha256(b"\x00" + blob)


def merkle_node(left: bytes, right: bytes) -> bytes:
    return sha256(b"\x01" + left + right)


def merkle_root(leaf_hashes) -> bytes:
    level = list(leaf_hashes)
    if not level:
        return merkle_leaf(b"")
    while len(level) > 1:
        level = [merkle_node(level[i], level[i + 1] if i + 1 < len(level) else level[i])
                 for i in range(0, len(level), 2)]
    return level[0]


def step_root(logits_row) -> bytes:
    b = np.ascontiguousarray(logits_row, dtype="<f4").tobytes()
    return merkle_root([merkle_leaf(b[i:i + V2_LEAF_BYTES]) for i in range(0, len(b), V2_LEAF_BYTES)])


def encode_canonical_v2(tokens, logits) -> bytes:
    t = np.ascontiguousarray(tokens, dtype="<u4")
    T = t.size
    lg = np.ascontiguousarray(logits, dtype="<f4").reshape(T, -1) if T else np.zeros((0, 0), "<f4")
    out = [V2_TAG, struct.pack("<I", T), t.tobytes(), struct.pack("<I", T)]
    for i in range(T):
        out += [struct.pack("<I", lg.shape[1]), step_root(lg[i])]
    return b"".join(out)


def hash_canonical_v2(tokens, logits) -> bytes:
    return sha256(encode_canonical_v2(tokens, logits))
