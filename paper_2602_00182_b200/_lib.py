"""ctypes binding of ``libdetgpu.so`` (the C-ABI in ``include/detgpu.h``).

There is no fallback: if the library is missing, importing this module raises. Build it with
``python -m paper_2602_00182_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# DETGPU_LIB selects an experiment build (build.py --variant) for A/B timing; default: the product.
LIB_PATH = Path(os.environ.get("DETGPU_LIB") or Path(__file__).resolve().parent / "libdetgpu.so")

DETGPU_OK = 0
DETGPU_EINVAL = 1
DETGPU_ECUDA = 2
DETGPU_ENOMEM = 3
DETGPU_ENONFINITE = 4
DETGPU_ENODEV = 5

GREEDY, TOP_K, NUCLEUS = 0, 1, 2
F_DEVICE_ONLY = 1
F_RECEIPT_V2 = 2
F_CONTINUOUS = 4


class Policy(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("has_k", C.c_uint8), ("has_p", C.c_uint8), ("reserved", C.c_uint8),
                ("k", C.c_uint32), ("p", C.c_float), ("max_tokens", C.c_uint32)]


class ModelInfo(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("d_model", C.c_uint32), ("n_heads", C.c_uint32),
                ("n_kv_heads", C.c_uint32), ("head_dim", C.c_uint32), ("ffn", C.c_uint32), ("vocab", C.c_uint32),
                ("toy", C.c_uint32), ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("n_params", C.c_uint64),
                ("weight_bytes", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("prefill_ms", C.c_float), ("decode_ms", C.c_float), ("d2h_ms", C.c_float), ("hash_ms", C.c_float),
                ("decode_steps", C.c_uint64), ("tokens", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("kernel_launches", C.c_uint64)]


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build the CUDA library first (python -m paper_2602_00182_b200.build)")
    lib = C.CDLL(str(LIB_PATH))
    vp, sz, u32, i32, i64, u64 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_int, C.c_int64, C.c_uint64
    sig = {
        "detgpu_version": (C.c_char_p, []),
        "detgpu_debug_check_canaries": (i32, [C.POINTER(u64), C.POINTER(u64)]),
        "detgpu_global_error": (C.c_char_p, []),
        "detgpu_arch_supported": (i32, [C.c_char_p]),
        "detgpu_create": (i32, [i32, C.c_char_p, C.c_char_p, u32, u32, C.POINTER(vp)]),
        "detgpu_destroy": (None, [vp]),
        "detgpu_get_model_info": (i32, [vp, C.POINTER(ModelInfo)]),
        "detgpu_last_error": (C.c_char_p, [vp]),
        "detgpu_generate": (i32, [vp, u32, C.POINTER(C.POINTER(u32)), C.POINTER(u32), C.POINTER(Policy),
                                  C.POINTER(u64), u32, C.POINTER(C.POINTER(u32)), C.POINTER(C.POINTER(C.c_float)),
                                  C.POINTER(C.c_uint8), u32, C.POINTER(Stats)]),
        "detgpu_stream": (vp, [vp]),
        "detgpu_profile_decode_step": (i32, [vp, u32, u32, u32, C.POINTER(C.c_float), C.POINTER(u32)]),
        "detgpu_profile_graph": (i32, [vp, u32, u32, u32, u32, C.POINTER(C.c_float)]),
        "detgpu_set_option": (i32, [vp, C.c_char_p, C.c_int64]),
        "detgpu_trace_read": (i32, [vp, vp, u32, C.POINTER(u32)]),
        "detgpu_sha256": (None, [vp, sz, vp]),
        "detgpu_canonical_size": (sz, [u32, u32]),
        "detgpu_encode_canonical": (None, [vp, u32, vp, u32, vp]),
        "detgpu_hash_canonical": (None, [vp, u32, vp, u32, vp]),
        "detgpu_step_root": (None, [vp, u32, vp]),
        "detgpu_hash_canonical_v2": (None, [vp, u32, vp, u32, vp]),
        "detgpu_k_step_roots": (i32, [vp, i32, i32, vp, vp]),
        "detgpu_encode_exec_tuple": (sz, [C.c_char_p, vp, C.c_char_p, C.c_char_p, C.POINTER(Policy), u64, vp, u32, vp]),
        "detgpu_decode_exec_tuple": (i32, [vp, sz, C.c_char_p, sz, vp, C.c_char_p, sz, C.c_char_p, sz,
                                           C.POINTER(Policy), C.POINTER(u64), vp, u32, C.POINTER(u32)]),
        "detgpu_k_gemm": (i32, [vp, vp, vp, i32, i32, i32, i64, vp]),
        "detgpu_k_gemm_split": (i32, [vp, vp, vp, i32, i32, i32, i64, i32, vp]),
        "detgpu_k_rmsnorm": (i32, [vp, vp, vp, i32, i32, C.c_float, vp]),
        "detgpu_k_expf": (i32, [vp, vp, i64, vp]),
        "detgpu_k_tree_sum": (i32, [vp, vp, i32, i32, vp]),
        "detgpu_k_init_tensor": (i32, [vp, u64, i64, i64, i32, i32, i32, i32, vp]),
        "detgpu_k_sample": (i32, [vp, i32, i32, C.POINTER(Policy), vp, vp, vp, vp, vp]),
        "detgpu_k_attention": (i32, [vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # reported by tests/test_abi.py, which requires every declared symbol
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int, handle=None) -> None:
    if rc == DETGPU_OK:
        return
    msg = (lib.detgpu_last_error(handle) if handle else lib.detgpu_global_error()) or b""
    msg = msg.decode(errors="replace")
    if rc in (DETGPU_EINVAL, DETGPU_ENONFINITE):
        raise ValueError(msg)  # the reference throws std::invalid_argument
    raise RuntimeError(f"detgpu error {rc}: {msg}")
