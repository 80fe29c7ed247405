"""Build the in-tree CUDA/C++ library ``libdetgpu.so`` for sm_100a (and the CPU oracle).

The library is the product: every kernel, the engine and the C-ABI declared in
``include/detgpu.h``. It is built with explicit ``-gencode arch=compute_100a,code=sm_100a`` (plain
``-arch=sm_100a`` emits compute_100 PTX that ptxas rejects for tcgen05) and ``--fmad=false`` so
that no multiply-add is contracted unless the source says ``__fmaf_rn`` (the reference's
determinism contract is ``-ffp-contract=off``, reference proj/CMakeLists.txt:10-12).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libdetgpu.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off,-msha,-msse4.1",
    "-Xptxas", "-v",
    "-I", str(ROOT / "include"), "-I", str(CSRC),
]


def _sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _stale(out: Path, inputs: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def build_lib(force: bool = False, verbose: bool = False, variant: str = "", defines: tuple = ()) -> Path:
    """`variant` + `defines` build an alternative libdetgpu_<variant>.so (A/B timing experiments,
    loaded with DETGPU_LIB=...); the default build is the product."""
    lib_out = LIB if not variant else PKG / f"libdetgpu_{variant}.so"
    srcs = _sources()
    deps = srcs + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))
    if not force and not _stale(lib_out, deps):
        return lib_out
    objdir = PKG / ("build" if not variant else f"build_{variant}")
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in srcs:
        obj = objdir / (src.name + ".o")
        hdrs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))
        if force or _stale(obj, [src] + hdrs):
            cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src.name}")
        objs.append(obj)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib_out), *map(str, objs),
           "-Xcompiler", "-fPIC", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link of libdetgpu.so failed")
    return lib_out


def build_oracle(force: bool = False) -> None:
    """The CPU oracle (test infrastructure) and, when /root/reference exists, oracle/_ref."""
    args = ["make", "-C", str(ROOT / "oracle")]
    if force:
        args.append("-B")
    r = subprocess.run(args, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("oracle build failed")
    if Path("/root/reference/proj/src/detcore.cpp").exists():
        r = subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref"], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("oracle/_ref build failed")
        # receipts/sign/sha256 over PyNaCl's libsodium: golden-vector generation only, optional
        r = subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref-receipts"], capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write("note: oracle/_ref/libref_receipts.so not built (golden receipts stay as committed)\n")


if __name__ == "__main__":
    force = "--force" in sys.argv
    if "--variant" in sys.argv:   # --variant NAME DEFINE [DEFINE ...]
        i = sys.argv.index("--variant")
        print(build_lib(force=force, variant=sys.argv[i + 1], defines=tuple(sys.argv[i + 2:])))
        sys.exit(0)
    build_lib(force=force, verbose="-v" in sys.argv)
    if "--lib-only" not in sys.argv:
        build_oracle(force=force)
    print(LIB)
