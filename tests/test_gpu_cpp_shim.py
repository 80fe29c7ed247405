"""The reference-shaped C++ shim (include/detgpu_detcore.hpp) compiled as a C++ program against
libdetgpu.so: golden toy receipts, batch invariance and invalid_argument, from C++."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def test_cpp_shim(tmp_path):
    exe = tmp_path / "shim_test"
    libdir = ROOT / "paper_2602_00182_b200"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", str(ROOT / "include"), str(ROOT / "tests/cpp/shim_test.cpp"),
                    "-L", str(libdir), "-l:libdetgpu.so", f"-Wl,-rpath,{libdir}", "-lpthread", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
