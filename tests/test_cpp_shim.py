"""The C++ host API (include/irismpc_b200.hpp) compiles, and on a B200 the
3-thread per-party drop-in matches the oracle (tests/cpp/shim_parity.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
SRC = os.path.join(ROOT, "tests", "cpp", "shim_parity.cpp")


def _build(out):
    cmd = [GXX, "-O1", "-std=c++20", "-pthread", "-I" + os.path.join(ROOT, "include"), "-I" + CUDA + "/include", SRC,
           "-L" + os.path.join(ROOT, "paper_2405_04463_b200"), "-lirismpc_gpu",
           "-L" + os.path.join(ROOT, "oracle"), "-loracle",
           "-L" + CUDA + "/lib64", "-lcudart",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2405_04463_b200"), "-Wl,-rpath," + os.path.join(ROOT, "oracle"),
           "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_shim_header_compiles(tmp_path):
    subprocess.run([GXX, "-std=c++20", "-fsyntax-only", "-I" + os.path.join(ROOT, "include"), "-I" + CUDA + "/include",
                    SRC], check=True)
    _build(str(tmp_path / "shim"))


@pytest.mark.gpu
def test_cpp_three_party_dropin_matches_oracle(tmp_path):
    exe = str(tmp_path / "shim")
    _build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim ok" in r.stdout
