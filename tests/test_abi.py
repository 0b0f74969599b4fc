"""CPU-side checks of the C-ABI library: it builds, loads without a GPU and
exports every entry point include/irismpc_gpu.h declares (no compute calls)."""
import ctypes
import os
import re

import pytest

import paper_2405_04463_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "irismpc_gpu.h")).read()
    return sorted(set(re.findall(r"\b(irismpc_gpu_[a-z_0-9]+)\s*\(", src)))


def test_header_and_python_binding_agree():
    assert _declared() == sorted(P.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = P.lib()
    for name in _declared():
        assert hasattr(L, name), name


def test_pure_host_entry_points():
    from oracle import pyoracle as O
    # seeds_from_master == deal_seeds of run_parties (reference-pinned oracle)
    assert bytes(P.seeds_from_master(7)) == bytes(O.party_seeds(7))
    assert P.record_bytes(P.SHAMIR, 12800) == O.record_bytes(O.SHAMIR, 12800)
    assert P.record_bytes(P.REPLICATED, 64) == O.record_bytes(O.REPLICATED, 64)
    for var in (P.PLAIN_MASK, P.MPC_LIFT, P.CONST_LIFT, P.NO_LIFT):
        for be in (P.SHAMIR, P.REPLICATED):
            for l in (8, 64, 12800):
                assert P.record_bytes(be, l, var) == O.record_bytes(be, l, var), (var, be, l)
    for persons, s, r, m in [(16, 100_000, 31, False), (1, 10, 1, True), (3, 0, 31, False)]:
        assert P.lane_count(persons, s, r, m) == O.lib().orc_lane_count(persons, s, r, 1 if m else 0)
    for ratio in (0.375, 0.3, 0.2, 0.0, 0.5):
        assert P.match_a(ratio) == O.lib().orc_match_a(ratio)


def test_bounds_rejected_before_device():
    # EngineConfig::validate: Shamir needs an even rotation stride (l/64)
    with pytest.raises(P.BoundsError):
        P.Session(P.EngineConfig(backend=P.SHAMIR, l=192, rotations=3), master_seed=1)
    with pytest.raises(P.BoundsError):
        P.Session(P.EngineConfig(backend=P.SHAMIR, l=64, rotations=2), master_seed=1)
    with pytest.raises(P.BoundsError):
        P.Session(P.EngineConfig(backend=P.REPLICATED, l=12), master_seed=1)
    # plain-mask: check_public_mask_bound(l, 16) needs l < 2^14 (iris.hpp:189-194)
    with pytest.raises(P.BoundsError):
        P.Session(P.EngineConfig(backend=P.SHAMIR, l=16384, rotations=1, variant=P.PLAIN_MASK), master_seed=1)
    # shared-mask variants fix m = 16 (engine.cpp:26)
    with pytest.raises(P.BoundsError):
        P.Session(P.EngineConfig(backend=P.SHAMIR, l=64, rotations=1, variant=P.NO_LIFT, m=15), master_seed=1)
    # oracle agrees on the same configs
    from oracle import pyoracle as O
    assert O.lib().orc_validate(O.make_config(O.SHAMIR, 16384, 0.375, 1, variant=O.PLAIN_MASK)) == 4
    assert O.lib().orc_validate(O.make_config(O.SHAMIR, 16376, 0.375, 1, variant=O.PLAIN_MASK)) == 0


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is not None and False, reason="")
def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.DeviceError):
        P.Session(P.EngineConfig(backend=P.SHAMIR, l=64, rotations=1), master_seed=1)


def test_header_compiles_as_c_and_links():
    """include/irismpc_gpu.h is plain C (a cgo / JNI / ctypes binding sees only
    C types): a C11 program that names every entry point compiles and links
    against the library without CUDA headers."""
    import re
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hdr = open(os.path.join(root, "include", "irismpc_gpu.h")).read()
    names = sorted(set(re.findall(r"\b(irismpc_gpu_[a-z0-9_]+)\s*\(", hdr)))
    src = "#include <stdio.h>\n#include \"irismpc_gpu.h\"\nint main(void) {\n  void* p[] = {\n"
    src += ",\n".join(f"    (void*)&{n}" for n in names) + "\n  };\n"
    src += "  printf(\"%d\\n\", (int)(sizeof(p) / sizeof(p[0])));\n  return 0;\n}\n"
    gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        pkg = os.path.join(root, "paper_2405_04463_b200")
        subprocess.run([gcc, "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(root, "include"), c, "-L" + pkg,
                        "-lirismpc_gpu", "-Wl,-rpath," + pkg, "-o", exe], check=True, capture_output=True, text=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
        assert int(out) == len(names) > 40
