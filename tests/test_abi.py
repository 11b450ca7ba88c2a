"""CPU checks of the drop-in boundary (no compute calls: no GPU here).

* the native library builds for sm_100a and loads;
* it exports every entry point declared in include/hsgn_b200.h, and the
  ctypes binding (paper_2601_02540_b200/_native.py) declares exactly those;
* the SASS is sm_100a and obeys the parity contract (no FMA outside the
  division / reciprocal sequences is checked on the GPU by bitwise tests;
  here we check the build flags and the architecture);
* the product package never imports the oracle (test infrastructure).
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hsgn_b200.h")
PKG = os.path.join(ROOT, "paper_2601_02540_b200")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hsgn_[a-z0-9_]+)\s*\(", text)) - {"hsgn_observer"})


@pytest.fixture(scope="module")
def lib():
    from paper_2601_02540_b200 import _native
    return _native.lib()


def test_library_loads_and_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_matches_header():
    from paper_2601_02540_b200 import _native
    assert sorted(_native.EXPORTS) == declared_symbols()


def test_build_info_and_arch(lib):
    assert b"sm_100a" in lib.hsgn_build_info()
    so = os.path.join(PKG, "_native", "libhsgn_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_build_flags_are_parity_safe():
    from paper_2601_02540_b200 import build
    assert "--fmad=false" in build.FLAGS
    assert build.ARCH == ["-gencode", "arch=compute_100a,code=sm_100a"]


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle_lib" not in src and "liboracle" not in src and "libhsgn_ref" not in src, f


def test_no_batched_memcpy_calls():
    """B200 driver issue (B200_PROFILING.md): never use the batched memcpy APIs."""
    bad = re.compile(r"cu(da)?Memcpy(3D)?BatchAsync")
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".cu", ".cuh", ".cpp", ".h", ".py")):
                assert not bad.search(open(os.path.join(dirpath, f)).read()), f


def test_status_codes_match_header():
    from paper_2601_02540_b200 import _native as N
    text = open(HEADER).read()
    for name, val in [("HSGN_OK", 0), ("HSGN_EINVAL", 1), ("HSGN_EDEPTH", 2), ("HSGN_ECUDA", 3), ("HSGN_ENCCL", 4)]:
        assert re.search(rf"{name}\s*=\s*{val}\b", text)
        assert getattr(N, name) == val


def test_struct_layouts_match_header():
    from paper_2601_02540_b200 import _native as N
    assert ctypes.sizeof(N.hsgn_grid) == 4 * 4 + 4 * 8
    assert ctypes.sizeof(N.hsgn_phys) == 3 * 8
    assert ctypes.sizeof(N.hsgn_cfg) == 10 * 8
    assert ctypes.sizeof(N.hsgn_record) == 8 + 4 * 8 + 4 + 256 + 4  # trailing pad to 8
    assert ctypes.sizeof(N.hsgn_scenario) == 32 + 48 + 4 * 8 + 8 * 4 + 2 * 4 + 16 * 8 + 8 * 8 + 2 * 4 + 24 * 8


def test_host_api_validation_without_gpu():
    """make_grid validation mirrors grid.hpp:51-55 (host-only)."""
    import paper_2601_02540_b200 as H
    with pytest.raises(ValueError, match="increasing"):
        H.make_grid(1.0, 0.0, 0.0, 1.0, 8, 8)
    with pytest.raises(ValueError, match="at least 4"):
        H.make_grid(0.0, 1.0, 0.0, 1.0, 3, 8)
    g = H.make_grid(-1.0, 1.0, -1.0, 1.0, 8, 9, H.BoundaryKind.periodic, H.BoundaryKind.bounded)
    assert g.dx == 0.25 and g.dy == 0.25
    assert H.eoc(0.1, 0.025, 1.0, 0.5) == pytest.approx(2.0)
