"""The C-ABI boundary, checked without a GPU.

* libswarmsim_b200.so loads and exports every function include/swarmsim_b200.h
  declares (and the ctypes binding declares exactly those);
* the ctypes struct mirrors have the C compiler's sizes and offsets
  (oracle/abi_layout prints them from the header);
* error codes map to the reference's exception types.
"""
import ctypes
import json
import re
import subprocess
from pathlib import Path

import pytest

from paper_2207_03530_b200 import _native as N
from paper_2207_03530_b200.errors import ContractViolation, UnknownScenario, UnsupportedShapePair

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "swarmsim_b200.h"


def header_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ss_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = header_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), f"{name} declared but not exported"
    assert sorted(N.exported_symbols()) == declared
    assert lib.ss_abi_version() == N.ABI_VERSION


def test_exported_symbols_are_plain_c():
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in header_functions():
        assert name in exported     # unmangled extern "C"


def test_ctypes_layout_matches_c_layout():
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "abi_layout"], check=True)
    c = json.loads(subprocess.run([str(ROOT / "oracle" / "abi_layout")], capture_output=True, text=True).stdout)
    for key, value in c.items():
        if key == "end":
            continue
        if "." in key:
            struct, field = key.split(".")
            assert getattr(getattr(N, struct), field).offset == value, key
        else:
            assert ctypes.sizeof(getattr(N, key)) == value, key


def test_error_mapping():
    with pytest.raises(ContractViolation):
        N.check(-1)
    with pytest.raises(UnsupportedShapePair):
        N.check(-2)
    with pytest.raises(UnknownScenario):
        N.check(-3)
    N.check(0)


def test_world_create_validates_descriptor_without_gpu():
    """Descriptor validation runs on the host before any device allocation."""
    d = N.SsWorldDesc()
    d.abi_version = N.ABI_VERSION + 7
    h = ctypes.c_void_p()
    with pytest.raises(ContractViolation, match="ABI version"):
        N.check(N.lib().ss_world_create(ctypes.byref(d), ctypes.byref(h)))
    d.abi_version = N.ABI_VERSION
    d.batch = 0
    with pytest.raises(ContractViolation, match="batch_size"):
        N.check(N.lib().ss_world_create(ctypes.byref(d), ctypes.byref(h)))


def test_sass_has_no_packed_fused_multiply_add():
    """The bit-exact contract forbids contracting a*b + c: ptxas fuses
    mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under -fmad=false, so the
    packed helpers (ss_internal.cuh) never chain them — checked on the SASS
    of the built library (scalar FFMA appears only in the explicit fma of the
    glibc expf / log1pf / sin-cos restatements)."""
    import shutil

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    assert "FMUL2" in sass or "FADD2" in sass          # the packed path is compiled in
    assert "FFMA2" not in sass
