"""The C-ABI boundary (include/gpcx.h) without a GPU: the library loads,
exports every declared symbol, sizes requests exactly like the reference's
dim_product rules, maps statuses onto gpc::Errc / ERR:<CODE>, and refuses to
compute without a device (no CPU fallback)."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1505_05655_b200 as G
from paper_1505_05655_b200 import _lib
from conftest import has_gpu

HEADER = Path(__file__).resolve().parent.parent / "include" / "gpcx.h"


def test_every_declared_symbol_is_exported():
    text = HEADER.read_text()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(gpcx_\w+)\s*\(", text, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS)
    lib = C.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name


def test_abi_version_and_flags():
    assert G.lib.gpcx_abi_version() == 2
    assert G.flags() == ["BAYER_BILINEAR", "BAYER_GRADIENT", "DEVINFO", "LSQ_POLYFIT", "LUT_APPLY",
                         "LUT_CORRECT", "LUT_GEN", "MATMUL"]
    assert G.required_params("LSQ_POLYFIT") == ["lines", "pixels", "order"]
    assert G.required_params("DEVINFO") == []
    assert G.required_params("BAYER_GRADIENT") == ["rows", "cols"]
    assert G.required_params("LUT_CORRECT") == ["rows", "cols"]
    assert G.required_params("MATMUL") == ["m", "k", "n"]


def test_status_names_follow_errc_order():
    for i, name in enumerate(_lib.ERRC_NAMES):
        assert G.lib.gpcx_status_name(i + 1).decode() == name
    assert G.lib.gpcx_status_name(0).decode() == "OK"
    codes = {n: G.lib.gpcx_response_code(s).decode() for n, s in _lib.STATUS.items()}
    assert codes["UnknownTask"] == "UNKNOWN_TASK"
    assert codes["MissingParam"] == "MISSING_PARAM"
    assert codes["PayloadMismatch"] == "PAYLOAD_MISMATCH"
    assert codes["Overflow"] == codes["TooLarge"] == "TOO_LARGE"
    for n in ("FieldTooLong", "InvalidCharacter", "BadMarker", "MalformedPadding", "DuplicateKey",
              "BadToken", "BadValue"):
        assert codes[n] == "BAD_HEADER"
    assert codes["TaskFailed"] == codes["Singular"] == "TASK_FAILED"


@pytest.mark.parametrize("flag,params,want", [
    ("LUT_GEN", "rows=4096,cols=4096", 33554432),
    ("LUT_CORRECT", "rows=4096,cols=4096,mode=stretch", 33554432),
    ("LUT_APPLY", "rows=2048,cols=2048", 131072 + 8388608),
    ("MATMUL", "m=4096,k=4096,n=4096", 134217728),
    ("MATMUL", "m=3,k=5,n=7,prec=bf16", (15 + 35) * 4),
    ("LUT_CORRECT", "rows=16384,cols=32768", 1 << 30),  # exactly the cap
])
def test_payload_len(flag, params, want):
    assert G.payload_len(flag, params) == want


@pytest.mark.parametrize("flag,params,code", [
    ("LUT_GEN", "rows=4", "MissingParam"),
    ("LUT_GEN", "rows=0,cols=4", "BadValue"),
    ("LUT_GEN", "rows=x,cols=4", "BadValue"),
    ("LUT_GEN", "rows=4,cols=4,dtype=f32", "BadValue"),
    ("LUT_GEN", "rows=4,cols=4,mode=gamma", "BadValue"),
    ("LUT_GEN", "rows=32768,cols=32768", "Overflow"),
    ("LUT_APPLY", "rows=16384,cols=32768", "Overflow"),  # cap + LUT
    ("MATMUL", "m=4,k=4,n=4,prec=f16", "BadValue"),
    ("MATMUL", "m=16384,k=16384,n=16384", "Overflow"),
    ("NOPE", "rows=4,cols=4", "UnknownTask"),
    ("LUT_GEN", "rows=4,,cols=4", "BadToken"),
    ("LUT_GEN", "rows=4,rows=4", "DuplicateKey"),
])
def test_payload_len_errors(flag, params, code):
    with pytest.raises(G.GpcxError) as e:
        G.payload_len(flag, params)
    assert e.value.code == code


def test_payload_rules_agree_with_reference_side_descriptors(refl):
    """The reference-registered oracle descriptors (oracle/ref_shim.cpp) and
    libgpcx size every request identically, including the failures."""
    cases = ["rows=4096,cols=4096", "rows=1,cols=1", "rows=0,cols=3", "rows=32768,cols=32768",
             "rows=16384,cols=32768", "rows=3,cols=3,dtype=u8", "rows=3,cols=3,mode=stretch",
             "m=5,k=7,n=9", "m=5,k=7,n=9,prec=tf32", "m=16384,k=16384,n=2", "m=1,k=0,n=1"]
    for flag in ("LUT_GEN", "LUT_APPLY", "LUT_CORRECT", "MATMUL"):
        for params in cases:
            n = C.c_uint64(0)
            rs = refl.ref.ref_expected_payload_len(flag.encode(), params.encode(), C.byref(n))
            try:
                ours = G.payload_len(flag, params)
                assert rs == 0, (flag, params)
                assert ours == n.value, (flag, params)
            except G.GpcxError as e:
                assert rs == e.status, (flag, params, rs, e.code)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    img = np.zeros(16, dtype=np.uint16)
    with pytest.raises(G.GpcxError) as e:
        G.run("LUT_CORRECT", "rows=4,cols=4", img)
    assert e.value.code == "TaskFailed"


def test_lut_workspace_size_includes_the_residual_plane():
    """gpcx_lut_workspace_size(n): the fixed part below 2^25 samples; from
    2^25 on plus the residual plane (u32 base per 512-sample block, 256-byte
    rounded, and 512 residual bytes per block -- DESIGN.md §4)."""
    def size(n):
        nb = C.c_uint64(0)
        assert G.lib.gpcx_lut_workspace_size(n, C.byref(nb)) == 0
        return nb.value
    fixed = size(1)
    assert size((1 << 25) - 1) == fixed
    for n in (1 << 25, (1 << 25) + 511, 1 << 30, (1 << 32) - 1):
        blocks = n >> 9
        assert size(n) == fixed + ((blocks * 4 + 255) & ~255) + blocks * 512, n
    nb = C.c_uint64(0)
    assert G.lib.gpcx_lut_workspace_size(1 << 32, C.byref(nb)) != 0  # n must fit u32
