"""CPU-side checks of the product library: it is built for sm_100a, loads,
exports every entry point include/rtlm.h declares, and refuses to run without
a GPU (no CPU fallback).  No compute calls here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rtlm.h")).read()
    return sorted(set(re.findall(r"^\s*(?:rt_status|const char\*|int|uint32_t|uint64_t)\s+(rt_\w+)\s*\(", src, re.M)))


def test_library_exports_header_symbols():
    from paper_2309_06619_b200 import _build, EXPORTS
    lib_path = _build.build()
    lib = ctypes.CDLL(lib_path)
    syms = header_symbols()
    assert len(syms) >= 13
    assert sorted(EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s
    lib.rt_abi_version.restype = ctypes.c_int
    assert lib.rt_abi_version() == 1


def test_library_is_sm100a():
    from paper_2309_06619_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch
    import paper_2309_06619_b200 as rt
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rt.RtlmError, match="no CUDA device"):
        rt.Context("vague:\nstuff\n")


def test_product_does_not_touch_oracle():
    """The product package never imports, links or calls oracle/ (DESIGN §3)."""
    pkg = os.path.join(ROOT, "paper_2309_06619_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "liboracle" not in txt and "rtlm_oracle" not in txt, f
