"""CPU checks of the drop-in boundary: the C-ABI library builds for sm_100a,
loads, and exports every symbol include/rapid_b200.h declares (no compute
calls — there is no GPU here); ops refuse CPU tensors (no fallback)."""

import ctypes
import os
import re

import pytest

from paper_2601_11822_b200 import ops
from paper_2601_11822_b200.build import build, lib_path

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "rapid_b200.h")


def declared_symbols():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^(?:const char\*|int)\s+(rb_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    build()
    return ctypes.CDLL(str(lib_path()))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "rb_gemm_bf16" in syms and "rb_decode_attention" in syms and "rb_green_split" in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_ops_binding_covers_header():
    assert set(declared_symbols()) <= set(ops.EXPORTED_SYMBOLS)


def test_version_string(lib):
    ops.load()
    assert b"sm_100a" in ops.load().rb_version()


def test_sass_uses_tcgen05_and_tma():
    """The GEMM is tensor-core gen-5 (UTCHMMA) fed by TMA (UTMALDG); decode attention uses TMA too."""
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump unavailable")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([exe, "-sass", str(lib_path())], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass
    assert "UTMALDG" in sass
    assert "LDTM" in sass


def test_ops_reject_cpu_tensors():
    import torch

    x = torch.zeros(4, 64, dtype=torch.bfloat16)
    w = torch.zeros(64, 64, dtype=torch.bfloat16)
    with pytest.raises(RuntimeError, match="CUDA tensors only"):
        ops.linear(x, w)
