"""CPU-side checks of the drop-in boundary: libvx.so builds for sm_100a, loads,
and exports exactly what include/vx.h declares; error mapping; no CPU
fallback when there is no device."""

import os
import re
import subprocess

import numpy as np
import pytest

from paper_2407_02363_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "vx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vx_[a-z0-9_]+)\s*\(", src)))


def test_header_declarations_match_binding_table():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    L = _lib.load()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.vx_abi_version() == 2


def test_library_is_sm100a_code():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_scratch_sizing_is_pure_host():
    L = _lib.load()
    n = 64 * 64 * 64
    b = L.vx_edt_scratch_bytes(64, 64, 64, 1)
    assert b >= 8 * n
    assert L.vx_edt_scratch_bytes(64, 64, 64, 4) >= 4 * 8 * n
    assert L.vx_edt_s2_bytes(512, 512, 512) == 4
    assert L.vx_edt_s2_bytes(1, 46341, 46341) == 8


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) != "" and
                    _lib.load() and __import__("torch").cuda.is_available(),
                    reason="a CUDA device is present")
def test_no_cpu_fallback_without_device():
    from paper_2407_02363_b200 import pba_edt
    with pytest.raises(RuntimeError, match="no CUDA device|no CPU fallback"):
        pba_edt(np.zeros((4, 4, 4), bool))
