"""INTEGRATION.md option B: the ctypes stub a voxarm maintainer would add,
binding libvx.so directly (no shim), gives the reference's site array."""
import ctypes
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2407_02363_b200", "libvx.so")


def test_ctypes_stub_pba_edt():
    _L = ctypes.CDLL(LIB)
    P, PP = ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)
    _L.vx_ctx_create.argtypes = [ctypes.c_int, PP]
    _L.vx_edt.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, PP]
    _L.vx_field_read_site.argtypes = [P, P]
    _L.vx_field_destroy.argtypes = [P]
    _L.vx_ctx_destroy.argtypes = [P]
    _L.vx_last_error.restype = ctypes.c_char_p
    ctx = ctypes.c_void_p()
    assert _L.vx_ctx_create(0, ctypes.byref(ctx)) == 0, _L.vx_last_error()

    def pba_edt(occupancy, voxel_size=1.0):                              # edt.py:466
        occ = np.ascontiguousarray(occupancy, dtype=np.uint8)
        f = ctypes.c_void_p()
        assert _L.vx_edt(ctx, occ.ctypes.data_as(P), *occ.shape, voxel_size, ctypes.byref(f)) == 0
        site = np.empty(occ.shape, np.int32)
        assert _L.vx_field_read_site(f, site.ctypes.data_as(P)) == 0
        _L.vx_field_destroy(f)
        return site

    rng = np.random.default_rng(11)
    for dims in [(40, 33, 28), (64, 64, 64)]:
        occ = rng.random(dims) < 0.01
        assert np.array_equal(pba_edt(occ), O.pba_edt_site(occ))
    # error path: a non-3D extent of zero -> VX_EINVAL (-22) and a message
    f = ctypes.c_void_p()
    rc = _L.vx_edt(ctx, None, 0, 4, 4, 1.0, ctypes.byref(f))
    assert rc != 0 and _L.vx_last_error()
    _L.vx_ctx_destroy(ctx)
