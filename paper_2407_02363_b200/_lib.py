"""ctypes binding of libvx.so (include/vx.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2407_02363_b200/csrc``) and loaded from this package directory.  There
is no CPU fallback: a missing library or a missing CUDA device raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# VX_LIB: another build of the same library (tuning experiments, tools/variant_bench.sh)
LIB_PATH = os.environ.get("VX_LIB") or os.path.join(_HERE, "libvx.so")

VX_OK = 0
VX_EINVAL = -22
VX_ERANGE = -34
VX_ENOMEM = -12
VX_ENODEV = -19
VX_ECUDA = -1000

# every symbol include/vx.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "vx_abi_version", "vx_last_error", "vx_ctx_create", "vx_ctx_destroy", "vx_ctx_stream",
    "vx_ctx_synchronize", "vx_host_alloc", "vx_host_free", "vx_ctx_launches",
    "vx_grid_create", "vx_grid_destroy", "vx_grid_clear", "vx_grid_insert_points",
    "vx_grid_insert_points_device", "vx_grid_last_stats", "vx_grid_insert_voxel_sets",
    "vx_grid_read_cells", "vx_grid_write_cells", "vx_grid_occupancy", "vx_edt", "vx_edt_grid",
    "vx_line_nearest_sites", "vx_field_destroy", "vx_field_dims", "vx_field_read_site",
    "vx_field_site_at", "vx_field_site_world", "vx_edt_scratch_bytes", "vx_edt_device",
    "vx_edt_s2_bytes", "vx_edt_pass12_device", "vx_edt_pass3_device", "vx_cycle_create",
    "vx_cycle_destroy", "vx_cycle_step", "vx_cycle_wait", "vx_cycle_fields", "vx_cycle_grids",
    "vx_cycle_profile", "vx_cycle_phase_ms", "vx_cycle_step_device", "vx_edt_pass12_scatter",
    "vx_cycle_use_graph", "vx_grid_insert_points_ex", "vx_outlier_mask", "vx_cycle_set_avoidance",
    "vx_cycle_set_joint_frames", "vx_cycle_rows", "vx_cycle_prefetch", "vx_cycle_step_staged", "vx_cycle_info", "vx_brute_force_edt", "vx_field_create", "vx_edt_grid_into",
    "vx_grid_occupancy_digest", "vx_fields_site_world", "vx_ctx_transfer_bytes", "vx_site_world_slab", "vx_grid_occupied_voxels", "vx_field_sq_distance",
    "vx_field_dump_squared",
)
CYCLE_PHASES = ("h2d", "self_map", "mask_stamp_reset", "scatter", "edt_pass1", "edt_pass2",
                "edt_pass3", "gather")


class InsertStatsC(ctypes.Structure):
    _fields_ = [("inserted", ctypes.c_int64), ("outliers_removed", ctypes.c_int64),
                ("robot_skipped", ctypes.c_int64), ("out_of_bounds", ctypes.c_int64)]


class CycleResultC(ctypes.Structure):
    _fields_ = [("stats", InsertStatsC), ("self_recomputed", ctypes.c_int32)]


_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load libvx.so (raises LibraryMissing if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2407_02363_b200/csrc); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        PP = ctypes.POINTER(ctypes.c_void_p)
        i32, i64, f32, f64, sz = (ctypes.c_int, ctypes.c_int64, ctypes.c_float,
                                  ctypes.c_double, ctypes.c_size_t)
        sig = {
            "vx_abi_version": ([], i32),
            "vx_last_error": ([], ctypes.c_char_p),
            "vx_ctx_create": ([i32, PP], i32),
            "vx_ctx_destroy": ([P], i32),
            "vx_ctx_stream": ([P, PP], i32),
            "vx_ctx_synchronize": ([P], i32),
            "vx_host_alloc": ([sz, PP], i32),
            "vx_host_free": ([P], i32),
            "vx_ctx_launches": ([P], i64),
            "vx_grid_create": ([P, i32, i32, i32, f64, P, PP], i32),
            "vx_grid_destroy": ([P], i32),
            "vx_grid_clear": ([P], i32),
            "vx_grid_insert_points": ([P, P, i64, f32, f64, P, ctypes.POINTER(InsertStatsC)], i32),
            "vx_grid_insert_points_device": ([P, P, i64, f32, f64, P], i32),
            "vx_grid_last_stats": ([P, ctypes.POINTER(InsertStatsC)], i32),
            "vx_grid_insert_voxel_sets": ([P, i32, P, P, P, P, P, f32, P], i32),
            "vx_grid_read_cells": ([P, P], i32),
            "vx_grid_write_cells": ([P, P], i32),
            "vx_grid_occupancy": ([P, f64, P], i32),
            "vx_edt": ([P, P, i32, i32, i32, f64, PP], i32),
            "vx_edt_grid": ([P, f64, PP], i32),
            "vx_line_nearest_sites": ([P, P, i32, i32, i32, P], i32),
            "vx_field_destroy": ([P], i32),
            "vx_field_dims": ([P, P], i32),
            "vx_field_read_site": ([P, P], i32),
            "vx_field_site_at": ([P, i64, i64, i64, ctypes.POINTER(ctypes.c_int32)], i32),
            "vx_field_site_world": ([P, P, f64, P, i64, P, P, P], i32),
            "vx_edt_scratch_bytes": ([i32, i32, i32, i32], sz),
            "vx_edt_device": ([P, P, i32, i32, i32, i32, P, P, sz], i32),
            "vx_edt_s2_bytes": ([i32, i32, i32], i32),
            "vx_edt_pass12_device": ([P, P, i32, i32, i32, i32, P, P, sz], i32),
            "vx_edt_pass3_device": ([P, P, i32, i32, i32, i32, i32, P, P, sz], i32),
            "vx_edt_pass12_scatter": ([P, P, i32, i32, i32, i32, i32, P, P, ctypes.c_longlong, P, sz], i32),
            "vx_cycle_create": ([P, i32, i32, i32, f64, P, i32, P, P, P, f64, P, i32, i64, i32, PP], i32),
            "vx_cycle_destroy": ([P], i32),
            "vx_cycle_step": ([P, P, i64, P, f32, f64, P, i32, i32], i32),
            "vx_cycle_wait": ([P, ctypes.POINTER(CycleResultC), P, P, P], i32),
            "vx_cycle_fields": ([P, PP, PP], i32),
            "vx_cycle_grids": ([P, PP, PP, PP], i32),
            "vx_cycle_profile": ([P, i32], i32),
            "vx_cycle_use_graph": ([P, i32], i32),
            "vx_cycle_set_avoidance": ([P, i32, P, P, P, i32, f64, f64], i32),
            "vx_cycle_set_joint_frames": ([P, P, P], i32),
            "vx_cycle_rows": ([P, P, P, P, P, P], i32),
            "vx_cycle_prefetch": ([P, P, i64, P], i32),
            "vx_cycle_info": ([P, P], i32),
            "vx_brute_force_edt": ([P, P, i32, i32, i32, PP], i32),
            "vx_field_create": ([P, i32, i32, i32, PP], i32),
            "vx_edt_grid_into": ([P, f64, P], i32),
            "vx_grid_occupancy_digest": ([P, f64, P], i32),
            "vx_fields_site_world": ([P, P, P, f64, P, i64, P, P, P], i32),
            "vx_ctx_transfer_bytes": ([P, P], i32),
            "vx_site_world_slab": ([P, P, i32, i32, i32, i32, i32, P, f64, P, i64, P, P, P], i32),
            "vx_cycle_step_staged": ([P, ctypes.c_uint64, P, f32, f64, P, i32, i32], i32),
            "vx_grid_occupied_voxels": ([P, f64, P, i64, ctypes.POINTER(ctypes.c_int64)], i32),
            "vx_field_sq_distance": ([P, P, i32], i32),
            "vx_field_dump_squared": ([P, P, i64, ctypes.POINTER(ctypes.c_int64)], i32),
            "vx_grid_insert_points_ex": ([P, P, i64, f32, f64, P, i32, f64, ctypes.POINTER(InsertStatsC)], i32),
            "vx_outlier_mask": ([P, P, i64, i32, f64, P, ctypes.POINTER(ctypes.c_int64)], i32),
            "vx_cycle_step_device": ([P, P, i64, P, f32, f64, P, i32, i32], i32),
            "vx_cycle_phase_ms": ([P, P, ctypes.POINTER(ctypes.c_int)], i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a vx return code to the reference's exception types."""
    if rc == VX_OK:
        return
    msg = load().vx_last_error().decode(errors="replace")
    if rc == VX_EINVAL:
        raise ValueError(msg)
    if rc == VX_ERANGE:
        raise IndexError(msg)
    if rc == VX_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libvx error {rc}: {msg}")


def ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class Context:
    """One CUDA device + stream (vx_ctx)."""

    def __init__(self, device: int = 0):
        L = load()
        h = ctypes.c_void_p()
        check(L.vx_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = int(device)

    def stream_handle(self) -> int:
        s = ctypes.c_void_p()
        check(load().vx_ctx_stream(self.handle, ctypes.byref(s)))
        return int(s.value or 0)

    def synchronize(self) -> None:
        check(load().vx_ctx_synchronize(self.handle))

    def launches(self) -> int:
        return int(load().vx_ctx_launches(self.handle))

    def close(self) -> None:
        if self.handle:
            load().vx_ctx_destroy(self.handle)
            self.handle = None


_ctx_local = threading.local()


def default_context(device: int | None = None) -> Context:
    """Per-thread context on `device` (default: CUDA_DEVICE / LOCAL_RANK / 0)."""
    if device is None:
        device = int(os.environ.get("VX_DEVICE", "0"))
    ctxs = getattr(_ctx_local, "ctxs", None)
    if ctxs is None:
        ctxs = _ctx_local.ctxs = {}
    c = ctxs.get(device)
    if c is None:
        c = ctxs[device] = Context(device)
    return c


class PinnedArray:
    """numpy view on pinned host memory from vx_host_alloc (async H2D)."""

    def __init__(self, shape, dtype):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = ctypes.c_void_p()
        check(load().vx_host_alloc(max(1, self.nbytes), ctypes.byref(p)))
        self._p = p
        buf = (ctypes.c_char * max(1, self.nbytes)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        try:
            if self._p:
                load().vx_host_free(self._p)
                self._p = None
        except Exception:
            pass
