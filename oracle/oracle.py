"""CPU ORACLE wrapper -- test infrastructure only.

ctypes bindings to ``oracle/_build/libvx_oracle.so`` (vx_oracle.c), a plain-C
restatement of the reference CPU path (voxarm edt.py / grids.py /
engine.py).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product package (``paper_2407_02363_b200``) never imports it and has no CPU
fallback.

Each wrapper names the reference function it restates; the C file cites the
exact lines.  ``brute_force_edt`` and ``proximate_sites_1d`` are small numpy /
pure-Python restatements used as independent checks (edt.py:487-508, 55-100).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libvx_oracle.so")
_lib = None

NO_SITE = -1
L_MIN = -2.0
L_MAX = 3.5


def build() -> str:
    """Compile the oracle (make -C oracle); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int, ctypes.c_int64
        L.vxo_sweep_lines.argtypes = [P, i32, i32, i32, i32, P, i32]
        L.vxo_slice_transform.argtypes = [P, i32, i32, i32, i32, i32, P, P, i32]
        L.vxo_column_transform.argtypes = [P, P, i32, i32, i32, i32, i32, P, i32]
        L.vxo_column_transform_slab.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, P, i32]
        L.vxo_pba_edt.argtypes = [P, i32, i32, i32, i32, i32, i32, P, i32]
        L.vxo_pba_edt.restype = i32
        L.vxo_insert_points.argtypes = [P, P, ctypes.c_double, P, P, i64, P,
                                        ctypes.c_float, ctypes.c_float, P, P]
        L.vxo_stamp_voxels.argtypes = [P, P, ctypes.c_double, P, P, i64, P,
                                       ctypes.c_double, P, ctypes.c_float]
        L.vxo_stamp_voxels.restype = i64
        L.vxo_site_world.argtypes = [P, P, ctypes.c_double, P, P, i64, P, P, P]
        L.vxo_max_threads.restype = i32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def max_threads() -> int:
    return int(lib().vxo_max_threads())


def _occ(occupancy) -> np.ndarray:
    """edt.py:455-463 (_as_occ)."""
    occ = np.ascontiguousarray(occupancy)
    if occ.ndim != 3:
        raise ValueError("occupancy must be a 3D array")
    if max(occ.shape) > (1 << 20):
        raise ValueError("grid extent too large for integer-exact transform")
    if occ.dtype != np.uint8:
        occ = occ.astype(np.uint8)
    return occ


def line_nearest_sites(occupancy, m1: int = 1, workers: int = 0) -> np.ndarray:
    """edt.py:444-452 -> pass 1 (edt.py:168-224)."""
    occ = _occ(occupancy)
    s1 = np.empty(occ.shape, np.int32)
    lib().vxo_sweep_lines(_ptr(occ), *occ.shape, int(m1), _ptr(s1), int(workers))
    return s1


def slice_transform(s1z: np.ndarray, m2: int = 1, m3: int = 2, workers: int = 0):
    """edt.py:227-317 (pass 2) -> (s2y, s2z)."""
    s1z = np.ascontiguousarray(s1z, dtype=np.int32)
    s2y = np.empty(s1z.shape, np.int32)
    s2z = np.empty(s1z.shape, np.int32)
    lib().vxo_slice_transform(_ptr(s1z), *s1z.shape, int(m2), int(m3), _ptr(s2y),
                              _ptr(s2z), int(workers))
    return s2y, s2z


def column_transform_slab(s2y: np.ndarray, s2z: np.ndarray, j0: int, ny_total: int,
                          m2: int = 1, m3: int = 2, workers: int = 0) -> np.ndarray:
    """edt.py:320-420 on a j-slab (nx, nyl, nz) holding global rows j0.. of a
    grid with ny_total rows (test support for the slab-decomposed path)."""
    s2y = np.ascontiguousarray(s2y, dtype=np.int32)
    s2z = np.ascontiguousarray(s2z, dtype=np.int32)
    site = np.empty(s2y.shape, np.int32)
    lib().vxo_column_transform_slab(_ptr(s2y), _ptr(s2z), *s2y.shape, int(j0), int(ny_total),
                                    int(m2), int(m3), _ptr(site), int(workers))
    return site


def pba_edt_site(occupancy, m1: int = 1, m2: int = 1, m3: int = 2,
                 workers: int = 0) -> np.ndarray:
    """edt.py:466-484: the int32 site array (flat nearest-site index)."""
    occ = _occ(occupancy)
    site = np.empty(occ.shape, np.int32)
    if lib().vxo_pba_edt(_ptr(occ), *occ.shape, int(m1), int(m2), int(m3),
                         _ptr(site), int(workers)) != 0:
        raise MemoryError("oracle scratch allocation failed")
    return site


def brute_force_site(occupancy) -> np.ndarray:
    """edt.py:487-508: exhaustive min, lexicographic ties (small grids)."""
    occ = _occ(occupancy)
    nx, ny, nz = occ.shape
    sites = np.argwhere(occ != 0).astype(np.int64)
    if sites.shape[0] == 0:
        return np.full(occ.shape, NO_SITE, np.int32)
    lin = ((sites[:, 0] * ny + sites[:, 1]) * nz + sites[:, 2]).astype(np.int32)
    vox = np.indices(occ.shape, dtype=np.int64).reshape(3, -1).T
    out = np.empty(vox.shape[0], np.int32)
    chunk = max(1, int(64e6) // (sites.shape[0] * 24))
    for lo in range(0, vox.shape[0], chunk):
        d = vox[lo:lo + chunk, None, :] - sites[None, :, :]
        out[lo:lo + chunk] = lin[np.argmin((d * d).sum(axis=2), axis=1)]
    return out.reshape(occ.shape)


def sq_distance_grid(site: np.ndarray) -> np.ndarray:
    """DistanceField.sq_distance_grid, edt.py:123-135."""
    _, ny, nz = site.shape
    flat = site.reshape(-1).astype(np.int64)
    out = np.full(flat.shape, -1, dtype=np.int64)
    ok = flat != NO_SITE
    if ok.any():
        vox = np.arange(flat.shape[0], dtype=np.int64)[ok]
        s = flat[ok]
        out[ok] = ((vox // (ny * nz) - s // (ny * nz)) ** 2
                   + ((vox // nz) % ny - (s // nz) % ny) ** 2
                   + (vox % nz - s % nz) ** 2)
    return out.reshape(site.shape)


def _dominated(ya, wa, yb, wb, yc, wc) -> bool:
    """edt.py:70-73."""
    return (wb + yb * yb - wa - ya * ya) * (yc - yb) >= (wc + yc * yc - wb - yb * yb) * (yb - ya)


def proximate_sites_1d(sites, column: int) -> list:
    """edt.py:76-100, returning the surviving site list."""
    coords, weights, payload = [], [], []
    last = None
    for coord, site in sites:
        coord = int(coord)
        if last is not None and coord <= last:
            raise ValueError("sites must be strictly increasing in sweep coordinate")
        last = coord
        w = (int(site[0]) - int(column)) ** 2
        while len(coords) >= 2 and _dominated(coords[-2], weights[-2], coords[-1],
                                               weights[-1], coord, w):
            coords.pop(); weights.pop(); payload.pop()
        coords.append(coord); weights.append(w); payload.append(site)
    return payload


def logit(p: float) -> float:
    """grids.py:24-25."""
    return math.log(p / (1.0 - p))


def insert_points(cells: np.ndarray, voxel_size: float, origin, world_pts,
                  mask_cells=None, occupancy_threshold: float = 0.5,
                  hit_logodds: float = 0.85):
    """VoxelGrid.insert_point_cloud with k_neighbors=0 (grids.py:149-188) on
    already-transformed world points.  cells is modified in place.
    Returns (inserted, robot_skipped, out_of_bounds)."""
    assert cells.dtype == np.float32 and cells.flags.c_contiguous
    dims = np.asarray(cells.shape, dtype=np.int32)
    org = np.ascontiguousarray(origin, dtype=np.float64).reshape(3)
    pts = np.ascontiguousarray(world_pts, dtype=np.float64).reshape(-1, 3)
    stats = np.zeros(3, np.int64)
    if pts.shape[0] == 0:
        return 0, 0, 0
    counts = np.zeros(cells.size, np.int32)
    mask = None if mask_cells is None else np.ascontiguousarray(mask_cells, np.float32)
    lib().vxo_insert_points(_ptr(cells), _ptr(dims), float(voxel_size), _ptr(org),
                            _ptr(pts), pts.shape[0],
                            None if mask is None else _ptr(mask),
                            float(np.float32(logit(occupancy_threshold))),
                            float(np.float32(hit_logodds)), _ptr(counts), _ptr(stats))
    return int(stats[0]), int(stats[1]), int(stats[2])


def stamp_voxels(cells: np.ndarray, voxel_size: float, origin, indices,
                 set_origin, set_voxel_size: float, transform=None,
                 value: float = L_MAX) -> int:
    """VoxelGrid.insert_voxel_set (grids.py:190-203); returns the OOB count."""
    dims = np.asarray(cells.shape, dtype=np.int32)
    org = np.ascontiguousarray(origin, dtype=np.float64).reshape(3)
    ijk = np.ascontiguousarray(indices, dtype=np.int32).reshape(-1, 3)
    lorg = np.ascontiguousarray(set_origin, dtype=np.float64).reshape(3)
    T = None if transform is None else np.ascontiguousarray(transform, np.float64).reshape(4, 4)
    return int(lib().vxo_stamp_voxels(_ptr(cells), _ptr(dims), float(voxel_size),
                                      _ptr(org), _ptr(ijk), ijk.shape[0], _ptr(lorg),
                                      float(set_voxel_size),
                                      None if T is None else _ptr(T), float(value)))


def site_world(site: np.ndarray, voxel_size: float, origin, centers):
    """SimEngine._site_world (engine.py:212-221) for many centres plus the
    tasks.py:102-104 distance.  Returns (site_lin, world (S,3), dist)."""
    dims = np.asarray(site.shape, dtype=np.int32)
    org = np.ascontiguousarray(origin, dtype=np.float64).reshape(3)
    c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    lin = np.empty(c.shape[0], np.int32)
    world = np.empty((c.shape[0], 3), np.float64)
    dist = np.empty(c.shape[0], np.float64)
    st = np.ascontiguousarray(site, np.int32)
    lib().vxo_site_world(_ptr(st), _ptr(dims), float(voxel_size), _ptr(org), _ptr(c),
                         c.shape[0], _ptr(lin), _ptr(world), _ptr(dist))
    return lin, world, dist
