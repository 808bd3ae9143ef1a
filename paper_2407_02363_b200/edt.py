"""Drop-in for voxarm.edt (pkg/src/voxarm/edt.py) backed by the sm_100a EDT.

Same names, signatures, results and exceptions as the reference:
  pba_edt             edt.py:466-484  -> vx_edt (K3 -> K4 -> K5 on the GPU)
  line_nearest_sites  edt.py:444-452  -> vx_line_nearest_sites (K3)
  DistanceField       edt.py:103-145  -> device site array, host copy on demand
  query_nearest_site  edt.py:148-161
  BandConfig / default_band_config edt.py:32-52 (validated; the GPU band
  layout is chosen per shape -- the result is band-invariant, test_edt.py:88-95)
  brute_force_edt     edt.py:487-508  -> vx_brute_force_edt (exhaustive, on the GPU)
  ProximateStack / proximate_sites_1d  edt.py:55-100 (host API helpers for
  one column's surviving sites; the GPU passes never call them)
The site array is bit-identical to the reference's (lexicographic
minimum nearest site).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib

NO_SITE = -1
_MAX_EXTENT = 1 << 20  # edt.py:29


@dataclass(frozen=True)
class BandConfig:
    """Band counts for the three passes (edt.py:32-47).  Accepted and
    validated for API parity; results do not depend on them."""

    m1: int = 1
    m2: int = 1
    m3: int = 2

    def __post_init__(self) -> None:
        if min(self.m1, self.m2, self.m3) < 1:
            raise ValueError("band counts must be positive")


def default_band_config(workers: int | None = None) -> BandConfig:
    """edt.py:50-52 (worker count defaults to os.cpu_count instead of numba's)."""
    w = max(1, int(workers) if workers else (os.cpu_count() or 1))
    return BandConfig(m1=w, m2=w, m3=2 * w)


def _check_workers(workers) -> None:
    if workers is not None and workers < 1:     # edt.py:432-433
        raise ValueError("workers must be positive")


def _as_occ(occupancy) -> np.ndarray:
    """edt.py:455-463."""
    occ = np.ascontiguousarray(occupancy)
    if occ.ndim != 3:
        raise ValueError("occupancy must be a 3D array")
    if max(occ.shape) > _MAX_EXTENT:
        raise ValueError("grid extent too large for integer-exact transform")
    if occ.dtype != np.uint8:
        occ = occ.astype(np.uint8)
    return occ


class DistanceField:
    """Per-voxel nearest occupied voxel as flat int32 indices (edt.py:103-145).

    Built either from a host ``site`` array (reference constructor) or from a
    device field returned by the GPU EDT; in the latter case ``site`` is
    copied to the host on first access only.
    """

    def __init__(self, site: np.ndarray | None, voxel_size: float, *, _handle=None, _dims=None,
                 _ctx=None, _owned=True):
        if site is not None:
            if site.ndim != 3:
                raise ValueError("site array must be 3D")
            self._site = site
            self.dims = site.shape
        else:
            self._site = None
            self.dims = tuple(int(d) for d in _dims)
        self.voxel_size = float(voxel_size)
        self._handle = _handle
        self._ctx = _ctx
        self._owned = _owned

    # -- device side --------------------------------------------------------
    @property
    def device_handle(self):
        return self._handle

    @property
    def site(self) -> np.ndarray:
        if self._site is None:
            out = np.empty(self.dims, np.int32)
            _lib.check(_lib.load().vx_field_read_site(self._handle, _lib.ptr(out)))
            self._site = out
        return self._site

    @site.setter
    def site(self, value) -> None:
        self._site = value

    def __del__(self):
        try:
            if self._handle is not None and self._owned:
                _lib.load().vx_field_destroy(self._handle)
                self._handle = None
        except Exception:
            pass

    # -- reference methods ----------------------------------------------------
    def _site_lin(self, i, j, k) -> int:
        if self._site is not None or self._handle is None:
            return int(self.site[i, j, k])
        out = ctypes.c_int32()
        _lib.check(_lib.load().vx_field_site_at(self._handle, int(i), int(j), int(k),
                                                ctypes.byref(out)))
        return int(out.value)

    def site_index(self, index) -> tuple[int, int, int] | None:
        """edt.py:113-121."""
        i, j, k = index
        nx, ny, nz = self.dims
        if self._site is None and self._handle is not None:
            # numpy indexing semantics (negative wrap) for the single lookup
            i, j, k = (int(v) + d if int(v) < 0 else int(v) for v, d in zip((i, j, k), self.dims))
            if not (0 <= i < nx and 0 <= j < ny and 0 <= k < nz):
                raise IndexError(f"index {index} out of bounds for shape {self.dims}")
        lin = self._site_lin(i, j, k)
        if lin == NO_SITE:
            return None
        return lin // (ny * nz), (lin // nz) % ny, lin % nz

    def _device_only(self) -> bool:
        # the host copy, once materialised, may have been edited in place:
        # from then on it is the source of truth (as _site_lin treats it)
        return self._site is None and self._handle is not None

    def sq_distance_grid(self) -> np.ndarray:
        """edt.py:123-135 (export format; int64, -1 where there is no site).
        Computed on the device (vx_field_sq_distance) for a device field."""
        if self._device_only():
            out = np.empty(self.dims, np.int64)
            _lib.check(_lib.load().vx_field_sq_distance(self._handle, _lib.ptr(out), 0))
            return out
        _, ny, nz = self.dims
        flat = self.site.reshape(-1).astype(np.int64)
        out = np.full(flat.shape, -1, dtype=np.int64)
        ok = flat != NO_SITE
        if ok.any():
            vox = np.arange(flat.shape[0], dtype=np.int64)[ok]
            site = flat[ok]
            vi, vj, vk = vox // (ny * nz), (vox // nz) % ny, vox % nz
            si, sj, sk = site // (ny * nz), (site // nz) % ny, site % nz
            out[ok] = (vi - si) ** 2 + (vj - sj) ** 2 + (vk - sk) ** 2
        return out.reshape(self.dims)

    def dump_squared(self, stream) -> None:
        """edt.py:137-145 (golden-file text format).  A device field is
        formatted on the device (vx_field_dump_squared) and written once."""
        if self._device_only():
            L = _lib.load()
            n = ctypes.c_int64()
            _lib.check(L.vx_field_dump_squared(self._handle, None, 0, ctypes.byref(n)))
            buf = ctypes.create_string_buffer(max(1, n.value))
            _lib.check(L.vx_field_dump_squared(self._handle, buf, n.value, ctypes.byref(n)))
            stream.write(buf.raw[:n.value].decode("ascii"))
            return
        sq = self.sq_distance_grid()
        nx, ny, nz = self.dims
        for k in range(nz):
            stream.write(f"slice k={k}\n")
            for j in range(ny):
                stream.write(" ".join(str(int(v)) for v in sq[:, j, k]))
                stream.write("\n")


def query_nearest_site(field: DistanceField, voxel_index):
    """edt.py:148-161: ((i,j,k), metres) or None; IndexError out of bounds."""
    i, j, k = (int(v) for v in voxel_index)
    nx, ny, nz = field.dims
    if not (0 <= i < nx and 0 <= j < ny and 0 <= k < nz):
        raise IndexError(f"voxel {voxel_index} outside grid {field.dims}")
    site = field.site_index((i, j, k))
    if site is None:
        return None
    d2 = (i - site[0]) ** 2 + (j - site[1]) ** 2 + (k - site[2]) ** 2
    return site, field.voxel_size * float(np.sqrt(d2))


def line_nearest_sites(occupancy: np.ndarray, m1: int = 1, workers: int | None = None) -> np.ndarray:
    """edt.py:444-452: pass 1 only (GPU kernel K3)."""
    _check_workers(workers)
    if m1 < 1:
        raise ValueError("band counts must be positive")
    occ = _as_occ(occupancy)
    s1 = np.empty(occ.shape, np.int32)
    if occ.size == 0:
        return s1
    ctx = _lib.default_context()
    _lib.check(_lib.load().vx_line_nearest_sites(ctx.handle, _lib.ptr(occ), *occ.shape,
                                                 _lib.ptr(s1)))
    return s1


def brute_force_edt(occupancy: np.ndarray, voxel_size: float = 1.0) -> DistanceField:
    """edt.py:487-508: exhaustive nearest site per voxel, ties to the
    lexicographically smallest site -- the reference's test oracle, computed
    on the GPU (vx_brute_force_edt).  Meant for grids up to about 48^3."""
    occ = _as_occ(occupancy)
    if occ.size == 0:
        return DistanceField(np.empty(occ.shape, np.int32), voxel_size)
    ctx = _lib.default_context()
    h = ctypes.c_void_p()
    _lib.check(_lib.load().vx_brute_force_edt(ctx.handle, _lib.ptr(occ), *occ.shape, ctypes.byref(h)))
    return DistanceField(None, voxel_size, _handle=h, _dims=occ.shape, _ctx=ctx)


@dataclass
class ProximateStack:
    """edt.py:55-67: the surviving (sweep_coord, site) entries of one column,
    in sweep order; each owns a non-empty 1D Voronoi interval."""

    entries: list

    def sites(self) -> list:
        return [site for _, site in self.entries]


def _dominated(y_a: int, w_a: int, y_b: int, w_b: int, y_c: int, w_c: int) -> bool:
    """edt.py:70-73: b on or above the segment a-c of (y, w + y^2), which the
    GPU column kernels test in the same integer form."""
    return (w_b + y_b * y_b - w_a - y_a * y_a) * (y_c - y_b) >= (w_c + y_c * y_c - w_b - y_b * y_b) * (y_b - y_a)


def proximate_sites_1d(sites, column: int) -> ProximateStack:
    """edt.py:76-100: prune an ordered (sweep_coord, site) list to the sites
    whose interval on `column` is non-empty; site = (x, y), weight
    (x - column)^2, exact Python integers.  Raises ValueError unless the
    sweep coordinates strictly increase."""
    kept: list = []   # (coord, weight, site)
    prev = None
    for coord, site in sites:
        c = int(coord)
        if prev is not None and c <= prev:
            raise ValueError("sites must be strictly increasing in sweep coordinate")
        prev = c
        w = (int(site[0]) - int(column)) ** 2
        while len(kept) >= 2 and _dominated(kept[-2][0], kept[-2][1], kept[-1][0], kept[-1][1], c, w):
            kept.pop()
        kept.append((c, w, site))
    return ProximateStack(entries=[(c, site) for c, _, site in kept])


def pba_edt(occupancy: np.ndarray, band_cfg: BandConfig | None = None, voxel_size: float = 1.0,
            workers: int | None = None) -> DistanceField:
    """edt.py:466-484: exact EDT on the GPU; bit-identical site array."""
    _check_workers(workers)
    occ = _as_occ(occupancy)
    if band_cfg is not None and not isinstance(band_cfg, BandConfig):
        band_cfg = BandConfig(*band_cfg)
    if occ.size == 0:   # nothing to transform (the reference returns an empty field)
        return DistanceField(np.empty(occ.shape, np.int32), voxel_size)
    ctx = _lib.default_context()
    h = ctypes.c_void_p()
    _lib.check(_lib.load().vx_edt(ctx.handle, _lib.ptr(occ), *occ.shape, float(voxel_size),
                                  ctypes.byref(h)))
    return DistanceField(None, voxel_size, _handle=h, _dims=occ.shape, _ctx=ctx)
