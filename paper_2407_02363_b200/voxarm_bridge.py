"""Route an unmodified voxarm engine through the GPU path.

voxarm's engine binds ``pba_edt`` and ``VoxelGrid`` by name at import
(engine.py:26-27); ``SimEngine.__init__`` builds its three grids from that
name (engine.py:143-145), the camera branch calls ``clear``,
``insert_voxel_set``, ``insert_point_cloud``, ``occupancy_mask``, a blake2b
digest of the mask and ``pba_edt`` (engine.py:234-268), and the per-tick
site lookup is ``SimEngine._site_world`` (engine.py:212-221).  ``install()``
keeps the engine's code and replaces what it calls:

  * ``VoxelGrid`` -> a device-resident grid whose ``occupancy_mask()``
    returns a *device occupancy* handle instead of an N-byte host array.
    Its ``tobytes()`` is a 16-byte digest of the occupied-voxel set computed
    on the device from the grid's touched list (vx_grid_occupancy_digest),
    so the engine's blake2b memo (engine.py:259-268) hashes 16 bytes, and
    the field is recomputed exactly when the occupancy changed;
  * ``pba_edt`` -> for a device occupancy handle, the EDT of the grid's
    device occupancy into a pooled device field (vx_edt_grid_into: no copy,
    no allocation per tick); any host array takes the ordinary drop-in;
  * ``SimEngine._site_world`` -> the first lookup of a tick answers every
    sphere centre on both fields in one batched K6 launch
    (vx_fields_site_world), the remaining lookups read that batch.  The
    centres are re-derived with the engine's own expression
    (engine.py:273-275), and a lookup of any other point is answered on the
    device directly.

Task-priority control, the tasks and the integration (tasks.py,
controller.py, engine.py:282-318) run unchanged on the host.

    from paper_2407_02363_b200 import voxarm_bridge
    with voxarm_bridge.installed():      # or voxarm_bridge.install()
        log = voxarm.engine.run_scenario(sc)

The engine's default statistical outlier filter (k_neighbors=8,
grids.py:224-240) runs on the device too (vx_outlier.cu), so the shipped
scenarios run unmodified; tests/test_acceptance_gpu.py checks their CSV logs
against the CPU engine's.
"""

from __future__ import annotations

import contextlib
import ctypes
import weakref

import numpy as np

from . import _lib, edt, grids

_saved: dict = {}


class DeviceOccupancy:
    """What EngineVoxelGrid.occupancy_mask returns: the grid's occupancy at a
    threshold, left on the device.  ``tobytes()`` is its 16-byte device
    digest (the engine hashes it); ``np.asarray`` copies the mask down for
    any other consumer."""

    __array_priority__ = 1.0

    def __init__(self, grid: "EngineVoxelGrid", threshold: float):
        self.grid = grid
        self.threshold = float(threshold)
        self.shape = tuple(grid.dims)
        self.ndim = 3
        self.dtype = np.dtype(bool)
        self._digest = None

    def tobytes(self) -> bytes:
        if self._digest is None:
            d = np.zeros(2, np.uint64)
            _lib.check(_lib.load().vx_grid_occupancy_digest(self.grid.handle, self.threshold, _lib.ptr(d)))
            self._digest = d.tobytes()
        return self._digest

    def __array__(self, dtype=None, copy=None):
        m = grids.VoxelGrid.occupancy_mask(self.grid, self.threshold)
        return m if dtype is None else m.astype(dtype)


class _FieldPool:
    """Two device fields per grid, reused across camera ticks: a buffer is
    refilled only once the DistanceField that exposed it is gone (the engine
    drops the previous field when it stores the new one)."""

    def __init__(self, grid):
        self.ctx = grid._ctx
        self.dims = tuple(grid.dims)
        self.handles: list = []
        self.views: list = []

    def take(self):
        for q, ref in enumerate(self.views):
            if ref() is None:
                return q
        h = ctypes.c_void_p()
        _lib.check(_lib.load().vx_field_create(self.ctx.handle, *self.dims, ctypes.byref(h)))
        self.handles.append(h)
        self.views.append(lambda: None)
        return len(self.handles) - 1

    def __del__(self):   # every view and the grid are gone
        try:
            L = _lib.load()
            for h in self.handles:
                L.vx_field_destroy(h)
            self.handles = []
        except Exception:
            pass


class EngineVoxelGrid(grids.VoxelGrid):
    """The drop-in VoxelGrid plus the device occupancy handle the engine's
    memo and EDT take (only the engine module sees this class)."""

    def occupancy_mask(self, threshold: float = grids.DEFAULT_OCCUPANCY_THRESHOLD):
        self._push()
        return DeviceOccupancy(self, threshold)

    def _field_pool(self) -> _FieldPool:
        pool = getattr(self, "_pool", None)
        if pool is None:
            pool = self._pool = _FieldPool(self)
        return pool


def engine_pba_edt(occupancy, band_cfg=None, voxel_size: float = 1.0, workers=None):
    """engine.py:265-267's pba_edt: a device occupancy handle is transformed
    where it lives, into the grid's field pool; anything else takes the
    ordinary drop-in (edt.pba_edt)."""
    if not isinstance(occupancy, DeviceOccupancy):
        return edt.pba_edt(occupancy, band_cfg=band_cfg, voxel_size=voxel_size, workers=workers)
    edt._check_workers(workers)
    if band_cfg is not None and not isinstance(band_cfg, edt.BandConfig):
        band_cfg = edt.BandConfig(*band_cfg)
    grid = occupancy.grid
    pool = grid._field_pool()
    q = pool.take()
    h = pool.handles[q]
    _lib.check(_lib.load().vx_edt_grid_into(grid.handle, occupancy.threshold, h))
    fld = edt.DistanceField(None, voxel_size, _handle=h, _dims=pool.dims, _ctx=pool.ctx, _owned=False)
    fld._pool_ref = pool   # the buffers outlive every view of them
    pool.views[q] = weakref.ref(fld)
    return fld


def _batched_site_world(self, key: str, center: np.ndarray):
    """SimEngine._site_world (engine.py:212-221): identical results, one
    batched device query per tick for all sphere centres on both maps."""
    fld = self._fields[key]
    if fld is None:
        return None
    c = np.asarray(center, dtype=np.float64).reshape(3)
    cache = getattr(self, "_vx_sites", None)
    stamp = (self.tick, id(self._fields["env"]), id(self._fields["self"]))
    if cache is None or cache[0] != stamp:
        # this tick's centres, exactly as engine.py:273-275 forms them
        frames = self.chain.forward_kinematics(self.q)
        centers = np.array([frames[s.link_index][:3, :3] @ s.center + frames[s.link_index][:3, 3]
                            for s in self.spheres])
        cache = (stamp, _query(self, centers))
        self._vx_sites = cache
    hit = cache[1].get(key, {}).get(c.tobytes())
    if hit is not None:
        return hit[0]
    return _query(self, c.reshape(1, 3))[key][c.tobytes()][0]


def _query(self, centers: np.ndarray) -> dict:
    """{key: {centre bytes: (world point or None,)}} for the present fields."""
    keys = [k for k in ("env", "self") if self._fields[k] is not None]
    flds = [self._fields[k] for k in keys]
    if any(f.device_handle is None for f in flds):   # a host-built field: the reference formula
        return {k: {c.tobytes(): (_host_site_world(self, f, c),) for c in centers} for k, f in zip(keys, flds)}
    s = centers.shape[0]
    nf = len(flds)
    lin = np.empty(nf * s, np.int32)
    world = np.empty((nf * s, 3), np.float64)
    dist = np.empty(nf * s, np.float64)
    c = np.ascontiguousarray(centers, np.float64)
    _lib.check(_lib.load().vx_fields_site_world(
        flds[0].device_handle, flds[1].device_handle if nf > 1 else None, _lib.ptr(self._origin),
        float(self.sc.grid.voxel_size), _lib.ptr(c), s, _lib.ptr(lin), _lib.ptr(world), _lib.ptr(dist)))
    out = {}
    for q, k in enumerate(keys):
        out[k] = {c[i].tobytes(): (None if lin[q * s + i] < 0 else world[q * s + i].copy(),) for i in range(s)}
    return out


def _host_site_world(self, fld, center):
    idx = np.floor((center - self._origin) / self.sc.grid.voxel_size)
    idx = np.clip(idx.astype(np.int64), 0, self._dims - 1)
    site = fld.site_index(tuple(int(v) for v in idx))
    if site is None:
        return None
    return self._origin + (np.asarray(site) + 0.5) * self.sc.grid.voxel_size


def install(engine_module=None) -> None:
    """Rebind voxarm.engine's VoxelGrid, pba_edt and SimEngine._site_world to
    the device-resident drop-ins."""
    if engine_module is None:
        import voxarm.engine as engine_module
    if "VoxelGrid" not in _saved:
        _saved["module"] = engine_module
        _saved["VoxelGrid"] = engine_module.VoxelGrid
        _saved["pba_edt"] = engine_module.pba_edt
        _saved["_site_world"] = engine_module.SimEngine._site_world
    engine_module.VoxelGrid = EngineVoxelGrid
    engine_module.pba_edt = engine_pba_edt
    engine_module.SimEngine._site_world = _batched_site_world


def uninstall() -> None:
    if "VoxelGrid" in _saved:
        m = _saved["module"]
        m.VoxelGrid = _saved.pop("VoxelGrid")
        m.pba_edt = _saved.pop("pba_edt")
        m.SimEngine._site_world = _saved.pop("_site_world")
        _saved.pop("module")


@contextlib.contextmanager
def installed(engine_module=None):
    install(engine_module)
    try:
        yield
    finally:
        uninstall()


def transfer_bytes(ctx=None) -> tuple[int, int]:
    """(host->device, device->host) bytes copied by libvx calls so far."""
    ctx = ctx or _lib.default_context()
    out = np.zeros(2, np.int64)
    _lib.check(_lib.load().vx_ctx_transfer_bytes(ctx.handle, _lib.ptr(out)))
    return int(out[0]), int(out[1])
