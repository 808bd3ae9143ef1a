"""GPU camera tick and sphere gather: the hot-path slice of voxarm's
SimEngine.step (pkg/src/voxarm/engine.py:225-322).

  site_world   SimEngine._site_world (engine.py:212-221) for many centres at
               once, plus the distance of tasks.py:102-104 (K6 on the GPU)
  MapCycle     one camera tick, engine.py:233-280: clear x3, stamp the
               self-obstacle links and the robot mask, scatter the cloud,
               EDT of env (and of self when its voxel set changed), and the
               per-sphere gather on both maps -- device resident, one
               C call per tick (vx_cycle_step)

The host controller (tasks.py / controller.py) is unchanged: it consumes
``(site_world, distance)`` exactly as it consumes _site_world today.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .edt import DistanceField
from .grids import L_MAX, VoxelGrid


def site_world(field: DistanceField, origin, voxel_size: float, centers):
    """For every centre: clip(floor((c - origin)/vs)) -> nearest-site flat
    index, its world centre and ||O - C||.  Returns (lin int32 (S,),
    world float64 (S,3), dist float64 (S,)); lin = -1, world NaN, dist inf
    where the reference returns None."""
    c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    s = c.shape[0]
    lin = np.empty(s, np.int32)
    world = np.empty((s, 3), np.float64)
    dist = np.empty(s, np.float64)
    if s == 0:
        return lin, world, dist
    org = np.ascontiguousarray(origin, dtype=np.float64).reshape(3)
    h = field.device_handle
    if h is None:  # a host-constructed field: upload it as a device field first
        raise ValueError("site_world needs a device field (from pba_edt / VoxelGrid.distance_field)")
    _lib.check(_lib.load().vx_field_site_world(h, _lib.ptr(org), float(voxel_size), _lib.ptr(c), s,
                                               _lib.ptr(lin), _lib.ptr(world), _lib.ptr(dist)))
    return lin, world, dist


class StagedCloud:
    """Ticket of a cloud staged on the device by MapCycle.prefetch."""

    __slots__ = ("cycle", "ticket", "array")

    def __init__(self, cycle, ticket: int, array):
        self.cycle, self.ticket, self.array = cycle, ticket, array


class MapCycle:
    """Device-resident camera tick (engine.py:233-280) for one robot.

    links: list of (ijk int32 (K,3), origin (3,)) voxel sets in link frames
    (robot.voxelize_link), link_voxel_size, self_links: the self-obstacle
    link indices (robot.self_obstacle_links).
    """

    def __init__(self, dims, voxel_size: float, origin, links, link_voxel_size: float, self_links,
                 max_points: int, max_spheres: int, ctx=None):
        self.ctx = ctx or _lib.default_context()
        self.dims = tuple(int(d) for d in dims)
        self.voxel_size = float(voxel_size)
        self.origin = np.ascontiguousarray(origin, dtype=np.float64).reshape(3)
        self._ijk = [np.ascontiguousarray(i, dtype=np.int32).reshape(-1, 3) for i, _ in links]
        ptrs = (ctypes.c_void_p * max(1, len(links)))(*[a.ctypes.data for a in self._ijk])
        counts = np.array([a.shape[0] for a in self._ijk], np.int64)
        origins = np.ascontiguousarray(np.array([o for _, o in links], np.float64).reshape(-1, 3))
        selfl = np.ascontiguousarray(self_links, dtype=np.int32).reshape(-1)
        self.nlinks = len(links)
        self.max_spheres = int(max_spheres)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().vx_cycle_create(
            self.ctx.handle, *self.dims, self.voxel_size, _lib.ptr(self.origin), self.nlinks, ptrs,
            _lib.ptr(counts), _lib.ptr(origins), float(link_voxel_size), _lib.ptr(selfl),
            selfl.shape[0], int(max_points), int(max_spheres), ctypes.byref(h)))
        self._h = h
        S = max(1, self.max_spheres)
        self._lin = _lib.PinnedArray((2, S), np.int32)
        self._world = _lib.PinnedArray((2, S, 3), np.float64)
        self._dist = _lib.PinnedArray((2, S), np.float64)
        self._s = 0
        L = _lib.load()
        self._step_staged, self._prefetch, self._wait = L.vx_cycle_step_staged, L.vx_cycle_prefetch, L.vx_cycle_wait
        self._hit_key, self._hit32 = None, 0.0

    def close(self):
        if self._h is not None:
            _lib.load().vx_cycle_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, points, link_frames, centers, hit_logodds: float = 0.85,
             occupancy_threshold: float = 0.5, sync: bool = True):
        """Run one tick.  points: (P,3) float64 world points (pinned for an
        async copy) or a StagedCloud from prefetch(); link_frames:
        (nlinks,4,4) FK frames, centers: (S,3)."""
        T = np.ascontiguousarray(link_frames, dtype=np.float64).reshape(-1, 16)
        c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
        self._s = c.shape[0]
        if isinstance(points, StagedCloud):
            if points.cycle is not self:
                raise ValueError("StagedCloud belongs to another MapCycle")
            # the per-tick call: plain integer addresses (ctypes converts them
            # for the c_void_p parameters), the float32 hit cached
            if hit_logodds != self._hit_key:
                self._hit_key, self._hit32 = hit_logodds, float(np.float32(hit_logodds))
            rc = self._step_staged(self._h, points.ticket, T.ctypes.data, self._hit32,
                                   float(occupancy_threshold), c.ctypes.data, c.shape[0], 1 if sync else 0)
            if rc:
                _lib.check(rc)
            pts = points.array
        else:
            pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
            _lib.check(_lib.load().vx_cycle_step(self._h, _lib.ptr(pts), pts.shape[0], _lib.ptr(T),
                                                 float(np.float32(hit_logodds)),
                                                 float(occupancy_threshold), _lib.ptr(c),
                                                 c.shape[0], 1 if sync else 0))
        self._keep = (pts, T, c)   # host buffers must outlive an async copy
        return self

    def prefetch(self, points) -> "StagedCloud":
        """Upload a later tick's cloud while the current one computes
        (vx_cycle_prefetch) and return its ticket; pass the ticket to step()
        in place of the points.  The upload is asynchronous: leave the
        (pinned) array unchanged until that tick has been waited for.  Two
        slots -- a third prefetch invalidates the oldest unconsumed ticket,
        and stepping with a consumed or invalidated ticket raises."""
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        t = ctypes.c_uint64()
        rc = self._prefetch(self._h, pts.ctypes.data, pts.shape[0], ctypes.byref(t))
        if rc:
            _lib.check(rc)
        self._pf = getattr(self, "_pf", [])[-1:] + [pts]   # alive until the upload ran
        return StagedCloud(self, int(t.value), pts)

    def wait(self):
        """Results of the last step: dict with stats and per-map (lin, world, dist)."""
        res = _lib.CycleResultC()
        s = self._s
        lin = np.empty((2, s), np.int32)
        world = np.empty((2, s, 3), np.float64)
        dist = np.empty((2, s), np.float64)
        rc = self._wait(self._h, ctypes.byref(res), lin.ctypes.data, world.ctypes.data, dist.ctypes.data)
        if rc:
            _lib.check(rc)
        st = res.stats
        return {"inserted": st.inserted, "robot_skipped": st.robot_skipped,
                "out_of_bounds": st.out_of_bounds, "self_recomputed": bool(res.self_recomputed),
                "env": (lin[0], world[0], dist[0]), "self": (lin[1], world[1], dist[1])}

    def info(self) -> dict:
        """How the last tick ran (vx_cycle_info)."""
        a = np.zeros(4, np.int32)
        _lib.check(_lib.load().vx_cycle_info(self._h, _lib.ptr(a)))
        return {"pass3_mode": int(a[0]), "graph": bool(a[1]), "captures": int(a[2]),
                "occupied_slices": int(a[3])}

    def set_avoidance(self, radius, buffer, link_index, n_joints: int, kappa: float,
                      x_star_offset=None):
        """Enable the on-device avoidance rows (tasks.py:88-123) for a fixed
        sphere set: radius/buffer/link_index per sphere (robot.build_spheres),
        n_joints = chain.n, AvoidanceConfig's kappa and x_star_offset (None
        means 2*buffer).  Steps with exactly this many centres build them."""
        r = np.ascontiguousarray(radius, dtype=np.float64).reshape(-1)
        b = np.ascontiguousarray(buffer, dtype=np.float64).reshape(-1)
        li = np.ascontiguousarray(link_index, dtype=np.int32).reshape(-1)
        if not (r.size == b.size == li.size):
            raise ValueError("radius, buffer and link_index lengths differ")
        off = -1.0 if x_star_offset is None else float(x_star_offset)
        _lib.check(_lib.load().vx_cycle_set_avoidance(self._h, r.size, _lib.ptr(r), _lib.ptr(b),
                                                      _lib.ptr(li), int(n_joints), float(kappa), off))
        self._av = (r.size, int(n_joints))

    def set_joint_frames(self, origins, axes):
        """chain.joint_frames(q) of the next step (robot.py:545-558)."""
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        a = np.ascontiguousarray(axes, dtype=np.float64).reshape(-1, 3)
        _lib.check(_lib.load().vx_cycle_set_joint_frames(self._h, _lib.ptr(o), _lib.ptr(a)))

    def rows(self):
        """Avoidance rows of the last step per map ("env", "self"): dict of
        J (s, n), activation, xdot_ref, value (s,) and flag (s,) -- 0 no site,
        1 built, 2 zero distance (activation 1, J zero: the caller applies
        its held direction, tasks.py:111-119)."""
        s, n = self._av
        J = np.zeros((2, s, n), np.float64)
        act = np.empty((2, s), np.float64)
        ref = np.empty((2, s), np.float64)
        val = np.empty((2, s), np.float64)
        flag = np.empty((2, s), np.int32)
        _lib.check(_lib.load().vx_cycle_rows(self._h, _lib.ptr(J), _lib.ptr(act), _lib.ptr(ref),
                                             _lib.ptr(val), _lib.ptr(flag)))
        return {k: {"J": J[m], "activation": act[m], "xdot_ref": ref[m], "value": val[m],
                    "flag": flag[m]} for m, k in enumerate(("env", "self"))}

    def fields(self):
        e, s = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.load().vx_cycle_fields(self._h, ctypes.byref(e), ctypes.byref(s)))
        mk = lambda h: DistanceField(None, self.voxel_size, _handle=h, _dims=self.dims,  # noqa: E731
                                     _ctx=self.ctx, _owned=False)
        return mk(e), mk(s)

    def grids(self):
        e, s, m = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.load().vx_cycle_grids(self._h, ctypes.byref(e), ctypes.byref(s),
                                              ctypes.byref(m)))
        mk = lambda h: VoxelGrid(self.dims, self.voxel_size, self.origin, _handle=h,  # noqa: E731
                                 _ctx=self.ctx, _owned=False)
        return mk(e), mk(s), mk(m)


__all__ = ["site_world", "MapCycle", "StagedCloud", "L_MAX"]
