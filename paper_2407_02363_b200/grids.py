"""Drop-in for voxarm.grids (pkg/src/voxarm/grids.py) with a device-resident grid.

``VoxelGrid`` keeps its float32 log-odds cells (plus a uint8 occupancy mirror,
a bincount scratch and the list of voxels touched since the last clear) in
GPU memory; insertion, stamping, clearing and the occupancy threshold run as
sm_100a kernels (vx_map.cu, K0-K2).  ``.cells`` is a host snapshot:
reading it copies the grid down, and in-place edits through it are uploaded
before the next device operation, so the reference's idioms
(``g.cells.fill(L_MAX)``, ``g2.cells[:] = g.cells``) keep working.

Reference line map:
  constants / logit        grids.py:17-25
  FilterConfig             grids.py:28-49
  PointCloud               grids.py:52-70   (world_points stays host numpy)
  VoxelSet                 grids.py:73-88
  InsertStats              grids.py:91-96
  VoxelGrid                grids.py:99-217
The statistical outlier filter (grids.py:224-240, k_neighbors > 0) runs on the
GPU too (vx_outlier.cu): exact kNN and numpy's summation order.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

L_MIN = -2.0
L_MAX = 3.5
DEFAULT_HIT_LOGODDS = 0.85
DEFAULT_OCCUPANCY_THRESHOLD = 0.5


def logit(p: float) -> float:
    return math.log(p / (1.0 - p))


@dataclass
class FilterConfig:
    k_neighbors: int = 8
    std_multiplier: float = 1.0
    hit_logodds: float = DEFAULT_HIT_LOGODDS
    miss_logodds: float = 0.0
    occupancy_threshold: float = DEFAULT_OCCUPANCY_THRESHOLD

    def __post_init__(self) -> None:
        if self.k_neighbors < 0:
            raise ValueError("k_neighbors must be >= 0")
        if self.std_multiplier <= 0.0:
            raise ValueError("std_multiplier must be > 0")
        if not (0.0 < self.occupancy_threshold < 1.0):
            raise ValueError("occupancy_threshold must lie in (0, 1)")


@dataclass
class PointCloud:
    points: np.ndarray
    sensor_pose: np.ndarray = field(default_factory=lambda: np.eye(4))

    def __post_init__(self) -> None:
        self.points = np.asarray(self.points, dtype=np.float64).reshape(-1, 3)
        self.sensor_pose = np.asarray(self.sensor_pose, dtype=np.float64)
        if self.sensor_pose.shape != (4, 4):
            raise ValueError("sensor_pose must be a 4x4 transform")
        if self.points.size and not np.isfinite(self.points).all():
            raise ValueError("point cloud contains non-finite coordinates")

    def world_points(self) -> np.ndarray:
        """grids.py:67-70 (host numpy, unchanged)."""
        R = self.sensor_pose[:3, :3]
        t = self.sensor_pose[:3, 3]
        return self.points @ R.T + t


@dataclass
class VoxelSet:
    origin: np.ndarray
    voxel_size: float
    indices: np.ndarray

    def __post_init__(self) -> None:
        self.origin = np.asarray(self.origin, dtype=np.float64).reshape(3)
        self.indices = np.asarray(self.indices, dtype=np.int32).reshape(-1, 3)
        if self.voxel_size <= 0.0:
            raise ValueError("voxel_size must be > 0")

    def centers(self) -> np.ndarray:
        return self.origin + (self.indices.astype(np.float64) + 0.5) * self.voxel_size


@dataclass
class InsertStats:
    inserted: int = 0
    outliers_removed: int = 0
    robot_skipped: int = 0
    out_of_bounds: int = 0


class VoxelGrid:
    """Dense 3D grid of clamped occupancy log-odds, resident on the GPU."""

    def __init__(self, dims, voxel_size: float, origin=(0.0, 0.0, 0.0), *, _handle=None,
                 _ctx=None, _owned=True):
        dims = tuple(int(d) for d in dims)
        if len(dims) != 3 or any(d <= 0 for d in dims):
            raise ValueError(f"dims must be three positive integers, got {dims}")
        if voxel_size <= 0.0:
            raise ValueError("voxel_size must be > 0")
        if dims[0] * dims[1] * dims[2] >= 2**31:
            raise ValueError("grid too large for 32-bit voxel addressing")
        self.dims = dims
        self.voxel_size = float(voxel_size)
        self.origin = np.asarray(origin, dtype=np.float64).reshape(3)
        self._ctx = _ctx or _lib.default_context()
        self._owned = _owned
        if _handle is None:
            h = ctypes.c_void_p()
            _lib.check(_lib.load().vx_grid_create(self._ctx.handle, *dims, self.voxel_size,
                                                  _lib.ptr(self.origin), ctypes.byref(h)))
            self._h = h
        else:
            self._h = _handle
        self._host = None   # host mirror handed out through .cells (None until asked for)
        self._snap = None   # its content as last synchronised with the device

    def __del__(self):
        try:
            if self._owned and self._h is not None:
                _lib.load().vx_grid_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        self._push()
        return self._h

    # -- host mirror ------------------------------------------------------------
    # Once .cells has been handed out, the mirror is refreshed after every
    # device mutation (so references held by the caller stay current, as the
    # reference's in-place numpy updates do) and any edit made through it is
    # uploaded before the next device operation.
    @property
    def cells(self) -> np.ndarray:
        if self._host is None:
            self._host = np.empty(self.dims, np.float32)
            self._sync_down()
        return self._host

    @cells.setter
    def cells(self, value) -> None:
        arr = np.ascontiguousarray(np.broadcast_to(np.asarray(value, np.float32), self.dims))
        _lib.check(_lib.load().vx_grid_write_cells(self._h, _lib.ptr(arr)))
        if self._host is not None:
            self._host[...] = arr
            self._snap = arr.copy()

    def _sync_down(self) -> None:
        _lib.check(_lib.load().vx_grid_read_cells(self._h, _lib.ptr(self._host)))
        self._snap = self._host.copy()

    def _push(self) -> None:
        if self._host is not None and not np.array_equal(self._host.view(np.uint32),
                                                         self._snap.view(np.uint32)):
            _lib.check(_lib.load().vx_grid_write_cells(self._h, _lib.ptr(self._host)))
            self._snap = self._host.copy()

    def _touched(self) -> None:
        if self._host is not None:
            self._sync_down()

    # -- geometry (grids.py:122-142) ------------------------------------------
    def world_to_voxel(self, point) -> tuple[int, int, int] | None:
        idx = np.floor((np.asarray(point, dtype=np.float64) - self.origin)
                       / self.voxel_size).astype(np.int64)
        if (idx < 0).any() or (idx >= self.dims).any():
            return None
        return int(idx[0]), int(idx[1]), int(idx[2])

    def world_to_voxel_many(self, points: np.ndarray):
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        idx = np.floor((pts - self.origin) / self.voxel_size).astype(np.int64)
        ok = ((idx >= 0) & (idx < np.asarray(self.dims))).all(axis=1)
        return idx, ok

    def voxel_center(self, index) -> np.ndarray:
        return self.origin + (np.asarray(index, dtype=np.float64) + 0.5) * self.voxel_size

    # -- mutation -------------------------------------------------------------
    def clear(self) -> None:
        """grids.py:146-147 (K0 sparse reset)."""
        self._push()
        _lib.check(_lib.load().vx_grid_clear(self._h))
        self._touched()

    def insert_point_cloud(self, cloud: PointCloud, cfg: FilterConfig,
                           robot_mask: "VoxelGrid | None" = None) -> InsertStats:
        """grids.py:149-188 on the GPU (K1 scatter + bincount/clip epilogue)."""
        if robot_mask is not None and not self.same_geometry(robot_mask):
            raise ValueError("robot_mask geometry does not match this grid")
        stats = InsertStats()
        pts = cloud.world_points()
        if pts.shape[0] == 0:
            return stats
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        self._push()
        mh = robot_mask.handle if robot_mask is not None else None
        st = _lib.InsertStatsC()
        # k_neighbors > 0: statistical outlier filter on the GPU first (grids.py:166-169)
        _lib.check(_lib.load().vx_grid_insert_points_ex(
            self._h, _lib.ptr(pts), pts.shape[0], float(np.float32(cfg.hit_logodds)),
            float(cfg.occupancy_threshold), mh, int(cfg.k_neighbors), float(cfg.std_multiplier),
            ctypes.byref(st)))
        self._touched()
        stats.inserted = int(st.inserted)
        stats.outliers_removed = int(st.outliers_removed)
        stats.robot_skipped = int(st.robot_skipped)
        stats.out_of_bounds = int(st.out_of_bounds)
        return stats

    def insert_voxel_set(self, vset: VoxelSet, transform: np.ndarray | None = None) -> int:
        """grids.py:190-203 on the GPU (K2 stamp); returns the out-of-grid count."""
        return self.insert_voxel_sets([vset], None if transform is None else [transform])[0]

    def insert_voxel_sets(self, vsets, transforms=None, value: float = L_MAX) -> list[int]:
        """Many insert_voxel_set calls in one launch (all links of a robot)."""
        n = len(vsets)
        if n == 0:
            return []
        idx = [np.ascontiguousarray(v.indices, dtype=np.int32) for v in vsets]
        ptrs = (ctypes.c_void_p * n)(*[i.ctypes.data for i in idx])
        counts = np.array([i.shape[0] for i in idx], np.int64)
        origins = np.ascontiguousarray(np.stack([v.origin for v in vsets]), np.float64)
        vss = np.array([v.voxel_size for v in vsets], np.float64)
        T = None
        if transforms is not None:
            T = np.ascontiguousarray(np.stack([np.asarray(t, np.float64).reshape(4, 4)
                                               for t in transforms]))
        oob = np.zeros(n, np.int64)
        self._push()
        _lib.check(_lib.load().vx_grid_insert_voxel_sets(
            self._h, n, ptrs, _lib.ptr(counts), _lib.ptr(origins), _lib.ptr(vss),
            None if T is None else _lib.ptr(T), float(value), _lib.ptr(oob)))
        self._touched()
        return [int(v) for v in oob]

    # -- queries ----------------------------------------------------------------
    def occupancy_mask(self, threshold: float = DEFAULT_OCCUPANCY_THRESHOLD) -> np.ndarray:
        """grids.py:207-208 (thresholded on the GPU, copied down as bool)."""
        self._push()
        out = np.empty(self.dims, np.uint8)
        _lib.check(_lib.load().vx_grid_occupancy(self._h, float(threshold), _lib.ptr(out)))
        return out.view(np.bool_)

    def occupied_voxels(self, threshold: float = DEFAULT_OCCUPANCY_THRESHOLD) -> np.ndarray:
        """grids.py:210-212: np.argwhere(occupancy_mask), compacted on the
        device in lexicographic order ((K,3) int64)."""
        self._push()
        L = _lib.load()
        n = ctypes.c_int64()
        _lib.check(L.vx_grid_occupied_voxels(self._h, float(threshold), None, 0, ctypes.byref(n)))
        out = np.empty((n.value, 3), np.int64)
        if n.value:
            _lib.check(L.vx_grid_occupied_voxels(self._h, float(threshold), _lib.ptr(out), n.value,
                                                 ctypes.byref(n)))
        return out

    def same_geometry(self, other: "VoxelGrid") -> bool:
        return (self.dims == other.dims
                and self.voxel_size == other.voxel_size
                and np.array_equal(self.origin, other.origin))

    # -- device-side EDT (no host round trip) ------------------------------------
    def distance_field(self, threshold: float = DEFAULT_OCCUPANCY_THRESHOLD):
        """pba_edt(self.occupancy_mask(threshold), voxel_size=self.voxel_size)
        computed without leaving the device."""
        from .edt import DistanceField
        self._push()
        h = ctypes.c_void_p()
        _lib.check(_lib.load().vx_edt_grid(self._h, float(threshold), ctypes.byref(h)))
        return DistanceField(None, self.voxel_size, _handle=h, _dims=self.dims, _ctx=self._ctx)


def new_grid(dims, voxel_size: float, origin=(0.0, 0.0, 0.0)) -> VoxelGrid:
    return VoxelGrid(dims, voxel_size, origin)


def statistical_outlier_filter(points: np.ndarray, k_neighbors: int,
                               std_multiplier: float) -> np.ndarray:
    """grids.py:224-240 on the GPU: the points whose mean k-NN distance is at
    most mean + std_multiplier * std (population); <= k points pass through."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    if pts.shape[0] <= k_neighbors or pts.shape[0] == 0:
        return pts
    keep = np.empty(pts.shape[0], np.uint8)
    removed = ctypes.c_int64()
    _lib.check(_lib.load().vx_outlier_mask(_lib.default_context().handle, _lib.ptr(pts),
                                           pts.shape[0], int(k_neighbors), float(std_multiplier),
                                           _lib.ptr(keep), ctypes.byref(removed)))
    return pts[keep.view(np.bool_)]


def load_point_cloud(path) -> PointCloud:
    """grids.py:243-256: a text cloud, one "x y z" per line, '#' comments and
    blank lines skipped; ValueError on a short line (host file I/O)."""
    rows = []
    with open(path) as fh:
        for raw in fh:
            text = raw.strip()
            if not text or text.startswith("#"):
                continue
            fields = text.split()
            if len(fields) < 3:
                raise ValueError(f"bad point line: {text!r}")
            rows.append([float(v) for v in fields[:3]])
    return PointCloud(points=np.asarray(rows, dtype=np.float64).reshape(-1, 3))

