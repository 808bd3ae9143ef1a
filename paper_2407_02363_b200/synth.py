"""Seeded synthetic inputs shared by the tests, the bench and the golden
generator.  Host-side numpy only; the same calls produce the same bits on the
build container and on the GPU box (same image, same numpy).

Generators follow the reference where it has one:
  * ``bernoulli_occupancy``  -- cli.py:78-79 (``default_rng(seed).random(dims) < p``)
  * ``oscillating_sphere_cloud`` -- movers.py:19-54, 66-87 + robot.Sphere.sample_surface
    (robot.py:175-178)
  * sphere centres -- engine.py:273-275
The rest (insert / stamp / site-world cases, the depth-camera cloud of config
C2) are this repo's own seeded generators; SURVEY.md section 8(d) defines them.
"""

from __future__ import annotations

import math

import numpy as np

# --------------------------------------------------------------------------
# occupancy grids
# --------------------------------------------------------------------------


def bernoulli_occupancy(dims, p: float, seed: int, slab: int = 64) -> np.ndarray:
    """``default_rng(seed).random(dims) < p`` (cli.py:78-79) as uint8, generated
    in i-slabs so 1024^3 does not need an 8 GB float temporary.  The PCG64
    stream is consumed in C order either way, so the bits are identical."""
    nx, ny, nz = (int(d) for d in dims)
    rng = np.random.default_rng(seed)
    out = np.empty((nx, ny, nz), np.uint8)
    for i0 in range(0, nx, slab):
        i1 = min(nx, i0 + slab)
        out[i0:i1] = rng.random((i1 - i0, ny, nz)) < p
    return out


def bernoulli_slab(dims, p: float, seed: int, i0: int, i1: int) -> np.ndarray:
    """Rows [i0, i1) of ``bernoulli_occupancy(dims, p, seed)`` without
    materialising the rest (skips the stream with ``rng.random`` in chunks)."""
    nx, ny, nz = (int(d) for d in dims)
    rng = np.random.default_rng(seed)
    plane = ny * nz
    skip = i0
    while skip > 0:                       # advance the stream i0 planes
        step = min(skip, max(1, (1 << 26) // plane))
        rng.random(step * plane)
        skip -= step
    return (rng.random((i1 - i0, ny, nz)) < p).astype(np.uint8)


def structured_occupancy(name: str, dims) -> np.ndarray:
    nx, ny, nz = (int(d) for d in dims)
    occ = np.zeros((nx, ny, nz), np.uint8)
    if name == "single_center":
        occ[nx // 2, ny // 2, nz // 2] = 1
    elif name == "single_corner":
        occ[0, 0, 0] = 1
    elif name == "full":
        occ[:] = 1
    elif name == "empty":
        pass
    elif name == "two_corners":
        occ[0, 0, 0] = 1
        occ[-1, -1, -1] = 1
    else:
        raise ValueError(name)
    return occ


# --------------------------------------------------------------------------
# obstacle clouds
# --------------------------------------------------------------------------


def sphere_surface(count: int, radius: float, rng) -> np.ndarray:
    """robot.Sphere.sample_surface (robot.py:175-178) with centre 0."""
    d = rng.normal(size=(count, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.zeros(3) + radius * d


def oscillating_sphere_cloud(t: float, *, obstacle_id: int, radius: float, points: int,
                             noise_std: float, seed: int, center, axis, amplitude: float,
                             period: float) -> np.ndarray:
    """movers.OscillatingMover(...).cloud_points(t) (movers.py:31-54, 66-87)."""
    rng = np.random.default_rng([int(seed) & 0xFFFFFFFF, int(obstacle_id)])
    base = sphere_surface(points, radius, rng)
    if noise_std > 0:
        base = base + rng.normal(0.0, noise_std, base.shape)
    axis = np.asarray(axis, dtype=np.float64).reshape(3)
    axis = axis / float(np.linalg.norm(axis))
    phase = float(np.sin(2.0 * np.pi * t / period))
    pos = np.asarray(center, dtype=np.float64).reshape(3) + axis * (amplitude * phase)
    return base + pos


_DESK7 = {}


def desk7_model() -> dict:
    """The desk7 robot at 2 cm as the host-side producers make it
    (robot.voxelize_link / forward_kinematics / build_spheres, robot.py:467-
    620): link voxel sets ("links": [(ijk int32 (K,3), origin (3,))]), the
    self-obstacle links "o_links", a trajectory of FK "frames" and the
    sphere table.  Generated once by the reference (tests/golden/make_golden.py)
    and shipped as package data: this repo does not rebuild the robot model."""
    if not _DESK7:
        import os
        z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "desk7_2cm.npz"))
        d = {k: z[k] for k in z.files}
        n = d["frames"].shape[1]
        d["links"] = [(d[f"link{li}_ijk"], d[f"link{li}_origin"]) for li in range(n)]
        _DESK7.update(d)
    return _DESK7


# config C1: 128^3 @ 2 cm, desk7 at GUARD_Q, 50k-point sphere
C1 = {"dims": (128, 128, 128), "voxel_size": 0.02, "origin": (-1.28, -1.28, -0.24),
      "points": 50_000, "seed": 0, "obstacle_radius": 0.15,
      "obstacle_center": (0.6, 0.0, 0.5), "n_spheres": 30}

GUARD_Q = (0.0, 0.0, 0.2, 0.0, 0.5, 0.0, 0.3, 0.0)


def c1_cloud(t: float) -> np.ndarray:
    return oscillating_sphere_cloud(t, obstacle_id=0, radius=C1["obstacle_radius"],
                                    points=C1["points"], noise_std=0.0, seed=C1["seed"],
                                    center=C1["obstacle_center"], axis=(0, 1, 0),
                                    amplitude=0.2, period=1.5)


def grid_aabb(dims, voxel_size, origin):
    lo = np.asarray(origin, np.float64)
    return lo, lo + np.asarray(dims, np.float64) * voxel_size


def extra_query_points(dims, voxel_size, origin, count: int = 9, seed: int = 30):
    lo, hi = grid_aabb(dims, voxel_size, origin)
    return np.random.default_rng(seed).uniform(lo, hi, size=(count, 3))


def sphere_centers(frames, sphere_link, sphere_center) -> np.ndarray:
    """engine.py:273-275, from FK frames and the build_spheres table."""
    return np.array([frames[li][:3, :3] @ c + frames[li][:3, 3]
                     for li, c in zip(sphere_link, sphere_center)])


def c1_sphere_centers_from(chain, q) -> np.ndarray:
    """30 C1 query centres from a live voxarm chain (golden generator only)."""
    frames = chain.forward_kinematics(q)
    sph = chain.build_spheres()
    c = sphere_centers(frames, [s.link_index for s in sph], [s.center for s in sph])
    extra = extra_query_points(C1["dims"], C1["voxel_size"], C1["origin"],
                               C1["n_spheres"] - len(sph))
    return np.vstack([c, extra])


def depth_camera_cloud(t: float, *, width: int = 640, height: int = 480,
                       eye=(-1.5, 0.0, 1.2), target=(0.6, 0.0, 0.4), fov_deg: float = 70.0,
                       sphere_center=(0.6, 0.0, 0.5), sphere_radius: float = 0.15,
                       amplitude: float = 0.2, period: float = 1.5, wall_x: float = 2.0,
                       noise_std: float = 0.002, seed: int = 2,
                       max_points: int | None = 300_000) -> np.ndarray:
    """Config C2's depth-camera-like cloud: a pinhole ray grid cast in f64
    against the floor z=0, a back wall x=wall_x and an oscillating sphere,
    plus N(0, noise) range noise.  Dense surfaces put many hits per voxel."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, [0.0, 0.0, 1.0])
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    f = 0.5 / math.tan(math.radians(fov_deg) / 2)
    u = (np.arange(width) + 0.5) / width - 0.5
    v = ((np.arange(height) + 0.5) / height - 0.5) * height / width
    uu, vv = np.meshgrid(u, v)
    d = (f * fwd[None, None, :] + uu[..., None] * right + vv[..., None] * up).reshape(-1, 3)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    n = d.shape[0]
    rng_t = np.full(n, np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        tf = np.where(d[:, 2] < 0, -eye[2] / d[:, 2], np.inf)            # floor
        tw = np.where(d[:, 0] > 0, (wall_x - eye[0]) / d[:, 0], np.inf)  # wall
    rng_t = np.minimum(rng_t, np.where(tf > 0, tf, np.inf))
    rng_t = np.minimum(rng_t, np.where(tw > 0, tw, np.inf))
    phase = float(np.sin(2.0 * np.pi * t / period))
    c = np.asarray(sphere_center, np.float64) + np.array([0.0, 1.0, 0.0]) * amplitude * phase
    oc = eye - c
    b = d @ oc
    disc = b * b - (oc @ oc - sphere_radius ** 2)
    ts = np.where(disc >= 0, -b - np.sqrt(np.maximum(disc, 0.0)), np.inf)
    rng_t = np.minimum(rng_t, np.where(ts > 0, ts, np.inf))
    hit = np.isfinite(rng_t)
    noise = np.random.default_rng(seed).normal(0.0, noise_std, size=n)
    pts = eye + d * (rng_t + noise)[:, None]
    pts = pts[hit]
    if max_points is not None:
        pts = pts[:max_points]
    return np.ascontiguousarray(pts)


# --------------------------------------------------------------------------
# map-side cases (parity tests)
# --------------------------------------------------------------------------


def rotation_from_quat(q) -> np.ndarray:
    x, y, z, w = (float(v) for v in q / np.linalg.norm(q))
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def random_pose(rng, translate: float = 0.3) -> np.ndarray:
    T = np.eye(4)
    T[:3, :3] = rotation_from_quat(rng.normal(size=4))
    T[:3, 3] = rng.uniform(-translate, translate, 3)
    return T


def insert_case(c: int) -> dict:
    rng = np.random.default_rng(1000 + c)
    dims = tuple(int(v) for v in rng.integers(2, 40, size=3))
    vs = float(rng.choice([0.02, 0.05, 0.1, 0.07, 1.0]))
    origin = tuple(float(v) for v in np.round(rng.uniform(-1, 1, 3), 3))
    lo, hi = grid_aabb(dims, vs, origin)
    pad = 0.2 * (hi - lo)
    clouds = []
    for _ in range(int(rng.integers(1, 4))):
        n = int(rng.integers(0, 3000)) if c else 0
        pts = rng.uniform(lo - pad, hi + pad, size=(n, 3))
        if n > 10:   # duplicates and exact voxel-boundary points
            pts[: n // 5] = pts[n // 5: 2 * (n // 5)]
            bidx = rng.integers(0, np.asarray(dims), size=(n // 10, 3))
            pts[2 * (n // 5): 2 * (n // 5) + n // 10] = lo + bidx * vs
        clouds.append(pts)
    pose = np.eye(4) if c % 3 else random_pose(rng, 0.1)
    mask_ijk = None
    if c % 2 == 1:
        k = int(rng.integers(1, 200))
        mask_ijk = rng.integers(0, np.asarray(dims), size=(k, 3)).astype(np.int32)
    hit = float(rng.choice([0.85, 0.3, 0.4, 1.7]))
    thr = float(rng.choice([0.5, 0.7, 0.55, 0.5124120603015075]))
    return {"dims": dims, "voxel_size": vs, "origin": origin, "clouds": clouds,
            "pose": pose, "mask_ijk": mask_ijk, "hit": hit, "thr": thr}


def stamp_case(c: int) -> dict:
    rng = np.random.default_rng(2000 + c)
    dims = tuple(int(v) for v in rng.integers(4, 48, size=3))
    vs = float(rng.choice([0.02, 0.04, 0.1]))
    origin = tuple(float(v) for v in np.round(rng.uniform(-0.5, 0.0, 3), 3))
    svs = vs * float(rng.choice([1.0, 0.5, 2.0]))
    set_origin = tuple(float(v) for v in rng.uniform(-0.3, 0.3, 3))
    k = int(rng.integers(1, 4000))
    ijk = rng.integers(0, 30, size=(k, 3)).astype(np.int32)
    T = None if c % 4 == 0 else random_pose(rng, 0.2)
    return {"dims": dims, "voxel_size": vs, "origin": origin, "set_origin": set_origin,
            "set_voxel_size": svs, "ijk": ijk, "T": T}


def site_world_case(c: int) -> dict:
    rng = np.random.default_rng(3000 + c)
    dims = tuple(int(v) for v in rng.integers(3, 40, size=3))
    vs = float(rng.choice([0.02, 0.05, 0.1]))
    origin = tuple(float(v) for v in rng.uniform(-1, 0, 3))
    occ = (rng.random(dims) < [0.0, 0.001, 0.01, 0.05, 0.2, 0.5][c]).astype(np.uint8)
    if c == 1 and not occ.any():
        occ[tuple(rng.integers(0, d) for d in dims)] = 1
    lo, hi = grid_aabb(dims, vs, origin)
    span = hi - lo
    centers = rng.uniform(lo - 0.3 * span, hi + 0.3 * span, size=(64, 3))  # some outside
    centers[:4] = [lo, hi, lo - 1e3, hi + 1e3]
    return {"occ": occ, "voxel_size": vs, "origin": origin, "centers": centers}


def arm_trajectory(q0, n: int):
    """q0 itself, then n-1 joint vectors near it (a deterministic sweep of
    joints 1..7)."""
    q0 = np.asarray(q0, np.float64)
    out = [q0.copy()]
    for s in range(1, n):
        q = q0.copy()
        q[1:] += 0.35 * np.sin(0.7 * s + np.arange(1, q.size))
        out.append(q)
    return out
