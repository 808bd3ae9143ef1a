"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

It imports voxarm from /root/reference/pkg/src and records what the reference
itself returns on seeded inputs, so that the oracle (oracle/) and the CUDA
path can be pinned on the GPU box, where /root/reference does not exist.

Outputs
  edt_cases.npz   small random grids: occupancy, pba_edt site, pass-1 s1
  golden.json     blake2b digests of reference outputs at larger sizes,
                  map-insert / stamp / site-world cases, the C1 cycle
  ../../paper_2407_02363_b200/data/desk7_2cm.npz
                  desk7 link voxel sets (robot.voxelize_link), sphere
                  link/centre table (build_spheres), FK frames for a q list
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import voxarm  # noqa: E402
from voxarm import BandConfig, line_nearest_sites, pba_edt  # noqa: E402
from voxarm.engine import SimEngine  # noqa: E402
from voxarm.grids import FilterConfig, PointCloud, VoxelGrid, VoxelSet  # noqa: E402
from voxarm.movers import OscillatingMover  # noqa: E402
from voxarm.robot import (Sphere, load_robot, self_obstacle_links,  # noqa: E402
                          shipped_robot_path, voxelize_link)

from paper_2407_02363_b200 import synth  # noqa: E402  (input generators)


def digest(a: np.ndarray) -> str:
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=16).hexdigest()


GUARD_Q = [0, 0, 0.2, 0, 0.5, 0, 0.3, 0]


def edt_cases():
    rng = np.random.default_rng(2026)
    arrays = {}
    meta = []
    dims_list = []
    # random grids (test_acceptance.py:35-55 style: dims 4-32, density 1-50%)
    for c in range(48):
        dims = tuple(int(d) for d in rng.integers(1, 33, size=3))
        dims_list.append(dims)
    # thin grids on every axis (test_edt.py:209-218)
    dims_list += [(1, 24, 16), (24, 1, 16), (24, 16, 1), (1, 1, 30), (30, 1, 1),
                  (1, 30, 1), (2, 2, 2), (1, 1, 1), (3, 2, 1), (5, 5, 5)]
    for c, dims in enumerate(dims_list):
        dens = float(rng.uniform(0.0, 0.6)) if c % 7 else float(rng.uniform(0.0, 0.03))
        occ = rng.random(dims) < dens
        bands = [int(v) for v in rng.integers(1, 6, size=3)]
        site = pba_edt(occ, BandConfig(*bands)).site
        s1 = line_nearest_sites(occ, m1=bands[0])
        arrays[f"occ{c}"] = occ.astype(np.uint8)
        arrays[f"site{c}"] = site
        arrays[f"s1_{c}"] = s1
        meta.append({"dims": list(dims), "bands": bands})
    np.savez_compressed(os.path.join(HERE, "edt_cases.npz"), **arrays)
    return meta


def edt_digests():
    out = []
    specs = [((16, 16, 16), 0.08, 16), ((64, 64, 64), 0.02, 0), ((128, 128, 128), 0.02, 0),
             ((128, 128, 128), 1e-4, 1), ((128, 128, 128), 0.3, 2), ((96, 96, 128), 0.02, 3),
             ((192, 192, 128), 0.02, 3), ((100, 37, 133), 0.05, 5), ((256, 256, 256), 0.02, 0),
             ((512, 512, 512), 0.02, 0)]
    for dims, p, seed in specs:
        occ = synth.bernoulli_occupancy(dims, p, seed)
        f = pba_edt(occ)
        rec = {"gen": "bernoulli", "dims": list(dims), "p": p, "seed": seed,
               "site": digest(f.site)}
        if np.prod(dims) <= 128 ** 3:
            rec["s1"] = digest(line_nearest_sites(occ))
            rec["sq"] = digest(f.sq_distance_grid())
        out.append(rec)
        print("edt", dims, p, seed, flush=True)
    for name, dims in [("single_center", (128, 128, 128)), ("single_corner", (128, 128, 128)),
                       ("full", (64, 64, 64)), ("empty", (64, 64, 64)),
                       ("single_center", (256, 256, 256))]:
        occ = synth.structured_occupancy(name, dims)
        f = pba_edt(occ)
        out.append({"gen": name, "dims": list(dims), "site": digest(f.site)})
    return out


def insert_cases():
    """grids.py insert/stamp semantics on seeded inputs (synth.insert_case)."""
    out = []
    for c in range(24):
        case = synth.insert_case(c)
        g = VoxelGrid(case["dims"], case["voxel_size"], case["origin"])
        mask = None
        if case["mask_ijk"] is not None:
            mask = VoxelGrid(case["dims"], case["voxel_size"], case["origin"])
            mask.insert_voxel_set(VoxelSet(case["origin"], case["voxel_size"], case["mask_ijk"]))
        cfg = FilterConfig(k_neighbors=0, hit_logodds=case["hit"],
                           occupancy_threshold=case["thr"])
        stats = []
        for pts in case["clouds"]:
            st = g.insert_point_cloud(PointCloud(pts, case["pose"]), cfg, mask)
            stats.append([st.inserted, st.robot_skipped, st.out_of_bounds])
        out.append({"case": c, "stats": stats, "cells": digest(g.cells),
                    "occ": digest(g.occupancy_mask(case["thr"])),
                    "n_occ": int(g.occupancy_mask(case["thr"]).sum())})
    return out


def stamp_cases():
    out = []
    for c in range(16):
        case = synth.stamp_case(c)
        g = VoxelGrid(case["dims"], case["voxel_size"], case["origin"])
        oob = g.insert_voxel_set(VoxelSet(case["set_origin"], case["set_voxel_size"],
                                          case["ijk"]), case["T"])
        out.append({"case": c, "oob": oob, "cells": digest(g.cells),
                    "occupied": g.occupied_voxels().tolist() if c < 4 else None})
    return out


def desk7():
    chain = load_robot(shipped_robot_path())
    links = [voxelize_link(link, 0.02) for link in chain.links]
    spheres = chain.build_spheres()
    qs = synth.arm_trajectory(GUARD_Q, 8)
    frames = np.array([[f for f in chain.forward_kinematics(q)] for q in qs])
    arrays = {"q": np.asarray(qs), "frames": frames,
              "sphere_link": np.array([s.link_index for s in spheres], np.int32),
              "sphere_center": np.array([s.center for s in spheres]),
              "sphere_radius": np.array([s.radius for s in spheres]),
              "o_links": np.array(self_obstacle_links(chain), np.int32)}
    for li, vs in enumerate(links):
        arrays[f"link{li}_ijk"] = vs.indices
        arrays[f"link{li}_origin"] = vs.origin
    np.savez_compressed(os.path.join(HERE, "..", "..", "paper_2407_02363_b200", "data", "desk7_2cm.npz"),
                        **arrays)
    return chain, links


class _FakeEngine:
    """Just the attributes SimEngine._site_world reads (engine.py:212-221)."""

    def __init__(self, fld, origin, vs, dims):
        self._fields = {"env": fld}
        self._origin = np.asarray(origin, np.float64)
        self._dims = np.asarray(dims, np.int64)

        class _G:
            voxel_size = vs

        class _S:
            grid = _G

        self.sc = _S


def site_world_cases():
    out = []
    for c in range(6):
        case = synth.site_world_case(c)
        occ = case["occ"]
        fld = pba_edt(occ, voxel_size=case["voxel_size"])
        eng = _FakeEngine(fld, case["origin"], case["voxel_size"], occ.shape)
        worlds, dists = [], []
        for ctr in case["centers"]:
            w = SimEngine._site_world(eng, "env", ctr)
            if w is None:
                worlds.append(None)
                dists.append(None)
            else:
                worlds.append([float(v) for v in w])
                dists.append(float(np.linalg.norm(w - ctr)))   # tasks.py:102-104
        out.append({"case": c, "world": worlds, "dist": dists})
    return out


def c1_cycle(chain, links):
    """One C1 camera tick (engine.py:234-268 + 272-280) at 128^3, k=0."""
    spec = synth.C1
    dims, vs, origin = spec["dims"], spec["voxel_size"], spec["origin"]
    env = VoxelGrid(dims, vs, origin)
    selfg = VoxelGrid(dims, vs, origin)
    mask = VoxelGrid(dims, vs, origin)
    q = np.asarray(GUARD_Q, np.float64)
    frames = chain.forward_kinematics(q)
    o_links = self_obstacle_links(chain)
    for li in o_links:
        selfg.insert_voxel_set(links[li], frames[li])
    for li in range(chain.n):
        mask.insert_voxel_set(links[li], frames[li])
    res = {}
    for f in (0, 5, 17):
        t = f / 30.0
        mover = OscillatingMover(0, Sphere((0, 0, 0), spec["obstacle_radius"]), spec["points"],
                                 0.0, spec["seed"], center=spec["obstacle_center"],
                                 axis=(0, 1, 0), amplitude=0.2, period=1.5)
        pts = mover.cloud_points(t)
        assert np.array_equal(pts, synth.c1_cloud(t)), "synth.c1_cloud diverged from voxarm"
        env.clear()
        st = env.insert_point_cloud(PointCloud(pts), FilterConfig(k_neighbors=0), robot_mask=mask)
        occ_env = env.occupancy_mask()
        fe = pba_edt(occ_env, voxel_size=vs)
        res[f] = {"stats": [st.inserted, st.robot_skipped, st.out_of_bounds],
                  "cloud": digest(pts), "env_cells": digest(env.cells),
                  "env_occ": digest(occ_env), "env_site": digest(fe.site)}
        centers = synth.c1_sphere_centers_from(chain, q)
        eng = _FakeEngine(fe, origin, vs, dims)
        res[f]["env_world"] = [None if w is None else [float(v) for v in w]
                               for w in (SimEngine._site_world(eng, "env", c) for c in centers)]
    fs = pba_edt(selfg.occupancy_mask(), voxel_size=vs)
    res["self_cells"] = digest(selfg.cells)
    res["mask_cells"] = digest(mask.cells)
    res["self_site"] = digest(fs.site)
    centers = synth.c1_sphere_centers_from(chain, q)
    eng = _FakeEngine(fs, origin, vs, dims)
    res["self_world"] = [None if w is None else [float(v) for v in w]
                         for w in (SimEngine._site_world(eng, "env", c) for c in centers)]
    res["centers"] = digest(np.asarray(centers))
    return res


def edt_digests_1024():
    """Config C5 inputs at 1024^3 (about 40 s and 17 GB each with numba)."""
    out = []
    for dims, p, seed in [((1024, 1024, 1024), 0.02, 0), ((1024, 1024, 1024), 1e-4, 1)]:
        occ = synth.bernoulli_occupancy(dims, p, seed)
        out.append({"gen": "bernoulli", "dims": list(dims), "p": p, "seed": seed,
                    "site": digest(pba_edt(occ).site)})
        del occ
    return out


def bench512_tick0():
    """bench.py's headline tick 0 (512^3, 300k-point depth camera, desk7 mask
    at the step's frames) through voxarm's own grids and pba_edt."""
    import bench
    d = synth.desk7_model()
    pts, frames, centers = bench.scene_inputs(0, 0, d)
    dims, vs, origin = bench.DIMS, bench.VS, bench.ORIGIN
    mask = VoxelGrid(dims, vs, origin)
    for li, (ijk, org) in enumerate(d["links"]):
        mask.insert_voxel_set(VoxelSet(np.asarray(org, np.float64), vs, ijk), frames[li])
    env = VoxelGrid(dims, vs, origin)
    st = env.insert_point_cloud(PointCloud(pts), FilterConfig(k_neighbors=0), robot_mask=mask)
    occ = env.occupancy_mask()
    fe = pba_edt(occ, voxel_size=vs)
    eng = _FakeEngine(fe, origin, vs, dims)
    return {"stats": [st.inserted, st.robot_skipped, st.out_of_bounds], "occ": digest(occ),
            "site": digest(fe.site), "cloud": digest(pts),
            "env_world": [None if w is None else [float(v) for v in w]
                          for w in (SimEngine._site_world(eng, "env", c) for c in centers)]}


def main():
    if "--bench512" in sys.argv:   # only the headline digest, merged into golden.json
        path = os.path.join(HERE, "golden.json")
        with open(path) as fh:
            gold = json.load(fh)
        gold["bench512_tick0"] = bench512_tick0()
        with open(path, "w") as fh:
            json.dump(gold, fh, indent=1)
        return
    if "--big" in sys.argv:   # only the 1024^3 digests, merged into golden.json
        path = os.path.join(HERE, "golden.json")
        with open(path) as fh:
            gold = json.load(fh)
        gold["edt_digests_1024"] = edt_digests_1024()
        with open(path, "w") as fh:
            json.dump(gold, fh, indent=1)
        return
    gold = {"reference": "voxarm @ /root/reference/pkg/src", "numpy": np.__version__}
    gold["edt_cases"] = edt_cases()
    chain, links = desk7()
    gold["insert"] = insert_cases()
    gold["stamp"] = stamp_cases()
    gold["site_world"] = site_world_cases()
    gold["c1"] = c1_cycle(chain, links)
    gold["edt_digests"] = edt_digests()
    old = os.path.join(HERE, "golden.json")
    if os.path.exists(old):   # keep the (slow) 1024^3 digests from a --big run
        with open(old) as fh:
            prev = json.load(fh)
        if "edt_digests_1024" in prev:
            gold["edt_digests_1024"] = prev["edt_digests_1024"]
        if "bench512_tick0" in prev:
            gold["bench512_tick0"] = prev["bench512_tick0"]
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(gold, fh, indent=1)
    print("wrote", HERE)


if __name__ == "__main__":
    main()
