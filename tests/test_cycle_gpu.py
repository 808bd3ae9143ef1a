"""The device-resident camera tick (MapCycle / vx_cycle_step, engine.py:233-280)
against the reference's own C1 tick (golden vectors from voxarm) and the
oracle: stats, env/self/mask cells, both EDT fields and the sphere gather."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_02363_b200 import synth
from paper_2407_02363_b200.engine import MapCycle
from tests.golden_util import desk7, digest, golden

pytestmark = pytest.mark.gpu


def _c1_cycle():
    d = desk7()
    s = synth.C1
    return MapCycle(s["dims"], s["voxel_size"], s["origin"], d["links"], s["voxel_size"], d["o_links"],
                    max_points=s["points"], max_spheres=32), d


def test_c1_cycle_vs_reference_golden():
    gold = golden()["c1"]
    cyc, d = _c1_cycle()
    s = synth.C1
    frames = d["frames"][0]
    centers = np.vstack([synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"]),
                         synth.extra_query_points(s["dims"], s["voxel_size"], s["origin"])])
    for f in ("0", "5", "17"):
        cyc.step(synth.c1_cloud(int(f) / 30.0), frames, centers)
        res = cyc.wait()
        assert [res["inserted"], res["robot_skipped"], res["out_of_bounds"]] == gold[f]["stats"]
        env, selfg, mask = cyc.grids()
        assert digest(env.cells) == gold[f]["env_cells"]
        assert digest(mask.cells) == gold["mask_cells"]
        assert digest(selfg.cells) == gold["self_cells"]
        fe, fs = cyc.fields()
        assert digest(fe.site) == gold[f]["env_site"]
        assert digest(fs.site) == gold["self_site"]
        lin, world, dist = res["env"]
        for q, w in enumerate(gold[f]["env_world"]):
            assert (lin[q] == -1) if w is None else (world[q].tolist() == w)
        lin, world, dist = res["self"]
        for q, w in enumerate(gold["self_world"]):
            assert (lin[q] == -1) if w is None else (world[q].tolist() == w)
        assert res["self_recomputed"] == (f == "0")   # memo: static torso


def test_cycle_moving_arm_vs_oracle():
    """FK frames change every tick (mask + self recomputed when o_links move)."""
    cyc, d = _c1_cycle()
    s = synth.C1
    dims, vs, origin = s["dims"], s["voxel_size"], s["origin"]
    for step in range(4):
        frames = d["frames"][step].copy()
        if step >= 2:     # move the torso too: the self map must be rebuilt
            frames[0][:3, 3] += 0.013 * step
        centers = synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"])
        pts = synth.c1_cloud(step / 30.0)
        cyc.step(pts, frames, centers)
        res = cyc.wait()
        selfc = np.zeros(dims, np.float32)
        maskc = np.zeros(dims, np.float32)
        for li in d["o_links"]:
            ijk, org = d["links"][li]
            O.stamp_voxels(selfc, vs, origin, ijk, org, vs, frames[li])
        for li, (ijk, org) in enumerate(d["links"]):
            O.stamp_voxels(maskc, vs, origin, ijk, org, vs, frames[li])
        env = np.zeros(dims, np.float32)
        st = O.insert_points(env, vs, origin, pts, maskc)
        assert (res["inserted"], res["robot_skipped"], res["out_of_bounds"]) == st
        site_e = O.pba_edt_site(env > 0)
        site_s = O.pba_edt_site(selfc > 0)
        fe, fs = cyc.fields()
        assert np.array_equal(fe.site, site_e)
        assert np.array_equal(fs.site, site_s)
        for key, site in (("env", site_e), ("self", site_s)):
            lin, world, dist = res[key]
            rl, rw, rd = O.site_world(site, vs, origin, centers)
            assert np.array_equal(lin, rl)
            ok = rl >= 0
            assert np.array_equal(world[ok], rw[ok])
            np.testing.assert_allclose(dist[ok], rd[ok], rtol=1e-6)   # north_star tolerance
        assert res["self_recomputed"] == (step in (0, 2, 3))


def test_graph_and_direct_launch_agree():
    """The CUDA-graph replay of the tick equals direct launches, across cloud
    sizes (the point count is read on the device inside the graph)."""
    from paper_2407_02363_b200 import _lib
    d = desk7()
    s = synth.C1
    outs = []
    for graph in (1, 0):
        cyc, _ = _c1_cycle()
        _lib.check(_lib.load().vx_cycle_use_graph(cyc._h, graph))
        res = []
        for step, npts in enumerate([50_000, 1234, 0, 50_000]):
            frames = d["frames"][step]
            centers = synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"])
            cyc.step(synth.c1_cloud(step / 30.0)[:npts], frames, centers)
            r = cyc.wait()
            fe, _ = cyc.fields()
            res.append((r["inserted"], r["robot_skipped"], r["out_of_bounds"], digest(fe.site),
                        r["env"][0].tolist(), r["self"][2].tolist()))
        outs.append(res)
        cyc.close()
    assert outs[0] == outs[1]


@pytest.mark.parametrize("which", ["env", "mask"])
def test_graph_tick_after_host_cell_writes(which):
    """Host writes to a cycle grid between ticks (MapCycle.grids() hands out
    writable grids) leave cells off the touched list and possibly out of
    range: the next replayed graph tick must reset that grid densely, exactly
    as the direct-launch tick does (the captured reset mode)."""
    from paper_2407_02363_b200 import _lib
    d = desk7()
    s = synth.C1
    rng = np.random.default_rng(5)
    junk = rng.uniform(-4.0, 6.0, s["dims"]).astype(np.float32)   # includes out-of-range values
    junk[rng.random(s["dims"]) < 0.5] = -0.0
    outs = []
    for graph in (1, 0):
        cyc, _ = _c1_cycle()
        _lib.check(_lib.load().vx_cycle_use_graph(cyc._h, graph))
        res = []
        for step in range(4):
            frames = d["frames"][step]
            centers = synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"])
            if step in (1, 3):   # after the graph exists: scribble on the grid
                env, _, mask = cyc.grids()
                (env if which == "env" else mask).cells = junk
            cyc.step(synth.c1_cloud(step / 30.0), frames, centers)
            r = cyc.wait()
            env, _, mask = cyc.grids()
            fe, _ = cyc.fields()
            res.append((r["inserted"], r["robot_skipped"], digest(env.cells), digest(mask.cells),
                        digest(fe.site), r["env"][2].tolist()))
        outs.append(res)
        cyc.close()
    assert outs[0] == outs[1]
    # and the tick after a write equals a tick on a never-written cycle
    ref, _ = _c1_cycle()
    frames = d["frames"][3]
    ref.step(synth.c1_cloud(3 / 30.0), frames,
             synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"]))
    r = ref.wait()
    env, _, mask = ref.grids()
    fe, _ = ref.fields()
    assert outs[0][3][:5] == (r["inserted"], r["robot_skipped"], digest(env.cells),
                              digest(mask.cells), digest(fe.site))


def test_prefetch_matches_plain_step():
    """vx_cycle_prefetch: the staged cloud gives the same tick as a plain step
    (and a stale / mismatched prefetch is ignored, not used)."""
    from paper_2407_02363_b200 import _lib
    s = synth.C1
    d = desk7()
    frames = d["frames"][0]
    centers = synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"])
    clouds = []
    for f in (0, 5, 17):
        pa = _lib.PinnedArray((s["points"], 3), np.float64)
        pa.array[...] = synth.c1_cloud(f / 30.0)
        clouds.append(pa)
    ref, _ = _c1_cycle()
    want = []
    for pa in clouds:
        ref.step(pa.array, frames, centers)
        r = ref.wait()
        fe, _ = ref.fields()
        want.append((r["inserted"], digest(fe.site), r["env"][2].copy()))
    cyc, _ = _c1_cycle()
    tk = cyc.prefetch(clouds[0].array)
    for q, pa in enumerate(clouds):
        cyc.step(tk, frames, centers, sync=False)
        if q + 1 < len(clouds):
            tk = cyc.prefetch(clouds[q + 1].array)
        r = cyc.wait()
        fe, _ = cyc.fields()
        assert (r["inserted"], digest(fe.site)) == want[q][:2], q
        assert np.array_equal(r["env"][2], want[q][2])
    # a staged cloud never leaks into a plain step of another buffer
    cyc.prefetch(clouds[2].array)
    cyc.step(clouds[0].array, frames, centers)
    r = cyc.wait()
    assert r["inserted"] == want[0][0]
    # a consumed ticket and an overwritten one fail loudly, never a stale cloud
    used = cyc.prefetch(clouds[1].array)
    cyc.step(used, frames, centers)
    cyc.wait()
    with pytest.raises(ValueError):
        cyc.step(used, frames, centers)
    old = cyc.prefetch(clouds[0].array)
    cyc.prefetch(clouds[1].array)
    cyc.prefetch(clouds[2].array)   # third prefetch: overwrites `old`'s slot
    with pytest.raises(ValueError):
        cyc.step(old, frames, centers)
    tk = cyc.prefetch(clouds[1].array)   # a fresh ticket after the failures still works
    cyc.step(tk, frames, centers)
    assert cyc.wait()["inserted"] == want[1][0]


@pytest.mark.parametrize("dims", [(96, 80, 72), (130, 64, 36), (64, 128, 30)],
                         ids=lambda d: "x".join(map(str, d)))
def test_cycle_odd_dims_matches_plain_calls(dims):
    """The fused tick on grids whose extents are not multiples of 32 (ragged
    k tiles; nz % 4 != 0 takes the non-TMA column kernels): its env field and
    gather equal a plain EDT of its occupancy and site_world on it."""
    from paper_2407_02363_b200 import pba_edt
    from paper_2407_02363_b200.engine import site_world
    vs = 0.02
    origin = np.array([-0.5, -0.6, -0.1])
    d = desk7()
    cyc = MapCycle(dims, vs, origin, d["links"], vs, d["o_links"], max_points=20000, max_spheres=16)
    rng = np.random.default_rng(sum(dims))
    ext = np.array(dims) * vs
    frames = d["frames"][1]
    for t in range(3):
        pts = origin + rng.random((20000, 3)) * ext * np.array([1.0, 1.0, 0.6])
        centers = origin + rng.random((16, 3)) * ext
        cyc.step(pts, frames, centers)
        res = cyc.wait()
        env, _, _ = cyc.grids()
        fe, _ = cyc.fields()
        want = pba_edt(env.occupancy_mask())
        assert np.array_equal(fe.site, want.site), t
        lin, world, dist = site_world(want, origin, vs, centers)
        assert np.array_equal(res["env"][0], lin)
        assert np.array_equal(res["env"][1], world)
        assert np.allclose(res["env"][2], dist, rtol=1e-12, equal_nan=True)
