"""K7 on-device avoidance rows against the reference's
own row builder, voxarm tasks.py:88-123 (_distance_rows), fed with the sites
the same device tick gathered.  Floating point: x, xdot_ref and the Jacobian
rows within rtol 1e-6 (the north-star tolerance for metric outputs; the
device sums the 3-vector products in a fixed order, numpy's matmul may fuse),
activation within 1e-9."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(REF) and REF not in sys.path:
    sys.path.append(REF)
voxarm = pytest.importorskip("voxarm")

from paper_2407_02363_b200 import synth  # noqa: E402
from paper_2407_02363_b200.engine import MapCycle  # noqa: E402

pytestmark = pytest.mark.gpu


def _setup(vs=0.02):
    from voxarm.robot import load_robot, self_obstacle_links, shipped_robot_path, voxelize_link
    chain = load_robot(shipped_robot_path())
    spheres = chain.build_spheres()
    links = [(v.indices, v.origin) for v in (voxelize_link(l, vs) for l in chain.links)]
    s = synth.C1
    cyc = MapCycle(s["dims"], s["voxel_size"], s["origin"], links, vs, self_obstacle_links(chain),
                   max_points=s["points"] + 1000, max_spheres=len(spheres))
    return chain, spheres, cyc


def _ref_rows(chain, q, spheres, centers, lin, world, cfg, label):
    from voxarm.tasks import _distance_rows
    sites = [None if lin[i] < 0 else world[i] for i in range(len(spheres))]
    return _distance_rows(chain, q, spheres, centers, sites, cfg, None, label)


@pytest.mark.parametrize("offset", [None, 0.12], ids=["offset-2b", "offset-0.12"])
def test_rows_match_reference_row_builder(offset):
    from voxarm.tasks import AvoidanceConfig
    chain, spheres, cyc = _setup()
    cfg = AvoidanceConfig(kappa=10.0, x_star_offset=offset)
    cyc.set_avoidance([s.radius for s in spheres], [s.buffer for s in spheres],
                      [s.link_index for s in spheres], chain.n, cfg.kappa, cfg.x_star_offset)
    rng = np.random.default_rng(3)
    active = 0
    for t in range(6):
        q = rng.uniform(chain.q_min, chain.q_max) * 0.6
        frames = chain.forward_kinematics(q)
        centers = np.array([frames[s.link_index][:3, :3] @ s.center + frames[s.link_index][:3, 3]
                            for s in spheres])
        # the cloud plus points scattered around the arm, so rows sit inside
        # their transition bands
        near = centers[rng.integers(0, len(spheres), 400)] + rng.normal(0, 0.08, (400, 3))
        pts = np.vstack([synth.c1_cloud(t / 30.0), near])
        cyc.set_joint_frames(*chain.joint_frames(q))
        cyc.step(pts, np.stack(frames[:chain.n]), centers)
        res = cyc.wait()
        rows = cyc.rows()
        for key, label in (("env", "obstacle_avoidance"), ("self", "self_collision")):
            lin, world, _ = res[key]
            lv = _ref_rows(chain, q, spheres, centers, lin, world, cfg, label)
            got = rows[key]
            assert np.array_equal(got["flag"], np.where(lin < 0, 0, 1)), key
            assert np.array_equal(np.isinf(got["value"]), np.isinf(lv.task_values))
            fin = np.isfinite(lv.task_values)
            np.testing.assert_allclose(got["value"][fin], lv.task_values[fin], rtol=1e-12)
            np.testing.assert_allclose(got["activation"], lv.activation, rtol=0, atol=1e-9)
            np.testing.assert_allclose(got["xdot_ref"], lv.xdot_ref, rtol=1e-6, atol=1e-12)
            np.testing.assert_allclose(got["J"], lv.J, rtol=1e-6, atol=1e-12)
            active += int(((lv.activation > 0) & (lv.activation < 1)).sum())
    assert active > 0   # the cosine ramp was exercised


def test_rows_disabled_and_bad_arguments():
    chain, spheres, cyc = _setup()
    n = len(spheres)
    with pytest.raises(ValueError):
        cyc.set_avoidance([0.05] * n, [0.0] * n, [0] * n, chain.n, 2.0)    # b must be > 0
    with pytest.raises(ValueError):
        cyc.set_avoidance([0.05] * n, [0.02] * n, [chain.n] * n, chain.n, 2.0)   # link range
    with pytest.raises(ValueError):
        cyc.set_avoidance([0.05] * n, [0.02] * n, [0] * n, chain.n, 0.0)   # kappa > 0
    with pytest.raises(ValueError):
        cyc.set_joint_frames(np.zeros((chain.n, 3)), np.zeros((chain.n, 3)))   # not enabled
