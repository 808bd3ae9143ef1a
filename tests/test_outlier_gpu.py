"""GPU statistical outlier filter (grids.py:224-240) against the reference's
own function (voxarm from baseline/_ref: scipy cKDTree + numpy).  The GPU
computes exact kNN distances as cKDTree does and sums in numpy's pairwise
order, so the surviving point arrays must be identical, not merely close."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(REF) and REF not in sys.path:
    sys.path.append(REF)
ref_grids = pytest.importorskip("voxarm.grids")

from paper_2407_02363_b200 import FilterConfig, PointCloud, VoxelGrid, synth  # noqa: E402
from paper_2407_02363_b200.grids import statistical_outlier_filter  # noqa: E402

pytestmark = pytest.mark.gpu


def _clouds():
    rng = np.random.default_rng(8)
    yield "normal", rng.normal(size=(5000, 3)) * 0.2
    yield "uniform", rng.uniform(-1, 1, size=(20000, 3))
    pts = rng.normal(size=(3000, 3)) * 0.05
    pts[:300] = pts[300:600]                      # exact duplicates
    pts[-5:] = rng.uniform(5, 6, size=(5, 3))     # far outliers
    yield "dups+far", pts
    yield "c1_sphere", synth.c1_cloud(0.1)
    yield "depth_camera", synth.depth_camera_cloud(0.2, max_points=120_000)
    flat = rng.uniform(-1, 1, size=(8000, 3))
    flat[:, 2] = 0.25                             # a plane (degenerate extent)
    yield "plane", flat


@pytest.mark.parametrize("k,m", [(8, 1.0), (1, 1.0), (5, 0.5), (16, 2.0), (31, 1.0)])
def test_filter_identical_to_reference(k, m):
    for name, pts in _clouds():
        want = ref_grids.statistical_outlier_filter(pts, k, m)
        got = statistical_outlier_filter(pts, k, m)
        assert np.array_equal(got, want), (name, k, m, got.shape, want.shape)


def test_reference_known_answers():           # pkg/tests/test_grids.py:58-81
    pts = np.zeros((11, 3))
    pts[:10] += np.linspace(0, 0.01, 10)[:, None]
    pts[10] = (10.0, 0.0, 0.0)
    kept = statistical_outlier_filter(pts, 5, 1.0)
    assert np.array_equal(kept, ref_grids.statistical_outlier_filter(pts, 5, 1.0))
    assert not (kept == pts[10]).all(axis=1).any()
    ident = np.tile([[1.0, 2.0, 3.0]], (20, 1))
    assert statistical_outlier_filter(ident, 5, 1.0).shape == (20, 3)
    small = np.random.default_rng(0).normal(size=(4, 3))
    assert np.array_equal(statistical_outlier_filter(small, 5, 1.0), small)
    assert statistical_outlier_filter(np.empty((0, 3)), 5, 1.0).shape == (0, 3)


def test_insert_with_filter_matches_reference():
    cfg_kw = dict(k_neighbors=8, std_multiplier=1.0)
    for t in (0.0, 0.3):
        pts = synth.c1_cloud(t)
        pts = np.vstack([pts, np.random.default_rng(3).uniform(-1.2, 1.2, size=(200, 3))])
        spec = synth.C1
        ref = ref_grids.VoxelGrid(spec["dims"], spec["voxel_size"], spec["origin"])
        rst = ref.insert_point_cloud(ref_grids.PointCloud(pts), ref_grids.FilterConfig(**cfg_kw))
        g = VoxelGrid(spec["dims"], spec["voxel_size"], spec["origin"])
        st = g.insert_point_cloud(PointCloud(pts), FilterConfig(**cfg_kw))
        assert (st.inserted, st.outliers_removed, st.robot_skipped, st.out_of_bounds) == \
            (rst.inserted, rst.outliers_removed, rst.robot_skipped, rst.out_of_bounds)
        assert st.outliers_removed > 0
        assert np.array_equal(g.cells, ref.cells)
