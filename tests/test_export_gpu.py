"""Device export formats against the oracle and the
reference's host formulas: sq_distance_grid (edt.py:123-135), dump_squared
(edt.py:137-145, golden test_edt.py:248-253) and occupied_voxels
(grids.py:210-212).  Integer/byte work: bit-exact."""
import io
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_02363_b200.edt import DistanceField, pba_edt
from paper_2407_02363_b200.grids import FilterConfig, PointCloud, VoxelGrid

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1, 1), (3, 2, 1), (7, 5, 3), (37, 5, 33), (16, 40, 129), (64, 64, 64), (128, 96, 160)]


def _occ(shape, p, seed):
    return np.random.default_rng(seed).random(shape) < p


def _host_dump(site):
    buf = io.StringIO()
    DistanceField(site, 1.0).dump_squared(buf)   # the host formatter (edt.py:137-145)
    return buf.getvalue()


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("p", [0.0, 0.01, 0.3])
def test_sq_distance_grid_device(shape, p):
    occ = _occ(shape, p, 1)
    f = pba_edt(occ)
    assert f._device_only()
    got = f.sq_distance_grid()
    assert got.dtype == np.int64 and got.shape == shape
    assert np.array_equal(got, O.sq_distance_grid(O.pba_edt_site(occ)))


@pytest.mark.parametrize("shape", SHAPES[:6], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("p", [0.0, 0.02])
def test_dump_squared_device_matches_host_format(shape, p):
    occ = _occ(shape, p, 2)
    f = pba_edt(occ)
    buf = io.StringIO()
    f.dump_squared(buf)
    assert buf.getvalue() == _host_dump(O.pba_edt_site(occ))


def test_dump_squared_device_golden():                   # test_edt.py:248-253
    occ = np.zeros((3, 2, 1), bool)
    occ[0, 0, 0] = True
    f = pba_edt(occ)
    assert f._device_only()
    buf = io.StringIO()
    f.dump_squared(buf)
    assert buf.getvalue() == "slice k=0\n0 1 4\n1 2 5\n"


def test_host_edits_win_over_the_device_copy():
    f = pba_edt(_occ((4, 4, 4), 0.2, 3))
    site = f.site                  # materialise, then edit in place
    site[0, 0, 0] = 63
    assert f.sq_distance_grid()[0, 0, 0] == 27


@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 5, 3), (33, 17, 9), (64, 64, 64), (100, 90, 80)],
                         ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("thr", [0.5, 0.7, 0.2])
def test_occupied_voxels_device(shape, thr):
    g = VoxelGrid(shape, 0.05, (0.0, 0.0, 0.0))
    rng = np.random.default_rng(4)
    cells = rng.uniform(-2.0, 3.5, shape).astype(np.float32)
    cells[rng.random(shape) < 0.7] = 0.0
    g.cells[:] = cells
    got = g.occupied_voxels(thr)
    want = np.argwhere(cells > math.log(thr / (1.0 - thr)))   # NEP 50: f32 compare
    assert got.dtype == want.dtype and np.array_equal(got, want)


def test_occupied_voxels_empty_and_after_insert():
    g = VoxelGrid((20, 30, 40), 0.1, (0.0, 0.0, 0.0))
    assert g.occupied_voxels().shape == (0, 3)
    pts = np.random.default_rng(5).uniform(0.0, 1.9, (500, 3))
    g.insert_point_cloud(PointCloud(pts), FilterConfig(k_neighbors=0))
    assert np.array_equal(g.occupied_voxels(), np.argwhere(g.cells > 0))
