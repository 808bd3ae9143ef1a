"""GPU EDT parity: the sm_100a K3/K4/K5 path vs the reference.

Bit-exact `site` arrays (integer work: no tolerance), checked against
  * golden vectors produced by the reference itself (tests/golden),
  * blake2b digests of reference outputs up to 512^3,
  * the CPU oracle (oracle/, pinned by test_oracle_golden.py) on seeded
    random grids, thin grids, degenerate grids and the wide/global-stack
    code paths,
  * the reference's own known-answer tests (pkg/tests/test_edt.py).
"""

import io
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_02363_b200 import (NO_SITE, BandConfig, line_nearest_sites, pba_edt,
                                   query_nearest_site, synth)
from tests.golden_util import digest, edt_cases, golden

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_golden_cases_bit_exact():
    for occ, site, s1, bands in edt_cases():
        got = pba_edt(occ, BandConfig(*bands))
        assert np.array_equal(got.site, site), occ.shape
        assert np.array_equal(line_nearest_sites(occ, bands[0]), s1), occ.shape


@pytest.mark.parametrize("rec", golden()["edt_digests"],
                         ids=lambda r: f"{r['gen']}-{'x'.join(map(str, r['dims']))}-{r.get('p', '')}")
def test_reference_digests(rec):
    if rec["gen"] == "bernoulli":
        occ = synth.bernoulli_occupancy(rec["dims"], rec["p"], rec["seed"])
    else:
        occ = synth.structured_occupancy(rec["gen"], rec["dims"])
    f = pba_edt(occ)
    assert digest(f.site) == rec["site"]
    if "s1" in rec:
        assert digest(line_nearest_sites(occ)) == rec["s1"]
        assert digest(f.sq_distance_grid()) == rec["sq"]


def test_random_grids_vs_oracle():
    rng = np.random.default_rng(77)
    for _ in range(150):
        dims = tuple(int(d) for d in rng.integers(1, 48, size=3))
        p = float(rng.choice([0.0005, 0.01, 0.05, 0.2, 0.5, 0.9]))
        occ = rng.random(dims) < p
        assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), (dims, p)


def test_thin_and_degenerate_grids():
    rng = np.random.default_rng(55)   # test_edt.py:209-218 plus more
    shapes = [(1, 24, 16), (24, 1, 16), (24, 16, 1), (1, 1, 30), (30, 1, 1), (1, 30, 1),
              (2, 2, 2), (1, 1, 1), (1, 1, 4097), (4097, 1, 1), (1, 4097, 1), (3, 5, 2100),
              (33, 65, 129), (130, 3, 7), (300, 7, 36), (5, 700, 20), (257, 513, 4)]
    for dims in shapes:
        for p in (0.0, 0.001, 0.25, 1.0):
            occ = rng.random(dims) < p
            assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), (dims, p)


def test_structured_extremes():
    for name in ("single_center", "single_corner", "two_corners", "full", "empty"):
        for dims in [(64, 64, 64), (37, 91, 53)]:
            occ = synth.structured_occupancy(name, dims)
            assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), (name, dims)


def test_long_columns_global_stack():
    # column lengths beyond the shared-memory stack limit (2000 x 32 x 4 B)
    rng = np.random.default_rng(3)
    for dims in [(2000, 3, 33), (3, 2100, 5), (1800, 40, 2)]:
        for p in (0.001, 0.05, 0.6):
            occ = rng.random(dims) < p
            assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), (dims, p)


_SUB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from oracle import oracle as O
from paper_2407_02363_b200 import pba_edt, synth
rng = np.random.default_rng(9)
for _ in range(40):
    dims = tuple(int(d) for d in rng.integers(1, 40, size=3))
    occ = rng.random(dims) < float(rng.choice([0.002, 0.05, 0.4]))
    assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), dims
for dims, p in [((128, 64, 96), 1e-4), ((96, 80, 64), 0.01)]:
    occ = synth.bernoulli_occupancy(dims, p, 4)
    assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), dims
print("ok")
"""


@pytest.mark.parametrize("env", [{"VX_FORCE_WIDE": "1"}, {"VX_FORCE_WIDE": "2"}, {"VX_FORCE_WIDE": "4"},
                                 {"VX_FORCE_WIDE": "3"}, {"VX_FORCE_GSTACK": "1"},
                                 {"VX_FORCE_WIDE": "3", "VX_FORCE_GSTACK": "1"},
                                 {"VX_NO_TMA": "1"}, {"VX_NO_SPARSE": "1"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_wide_and_gstack_variants(env):
    """Every template variant (int64 weights, int64 hull-test products only,
    u64 entries / codes, global stacks) on small grids, in a subprocess so the env knob is seen."""
    r = subprocess.run([sys.executable, "-c", _SUB.format(root=ROOT)], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_sparse_slices():
    """Occupied-slice list path: empty slices at the ends, in the middle, in
    runs, a single occupied slice, all occupied."""
    rng = np.random.default_rng(21)
    for dims in [(96, 64, 64), (200, 40, 36), (33, 128, 32)]:
        for pattern in ("ends", "middle", "runs", "one", "all"):
            occ = (rng.random(dims) < 0.01).astype(np.uint8)
            nx = dims[0]
            if pattern == "ends":
                occ[: nx // 3] = 0
                occ[-nx // 4:] = 0
            elif pattern == "middle":
                occ[nx // 3: 2 * nx // 3] = 0
            elif pattern == "runs":
                for i0 in range(0, nx, 7):
                    occ[i0: i0 + 3] = 0
            elif pattern == "one":
                occ[:] = 0
                occ[nx // 2, 3, 5] = 1
            assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), (dims, pattern)


def test_density_sweep_256():
    for p, seed in [(1e-5, 1), (0.3, 2), (0.9, 3)]:
        occ = synth.bernoulli_occupancy((96, 80, 112), p, seed)
        assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ, 4, 4, 8)), p


# -- reference known-answer tests (pkg/tests/test_edt.py) ------------------------

def test_single_site_analytic_distances():          # test_edt.py:30-36
    occ = np.zeros((5, 5, 5), bool)
    occ[2, 2, 2] = True
    sq = pba_edt(occ).sq_distance_grid()
    assert sq[4, 2, 2] == 4 and sq[4, 4, 4] == 12 and sq[2, 2, 2] == 0


def test_empty_grid_all_no_site():                   # test_edt.py:39-43
    df = pba_edt(np.zeros((8, 8, 8), bool))
    assert (df.site == NO_SITE).all()
    assert df.site_index((3, 3, 3)) is None
    assert query_nearest_site(df, (0, 0, 0)) is None


def test_nonempty_grid_has_no_sentinel():            # test_edt.py:46-51
    rng = np.random.default_rng(2)
    occ = np.zeros((9, 7, 11), bool)
    occ[tuple(rng.integers(0, s) for s in occ.shape)] = True
    assert (pba_edt(occ).site != NO_SITE).all()


def test_band_and_worker_invariance():               # test_edt.py:88-95
    rng = np.random.default_rng(4)
    occ = rng.random((20, 17, 23)) < 0.2
    ref = pba_edt(occ, BandConfig(1, 1, 1), workers=1).site
    for cfg in (BandConfig(2, 4, 2), BandConfig(64, 64, 64), BandConfig(3, 5, 7)):
        for workers in (1, 2, 8):
            assert np.array_equal(pba_edt(occ, cfg, workers=workers).site, ref)


def test_sites_are_occupied_voxels():                # test_edt.py:117-124
    rng = np.random.default_rng(21)
    occ = rng.random((16, 12, 14)) < 0.1
    lin = pba_edt(occ).site.reshape(-1).astype(np.int64)
    ny, nz = occ.shape[1:]
    assert occ[lin // (ny * nz), (lin // nz) % ny, lin % nz].all()


def test_line_nearest_sites_band_invariant():        # test_edt.py:143-148
    rng = np.random.default_rng(32)
    occ = rng.random((8, 8, 29)) < 0.1
    ref = line_nearest_sites(occ, m1=1)
    assert np.array_equal(ref, O.line_nearest_sites(occ))
    for m1 in (2, 3, 4, 8, 29, 64):
        assert np.array_equal(ref, line_nearest_sites(occ, m1=m1))


def test_query_three_four_five():                    # test_edt.py:223-229
    occ = np.zeros((5, 6, 3), bool)
    occ[3, 4, 0] = True
    site, dist = query_nearest_site(pba_edt(occ, voxel_size=0.1), (0, 0, 0))
    assert site == (3, 4, 0) and dist == pytest.approx(0.5)


def test_query_own_site():                           # test_edt.py:232-237
    occ = np.zeros((4, 4, 4), bool)
    occ[1, 2, 3] = True
    site, dist = query_nearest_site(pba_edt(occ, voxel_size=0.25), (1, 2, 3))
    assert site == (1, 2, 3) and dist == 0.0


def test_query_out_of_bounds_raises():               # test_edt.py:240-245
    df = pba_edt(np.ones((3, 3, 3), bool))
    with pytest.raises(IndexError):
        query_nearest_site(df, (3, 0, 0))
    with pytest.raises(IndexError):
        query_nearest_site(df, (0, -1, 0))


def test_dump_squared_golden():                      # test_edt.py:248-253
    occ = np.zeros((3, 2, 1), bool)
    occ[0, 0, 0] = True
    buf = io.StringIO()
    pba_edt(occ).dump_squared(buf)
    assert buf.getvalue() == "slice k=0\n0 1 4\n1 2 5\n"


def test_validation_errors():                        # test_edt.py:256-260, edt.py:457-460
    with pytest.raises(ValueError):
        BandConfig(0, 1, 1)
    with pytest.raises(ValueError):
        pba_edt(np.ones((2, 2, 2), bool), workers=0)
    with pytest.raises(ValueError):
        pba_edt(np.ones((4, 4), bool))
    with pytest.raises(ValueError):
        pba_edt(np.zeros((1, 1, (1 << 20) + 1), bool))


def test_monotonicity_adding_sites():                # test_edt.py:106-114
    rng = np.random.default_rng(12)
    occ = rng.random((12, 12, 12)) < 0.05
    sq = pba_edt(occ).sq_distance_grid()
    free = np.argwhere(~occ)
    occ[tuple(free[rng.integers(0, free.shape[0])])] = True
    assert (pba_edt(occ).sq_distance_grid() <= sq).all()


def _stream_grid(seed, deep):
    """(256, 512, 160): 2560 pass-3 tiles (>= 16 per SM) and m <= L/2 occupied
    slices, so pass 3 takes the one-warp kernel.  deep: every occupied slice
    carries the same sites, so every column's hull keeps all m candidates
    (m > the 63 shared-memory entries: the global spill path)."""
    rng = np.random.default_rng(seed)
    occ = np.zeros((256, 512, 160), np.uint8)
    xs = np.sort(rng.choice(256, 100 if deep else 60, replace=False))
    if deep:
        pts = rng.integers(0, [512, 160], size=(40, 2))
        for x in xs:
            occ[x, pts[:, 0], pts[:, 1]] = 1
    else:
        for x in xs:
            occ[x][rng.random((512, 160)) < 0.002] = 1
    return occ


@pytest.mark.parametrize("deep", [False, True], ids=["shallow", "deep-spill"])
def test_pass3_one_warp_kernel_vs_oracle(deep, monkeypatch):
    """k_pass3_stream (few occupied slices, many tiles), with and without
    stack spills, bit-identical to the oracle and to the banded kernel."""
    occ = _stream_grid(5, deep)
    want = O.pba_edt_site(occ)
    got = pba_edt(occ).site
    assert np.array_equal(got, want)
    monkeypatch.setenv("VX_STREAM_MAX", "-1")   # banded kernel only
    assert np.array_equal(pba_edt(occ).site, want)


@pytest.mark.parametrize("deep", [False, True], ids=["shallow", "deep-spill"])
def test_pass3_one_warp_kernel_multi_tile(deep, monkeypatch):
    """k_pass3_stream with more tiles than warps (6400 tiles > 148 x 32): warps
    walk a second tile after their first, re-using their stacks (deep: the
    global spill slab too); equal to the oracle and to the banded kernel."""
    rng = np.random.default_rng(11)
    occ = np.zeros((160, 1536, 128), np.uint8)
    xs = np.sort(rng.choice(160, 80 if deep else 50, replace=False))
    pts = rng.integers(0, [1536, 128], size=(50, 2))
    for x in xs:
        occ[x][rng.random((1536, 128)) < 0.001] = 1
        if deep:
            occ[x, pts[:, 0], pts[:, 1]] = 1
    want = O.pba_edt_site(occ)
    assert np.array_equal(pba_edt(occ).site, want)
    monkeypatch.setenv("VX_STREAM_MAX", "-1")   # banded kernel only
    assert np.array_equal(pba_edt(occ).site, want)


@pytest.mark.parametrize("m", [1, 15, 16, 17, 33, 100])
def test_pass3_one_warp_kernel_batches_and_ragged_tiles(m, monkeypatch):
    """k_pass3_stream's batch edges and partial warps: occupied-slice counts
    around the 16-row candidate batches (the padded list's predicated tail,
    the once-per-batch spill vote) and nz = 150, whose last k-tile leaves 10
    lanes idle (the warp votes and the first-switch minimum then run on a
    partial mask); half the slices carry shared sites, so some columns have
    late first switches and long hulls.  Equal to the oracle and to the
    banded kernel."""
    rng = np.random.default_rng(100 + m)
    occ = np.zeros((200, 512, 150), np.uint8)
    xs = np.sort(rng.choice(200, m, replace=False))
    pts = rng.integers(0, [512, 150], size=(30, 2))
    for n, x in enumerate(xs):
        occ[x][rng.random((512, 150)) < 0.001] = 1
        if n % 2 == 0:
            occ[x, pts[:, 0], pts[:, 1]] = 1
    want = O.pba_edt_site(occ)
    assert np.array_equal(pba_edt(occ).site, want)
    monkeypatch.setenv("VX_STREAM_MAX", "-1")   # banded kernel only
    assert np.array_equal(pba_edt(occ).site, want)


def test_cycle_pass3_kernel_choice(monkeypatch):
    """The camera tick picks its pass-3 kernel from the previous tick's
    occupied-slice count (host-mapped hint); every choice, and every switch
    between them (graph re-capture), gives the field of a plain EDT."""
    from paper_2407_02363_b200.engine import MapCycle
    dims, vs, origin = (256, 512, 160), 0.02, (-2.56, -5.12, -0.2)
    rng = np.random.default_rng(7)
    cyc = MapCycle(dims, vs, origin, [], vs, [], max_points=40000, max_spheres=4)
    centers = np.zeros((4, 3))
    for t, smax in enumerate([None, None, None, "10", "10", None]):
        if smax is None:
            monkeypatch.delenv("VX_STREAM_MAX", raising=False)
        else:
            monkeypatch.setenv("VX_STREAM_MAX", smax)   # forces the banded choice
        # points in ~40 i-slices
        xs = rng.choice(256, 40, replace=False)
        i = rng.choice(xs, 40000)
        pts = np.stack([origin[0] + (i + rng.random(40000)) * vs,
                        origin[1] + rng.random(40000) * 512 * vs,
                        origin[2] + rng.random(40000) * 160 * vs], axis=1)
        cyc.step(pts, np.zeros((0, 16)), centers)
        cyc.wait()
        env, _, _ = cyc.grids()
        fe, _ = cyc.fields()
        occ = env.occupancy_mask()
        monkeypatch.setenv("VX_STREAM_MAX", "-1")
        assert np.array_equal(fe.site, pba_edt(occ).site), t


def test_pass3_one_warp_kernel_512_specialisation(monkeypatch):
    """The 512^3 specialisation of the one-warp pass 3 (constant strides) on a
    scene-like grid (90 occupied slices, clustered sites, some deep hulls)
    equals the banded kernel, which the 512^3 reference digests pin."""
    rng = np.random.default_rng(512)
    occ = np.zeros((512, 512, 512), np.uint8)
    xs = np.sort(rng.choice(512, 90, replace=False))
    pts = rng.integers(0, 512, size=(60, 2))
    for n, x in enumerate(xs):
        sl = occ[x]
        sl[rng.random((512, 512)) < 2e-4] = 1
        if n % 3 == 0:   # shared sites across slices: hulls keep every candidate
            sl[pts[:, 0], pts[:, 1]] = 1
    got = pba_edt(occ).site
    monkeypatch.setenv("VX_STREAM_MAX", "-1")
    assert np.array_equal(got, pba_edt(occ).site)


@pytest.mark.parametrize("narrow", ["1", "0"], ids=["16col-tiles", "32col-tiles"])
def test_long_columns_vs_oracle(narrow, monkeypatch):
    """Columns longer than 512 rows (32 bands): 16-column tiles at three CTAs
    per SM, or 32-column tiles of 1024 threads (VX_NARROW_TILES=0); dense,
    ragged nz, and few occupied i-slices (the compact pass-3 row staging)."""
    monkeypatch.setenv("VX_NARROW_TILES", narrow)
    rng = np.random.default_rng(31)
    cases = [((700, 48, 64), 0.02), ((40, 1024, 36), 0.01), ((1024, 24, 20), 0.003)]
    for dims, p in cases:
        occ = (rng.random(dims) < p).astype(np.uint8)
        assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), dims
    occ = np.zeros((900, 40, 48), np.uint8)
    for x in rng.choice(900, 25, replace=False):
        occ[x][rng.random((40, 48)) < 0.01] = 1
    assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ))
