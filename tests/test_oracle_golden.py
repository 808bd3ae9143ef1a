"""Pin the CPU oracle (oracle/) against the reference's own outputs.

Golden fixtures were produced by importing the reference (voxarm) in the
build container (tests/golden/make_golden.py); known-answer tests are the
reference's own (pkg/tests/test_edt.py, test_grids.py).  CPU only.
"""

import io

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_02363_b200 import synth
from tests.golden_util import desk7, digest, edt_cases, golden, world_points


def test_edt_cases_bit_exact_vs_reference():
    for occ, site, s1, bands in edt_cases():
        got = O.pba_edt_site(occ, *bands)
        assert np.array_equal(got, site), occ.shape
        assert np.array_equal(O.line_nearest_sites(occ, bands[0]), s1)


def test_edt_cases_match_brute_force_lexmin():
    # pba site == brute-force lexicographic-min site, bit for bit
    for occ, site, _, _ in edt_cases()[:30]:
        assert np.array_equal(O.brute_force_site(occ), site)


@pytest.mark.parametrize("rec", [r for r in golden()["edt_digests"]
                                 if np.prod(r["dims"]) <= 192 * 192 * 128],
                         ids=lambda r: f"{r['gen']}-{'x'.join(map(str, r['dims']))}")
def test_edt_digests(rec):
    if rec["gen"] == "bernoulli":
        occ = synth.bernoulli_occupancy(rec["dims"], rec["p"], rec["seed"])
    else:
        occ = synth.structured_occupancy(rec["gen"], rec["dims"])
    site = O.pba_edt_site(occ, 2, 2, 4)
    assert digest(site) == rec["site"]
    if "s1" in rec:
        assert digest(O.line_nearest_sites(occ)) == rec["s1"]
        assert digest(O.sq_distance_grid(site)) == rec["sq"]


# -- reference known-answer tests (pkg/tests/test_edt.py) -------------------

def test_single_site_analytic():               # test_edt.py:30-36
    occ = np.zeros((5, 5, 5), bool)
    occ[2, 2, 2] = True
    sq = O.sq_distance_grid(O.pba_edt_site(occ))
    assert sq[4, 2, 2] == 4 and sq[4, 4, 4] == 12 and sq[2, 2, 2] == 0


def test_empty_all_no_site():                  # test_edt.py:39-43
    assert (O.pba_edt_site(np.zeros((8, 8, 8), bool)) == O.NO_SITE).all()


def test_two_sites_1d_split():                 # test_edt.py:60-66
    occ = np.zeros((8, 1, 1), bool)
    occ[0] = occ[7] = True
    site = O.pba_edt_site(occ)
    assert site.reshape(-1).tolist() == [0, 0, 0, 0, 7, 7, 7, 7]


def test_dump_golden():                        # test_edt.py:248-253
    occ = np.zeros((3, 2, 1), bool)
    occ[0, 0, 0] = True
    sq = O.sq_distance_grid(O.pba_edt_site(occ))
    buf = io.StringIO()
    for k in range(1):
        buf.write(f"slice k={k}\n")
        for j in range(2):
            buf.write(" ".join(str(int(v)) for v in sq[:, j, k]) + "\n")
    assert buf.getvalue() == "slice k=0\n0 1 4\n1 2 5\n"


def test_proximate_stack_cases():              # test_edt.py:175-194
    assert O.proximate_sites_1d([(0, (3, 0)), (10, (3, 10))], 0) == [(3, 0), (3, 10)]
    assert O.proximate_sites_1d([(0, (0, 0)), (5, (10, 5)), (10, (0, 10))], 0) == \
        [(0, 0), (0, 10)]
    with pytest.raises(ValueError):
        O.proximate_sites_1d([(5, (0, 5)), (5, (1, 5))], 0)


# -- map side -----------------------------------------------------------------

def _oracle_insert_case(c):
    case = synth.insert_case(c)
    cells = np.zeros(case["dims"], np.float32)
    mask = None
    if case["mask_ijk"] is not None:
        mask = np.zeros(case["dims"], np.float32)
        O.stamp_voxels(mask, case["voxel_size"], case["origin"], case["mask_ijk"],
                       case["origin"], case["voxel_size"])
    stats = []
    for pts in case["clouds"]:
        st = O.insert_points(cells, case["voxel_size"], case["origin"],
                             world_points(pts, case["pose"]), mask, case["thr"], case["hit"])
        stats.append(list(st))
    return case, cells, stats


def test_insert_cases_vs_reference():
    for rec in golden()["insert"]:
        case, cells, stats = _oracle_insert_case(rec["case"])
        assert stats == rec["stats"], rec["case"]
        assert digest(cells) == rec["cells"], rec["case"]
        thr = np.float32(O.logit(case["thr"]))
        assert digest(cells > thr) == rec["occ"]


def test_stamp_cases_vs_reference():
    for rec in golden()["stamp"]:
        case = synth.stamp_case(rec["case"])
        cells = np.zeros(case["dims"], np.float32)
        oob = O.stamp_voxels(cells, case["voxel_size"], case["origin"], case["ijk"],
                             case["set_origin"], case["set_voxel_size"], case["T"])
        assert oob == rec["oob"]
        assert digest(cells) == rec["cells"], rec["case"]


def test_site_world_cases_vs_reference():
    for rec in golden()["site_world"]:
        case = synth.site_world_case(rec["case"])
        site = O.pba_edt_site(case["occ"])
        lin, world, dist = O.site_world(site, case["voxel_size"], case["origin"],
                                        case["centers"])
        for q, (w, d) in enumerate(zip(rec["world"], rec["dist"])):
            if w is None:
                assert lin[q] == -1 and np.isinf(dist[q])
            else:
                assert world[q].tolist() == w
                assert dist[q] == pytest.approx(d, rel=1e-12)


def test_c1_cycle_vs_reference():
    """One full C1 camera tick through the oracle == the reference engine."""
    g = golden()["c1"]
    d = desk7()
    spec = synth.C1
    dims, vs, origin = spec["dims"], spec["voxel_size"], spec["origin"]
    frames = d["frames"][0]                       # q = GUARD_Q
    selfc = np.zeros(dims, np.float32)
    maskc = np.zeros(dims, np.float32)
    for li in d["o_links"]:
        ijk, org = d["links"][li]
        O.stamp_voxels(selfc, vs, origin, ijk, org, vs, frames[li])
    for li, (ijk, org) in enumerate(d["links"]):
        O.stamp_voxels(maskc, vs, origin, ijk, org, vs, frames[li])
    assert digest(selfc) == g["self_cells"]
    assert digest(maskc) == g["mask_cells"]
    centers = np.vstack([synth.sphere_centers(frames, d["sphere_link"], d["sphere_center"]),
                         synth.extra_query_points(dims, vs, origin)])
    assert digest(centers) == g["centers"]
    for f in ("0", "5"):
        pts = synth.c1_cloud(int(f) / 30.0)
        assert digest(pts) == g[f]["cloud"]
        env = np.zeros(dims, np.float32)
        st = O.insert_points(env, vs, origin, pts, maskc)
        assert list(st) == g[f]["stats"]
        assert digest(env) == g[f]["env_cells"]
        site = O.pba_edt_site(env > 0, 4, 4, 8)
        assert digest(site) == g[f]["env_site"]
        lin, world, dist = O.site_world(site, vs, origin, centers)
        for q, w in enumerate(g[f]["env_world"]):
            assert (lin[q] == -1) if w is None else (world[q].tolist() == w)
    site = O.pba_edt_site(selfc > 0)
    assert digest(site) == g["self_site"]


def test_bench512_tick0_vs_reference():
    """The headline workload (bench.py tick 0 at 512^3) through the oracle
    equals voxarm's own grids + pba_edt + _site_world on it."""
    import bench
    g = golden()["bench512_tick0"]
    d = desk7()
    pts, frames, centers = bench.scene_inputs(0, 0, d)
    assert digest(pts) == g["cloud"]
    mask = np.zeros(bench.DIMS, np.float32)
    for li, (ijk, org) in enumerate(d["links"]):
        O.stamp_voxels(mask, bench.VS, bench.ORIGIN, ijk, org, bench.VS, frames[li])
    env = np.zeros(bench.DIMS, np.float32)
    st = O.insert_points(env, bench.VS, bench.ORIGIN, pts, mask)
    assert list(st) == g["stats"]
    occ = env > 0
    assert digest(occ) == g["occ"]
    site = O.pba_edt_site(occ)
    assert digest(site) == g["site"]
    lin, world, _ = O.site_world(site, bench.VS, bench.ORIGIN, centers)
    for q, w in enumerate(g["env_world"]):
        assert (lin[q] == -1) if w is None else (world[q].tolist() == w)


def test_shim_proximate_stack_matches_oracle_and_reference_cases():
    """The shim's host API mirror of edt.py:55-100 (ProximateStack,
    proximate_sites_1d) against the oracle restatement (itself pinned on the
    reference's cases, test_proximate_stack_cases) and its ValueError."""
    from paper_2407_02363_b200 import ProximateStack, proximate_sites_1d
    rng = np.random.default_rng(9)
    for _ in range(300):
        n = int(rng.integers(0, 12))
        coords = np.sort(rng.choice(40, size=n, replace=False))
        sites = [(int(c), (int(rng.integers(-20, 20)), int(c))) for c in coords]
        col = int(rng.integers(-10, 10))
        got = proximate_sites_1d(sites, col)
        assert isinstance(got, ProximateStack)
        assert got.sites() == O.proximate_sites_1d(sites, col)
        assert [c for c, _ in got.entries] == [c for c, s in sites if s in got.sites()]
    with pytest.raises(ValueError):
        proximate_sites_1d([(3, (0, 0)), (3, (1, 0))], 0)


def test_shim_load_point_cloud(tmp_path):
    """grids.py:243-256: comments and blank lines skipped, short lines rejected."""
    from paper_2407_02363_b200 import load_point_cloud
    f = tmp_path / "c.txt"
    f.write_text("# cloud\n0.5 1 2\n\n -1e-3 4 5.25 extra\n")
    pc = load_point_cloud(f)
    assert pc.points.tolist() == [[0.5, 1.0, 2.0], [-1e-3, 4.0, 5.25]]
    f.write_text("1 2\n")
    with pytest.raises(ValueError):
        load_point_cloud(f)
