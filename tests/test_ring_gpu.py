"""The windowed exact search for dense scenes (k_column_ring, passes 2 and 3)
and its hand-back of tiles to the banded kernel.

The search returns, per query row, the first row minimising (q - y)^2 + w_y
-- the answer of edt.py:300-317's strict-< walk over the lower envelope
(edt.py:253-276) -- so `site` must stay bit-identical to the reference.
Every case runs under knob settings that force each route: default
(dense scenes searched, sparse ones banded), VX_RING=0 (banded only),
VX_RING_CAP=1/2 (nearly every tile handed back mid-search), VX_RING_MIN=0
(the search attempted on every scene, sparse ones included), a tiny
radius budget (tiles handed back for cost), and no limits at all (the
search alone, windows as wide as the column).
"""
import ctypes

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_02363_b200 import _lib, pba_edt, synth
from tests.golden_util import edt_cases

pytestmark = pytest.mark.gpu

KNOBS = [{}, {"VX_RING": "0"}, {"VX_RING_CAP": "1"}, {"VX_RING_CAP": "2"}, {"VX_RING_MIN": "0"},
         {"VX_RING_MIN": "0", "VX_RING_CAP": "3"}, {"VX_RING_BUDGET2": "1", "VX_RING_BUDGET3": "2"},
         {"VX_RING_MIN": "0", "VX_RING_BUDGET2": "1000", "VX_RING_BUDGET3": "1000", "VX_RING_CAP": "1000"}]
KID = lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default"  # noqa: E731


def _set(monkeypatch, env):
    for k in ("VX_RING", "VX_RING_CAP", "VX_RING_MIN", "VX_RING_BUDGET2", "VX_RING_BUDGET3"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)


@pytest.mark.parametrize("env", KNOBS, ids=KID)
def test_reference_golden_cases(env, monkeypatch):
    """The 58 reference-generated grids (voxarm's own pba_edt site arrays)."""
    _set(monkeypatch, env)
    for occ, site, _, _ in edt_cases():
        assert np.array_equal(pba_edt(occ).site, site), occ.shape


@pytest.mark.parametrize("env", KNOBS, ids=KID)
@pytest.mark.parametrize("dims,p", [((96, 96, 96), 0.02), ((64, 70, 36), 0.3), ((80, 64, 100), 0.05),
                                    ((128, 96, 64), 0.005), ((40, 600, 32), 0.02), ((600, 40, 32), 0.02),
                                    ((70, 50, 200), 0.6), ((50, 64, 64), 0.0005), ((1100, 40, 32), 0.02),
                                    ((40, 1100, 32), 0.02)],
                         ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple) else str(v))
def test_dense_grids_vs_oracle(dims, p, env, monkeypatch):
    """Densities from 0.05 % to 60 %, ragged k tiles (nz % 32 != 0), columns
    longer than 512 in pass 2 (ny = 600) and pass 3 (nx = 600: 16-column
    tiles), against the oracle."""
    _set(monkeypatch, env)
    occ = synth.bernoulli_occupancy(dims, p, 11)
    assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ))


def test_structured_dense_cases(monkeypatch):
    """Ties everywhere (a lattice of sites), a full grid, a grid with one
    empty slice in the middle (dense scene, one slice without codes), and
    a grid with empty k-lines."""
    _set(monkeypatch, {})
    dims = (64, 64, 64)
    lattice = np.zeros(dims, np.uint8)
    lattice[::4, ::4, ::4] = 1
    full = np.ones(dims, np.uint8)
    hole = synth.bernoulli_occupancy(dims, 0.05, 3)
    hole[30] = 0
    lines = synth.bernoulli_occupancy(dims, 0.05, 4)
    lines[:, ::3, :] = 0
    for occ in (lattice, full, hole, lines):
        assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ))


@pytest.mark.parametrize("env", [{}, {"VX_RING_CAP": "2"}], ids=KID)
def test_batched_dense_and_sparse_scenes(env, monkeypatch):
    """One batched launch mixing dense scenes (searched) and sparse ones
    (banded), with hand-backs under a tiny cap."""
    import torch
    _set(monkeypatch, env)
    dims = (64, 48, 64)
    ps = [0.02, 1e-3, 0.2, 0.0, 0.05, 2e-4]
    occ = np.stack([synth.bernoulli_occupancy(dims, p, 30 + s) for s, p in enumerate(ps)])
    ctx = _lib.default_context()
    L = _lib.load()
    d_occ = torch.from_numpy(occ).cuda()
    site = torch.empty((len(ps),) + dims, dtype=torch.int32, device="cuda")
    _lib.check(L.vx_edt_device(ctx.handle, ctypes.c_void_p(d_occ.data_ptr()), *dims, len(ps),
                               ctypes.c_void_p(site.data_ptr()), None, 0))
    ctx.synchronize()
    got = site.cpu().numpy()
    for s in range(len(ps)):
        assert np.array_equal(got[s], O.pba_edt_site(occ[s])), s


def test_dense_512_reference_digest_all_routes(monkeypatch):
    """512^3 Bernoulli(0.02) -- the C3 bench grid -- against voxarm's digest
    through the search, the banded kernel, and a cap that hands tiles back."""
    from tests.golden_util import digest, golden
    rec = next(r for r in golden()["edt_digests"]
               if r.get("gen") == "bernoulli" and r["dims"] == [512, 512, 512] and r["p"] == 0.02)
    occ = synth.bernoulli_occupancy(rec["dims"], rec["p"], rec["seed"])
    for env in ({}, {"VX_RING": "0"}, {"VX_RING_CAP": "6"}):
        _set(monkeypatch, env)
        assert digest(pba_edt(occ).site) == rec["site"], env
