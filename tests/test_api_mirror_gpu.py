"""The shim's full voxarm/__init__.py:16-37 surface for the distance path:
brute_force_edt on the GPU against the reference's own site arrays, and
voxarm's own self-checks (cli.py:100-118, `voxarm verify`) run against the
shim's pba_edt / brute_force_edt in place of voxarm's."""
import os
import sys

import numpy as np
import pytest

from paper_2407_02363_b200 import brute_force_edt, pba_edt
from tests.golden_util import edt_cases

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def test_brute_force_edt_vs_reference_sites():
    """edt.py:487-508 (lexicographic ties) == the reference's pba_edt sites
     on the reference-generated cases up to ~32^3."""
    for occ, site, _, _ in edt_cases():
        if occ.size > 40000:
            continue
        assert np.array_equal(brute_force_edt(occ).site, site), occ.shape


def test_brute_force_edt_empty_and_full():
    assert (brute_force_edt(np.zeros((5, 6, 7), bool)).site == -1).all()
    full = np.ones((4, 3, 5), bool)
    assert np.array_equal(brute_force_edt(full).site, np.arange(60, dtype=np.int32).reshape(4, 3, 5))


@pytest.fixture
def voxarm_cli():
    if os.path.isdir(REF) and REF not in sys.path:
        sys.path.append(REF)
    return pytest.importorskip("voxarm.cli")


def test_voxarm_verify_edt_checks_on_the_shim(voxarm_cli, monkeypatch):
    """voxarm's `_check_edt_exact` (12 random grids, pba_edt vs brute_force_edt
    squared distances) and `_check_edt_workers` (site bit-identity across
    worker counts), with both names bound to the shim."""
    monkeypatch.setattr(voxarm_cli, "pba_edt", pba_edt)
    monkeypatch.setattr(voxarm_cli, "brute_force_edt", brute_force_edt)
    for seed in (0, 1, 2):
        rng = np.random.default_rng(seed)
        assert voxarm_cli._check_edt_exact(rng) is None
        assert voxarm_cli._check_edt_workers(rng) is None
