"""int16 line sites (EdtPlan::s1_16): pass 1 writes 2-byte sites and pass 2
widens its 16-bit TMA tiles in shared memory (vx_edt.cu widen16).  The plan
turns it on for pass-2 columns of 64..1024 rows (a power of two) and
nz % 8 == 0; every pass-1 kernel variant (16 voxels per lane, 4 per lane,
generic) then writes int16.  Each case runs with it forced off (VX_S1_16=0)
and on, against the oracle (edt.py:188-420 via oracle/), on the windowed,
banded and one-warp paths."""
import ctypes

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2407_02363_b200 import _lib, pba_edt, synth

pytestmark = pytest.mark.gpu


def _scene_slices(dims, nocc, p, seed):
    """Few occupied x slices (the camera tick's shape): one-warp pass 3."""
    rng = np.random.default_rng(seed)
    occ = np.zeros(dims, np.uint8)
    xs = rng.choice(dims[0], nocc, replace=False)
    occ[xs] = (rng.random((nocc,) + tuple(dims[1:])) < p).astype(np.uint8)
    return occ


CASES = [
    ("64^3", lambda: synth.bernoulli_occupancy((64, 64, 64), 0.02, 3)),
    ("v4 nz=200", lambda: synth.bernoulli_occupancy((40, 128, 200), 0.05, 4)),
    ("v4 nz=1000", lambda: synth.bernoulli_occupancy((33, 256, 1000), 0.01, 5)),
    ("generic nz=2056", lambda: synth.bernoulli_occupancy((6, 64, 2056), 0.01, 6)),
    ("L=1024 pass 2", lambda: synth.bernoulli_occupancy((16, 1024, 16), 0.05, 7)),
    ("sparse", lambda: synth.bernoulli_occupancy((64, 512, 128), 0.0005, 8)),
    ("dense 0.4", lambda: synth.bernoulli_occupancy((48, 256, 64), 0.4, 9)),
    ("few slices", lambda: _scene_slices((256, 128, 64), 20, 0.05, 10)),
    ("empty", lambda: np.zeros((32, 64, 64), np.uint8)),
    ("one voxel", lambda: np.pad(np.ones((1, 1, 1), np.uint8), ((5, 26), (40, 23), (7, 56)))),
]


@pytest.mark.parametrize("s16", ["0", "1"])
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_s1_16_vs_oracle(name, make, s16, monkeypatch):
    monkeypatch.setenv("VX_S1_16", s16)
    occ = make()
    assert np.array_equal(pba_edt(occ).site, O.pba_edt_site(occ)), name


@pytest.mark.parametrize("s16", ["0", "1"])
def test_s1_16_batched(s16, monkeypatch):
    """A batch of scenes (the C4 path) through vx_edt_device."""
    monkeypatch.setenv("VX_S1_16", s16)
    dims = (32, 128, 64)
    ps = [0.02, 0.3, 0.0005, 0.0]
    occ = np.stack([synth.bernoulli_occupancy(dims, p, 20 + s) for s, p in enumerate(ps)])
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
