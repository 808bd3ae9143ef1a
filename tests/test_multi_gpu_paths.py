"""GPU tests of the two multi-GPU decompositions on one device:
  * data-parallel scene batches (config C4): one batched launch over S scenes
    == S single EDTs == the oracle;
  * slab mode (config C5): the fused pass-2 exchange epilogue, emulated for G
    virtual ranks in one process (sequential, no inter-rank waiting), for
    both transports' addressing; assembled j-slabs == the single-grid EDT.
Bit-exact integer comparisons."""
import ctypes

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2407_02363_b200 import _lib, pba_edt, synth
from paper_2407_02363_b200.slab import SlabEDT, emulate_ranks

pytestmark = pytest.mark.gpu


def _edt_batched(occ_batch: torch.Tensor) -> torch.Tensor:
    S, nx, ny, nz = occ_batch.shape
    ctx = _lib.default_context()
    L = _lib.load()
    site = torch.empty((S, nx, ny, nz), dtype=torch.int32, device=occ_batch.device)
    _lib.check(L.vx_edt_device(ctx.handle, ctypes.c_void_p(occ_batch.data_ptr()), nx, ny, nz, S,
                               ctypes.c_void_p(site.data_ptr()), None, 0))
    ctx.synchronize()
    return site


@pytest.mark.parametrize("dims", [(64, 64, 64), (33, 47, 20), (16, 128, 36)])
def test_batched_scenes_match_single(dims):
    S = 6
    occ = np.stack([synth.bernoulli_occupancy(dims, [0.02, 0.3, 1e-3, 0.0, 0.6, 0.05][s], s)
                    for s in range(S)])
    site = _edt_batched(torch.from_numpy(occ).cuda()).cpu().numpy()
    for s in range(S):
        assert np.array_equal(site[s], O.pba_edt_site(occ[s])), s


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_slab_emulated_ranks(world, exchange):
    for dims, p, seed in [((64, 64, 64), 0.02, 0), ((40, 50, 36), 0.2, 1), ((24, 17, 12), 0.001, 2)]:
        occ = synth.bernoulli_occupancy(dims, p, seed)
        got = emulate_ranks(torch.from_numpy(occ).cuda(), world, exchange).cpu().numpy()
        assert np.array_equal(got, O.pba_edt_site(occ)), (dims, world, exchange)


def test_slab_emulated_256_vs_single_gpu():
    occ = synth.bernoulli_occupancy((256, 256, 256), 0.02, 5)
    ref = pba_edt(occ).site
    for world in (2, 8):
        got = emulate_ranks(torch.from_numpy(occ).cuda(), world, "p2p").cpu().numpy()
        assert np.array_equal(got, ref), world


def test_slab_single_rank_api():
    occ = synth.bernoulli_occupancy((48, 40, 32), 0.05, 3)
    slab = SlabEDT(occ.shape, exchange="nccl")
    site = slab(torch.from_numpy(occ).cuda()).cpu().numpy()
    assert np.array_equal(site, O.pba_edt_site(occ))


@pytest.mark.parametrize("rec", __import__("tests.golden_util", fromlist=["golden"]).golden()
                         .get("edt_digests_1024", []), ids=lambda r: f"1024-{r['p']}")
def test_c5_1024_single_gpu_and_slab_vs_reference(rec):
    """Config C5 (1024^3): the single-GPU EDT and the 8-rank slab pipeline
    (emulated, both transports' addressing) against the reference digest."""
    from tests.golden_util import digest
    occ = synth.bernoulli_occupancy(rec["dims"], rec["p"], rec["seed"])
    d_occ = torch.from_numpy(occ).cuda()
    del occ
    site = _edt_batched(d_occ.unsqueeze(0))[0]
    assert digest(site.cpu().numpy()) == rec["site"]
    del site
    torch.cuda.empty_cache()
    got = emulate_ranks(d_occ, 8, "p2p").cpu().numpy()
    assert digest(got) == rec["site"]


_P2P_SCRIPT = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["VX_ROOT"])
from oracle import oracle as O
from paper_2407_02363_b200 import synth
from paper_2407_02363_b200.slab import SlabEDT
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
for exchange, chunks in (("p2p", None), ("nccl", 1), ("nccl", 3)):
    for dims, p, seed in [((64, 48, 40), 0.03, 4), ((33, 20, 16), 0.2, 5)]:
        slab = SlabEDT(dims, exchange=exchange, chunks=chunks)
        for rep in range(3):   # repeated calls reuse the receive buffer
            occ = synth.bernoulli_occupancy(dims, p, seed + rep)
            site = slab(torch.from_numpy(occ).cuda()).cpu().numpy()
            assert np.array_equal(site, O.pba_edt_site(occ)), (exchange, dims, rep)
dist.destroy_process_group()
print("P2P-WORLD1-OK")
"""


def test_slab_p2p_symmetric_memory_world1():
    """SlabEDT(exchange="p2p") for real: a one-rank NCCL group sets up the
    torch symmetric-memory receive buffer (rendezvous, peer pointer table),
    and the pass-2 epilogue stores through the mapped peer pointer; the
    barriers run on the library stream.  Repeated calls, vs the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VX_ROOT=root, MASTER_ADDR="127.0.0.1", MASTER_PORT="29517")
    r = subprocess.run([sys.executable, "-c", _P2P_SCRIPT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "P2P-WORLD1-OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_slab_site_world_on_j_slabs_vs_whole_field():
    """vx_site_world_slab: split a whole field into j-slabs (2/3/5 ranks'
    worth); every centre is answered by exactly the slab that holds its
    clipped row, and the combined answers equal K6 on the whole field
    (engine.py:212-221; world point bit-exact, distance rtol 1e-6)."""
    from paper_2407_02363_b200.engine import site_world
    from paper_2407_02363_b200.slab import CudaBackend, even_split
    dims, vs, origin = (40, 50, 36), 0.05, np.array([-1.0, -1.2, -0.3])
    occ = synth.bernoulli_occupancy(dims, 0.01, 8)
    fld = pba_edt(occ, voxel_size=vs)
    full = torch.from_numpy(fld.site).cuda()
    rng = np.random.default_rng(3)
    centers = rng.uniform(origin - 0.3, origin + np.array(dims) * vs + 0.3, size=(64, 3))
    want = site_world(fld, origin, vs, centers)
    be = CudaBackend()
    for world in (2, 3, 5):
        js = even_split(dims[1], world)
        lin = np.full(64, -2, np.int32)
        wpt = np.full((64, 3), np.nan)
        dd = np.full(64, np.nan)
        for q in range(world):
            part = full[:, js[q]:js[q + 1]].contiguous()
            l_, w_, d_ = be.site_world_slab(part, dims, js[q], centers, origin, vs)
            own = l_ != -2
            assert not (own & (lin != -2)).any()   # one owner per centre
            lin[own], wpt[own], dd[own] = l_[own], w_[own], d_[own]
        assert np.array_equal(lin, want[0])
        ok = want[0] >= 0
        assert np.array_equal(wpt[ok], want[1][ok])
        np.testing.assert_allclose(dd[ok], want[2][ok], rtol=1e-6)


def test_slab_single_rank_site_world():
    from paper_2407_02363_b200.engine import site_world
    dims, vs, origin = (48, 40, 32), 0.04, np.zeros(3)
    occ = synth.bernoulli_occupancy(dims, 0.05, 3)
    slab = SlabEDT(dims, exchange="nccl", chunks=3)
    slab(torch.from_numpy(occ).cuda())
    centers = np.random.default_rng(1).uniform(-0.2, 2.0, size=(30, 3))
    got = slab.site_world(centers, origin, vs)
    want = site_world(pba_edt(occ, voxel_size=vs), origin, vs, centers)
    assert np.array_equal(got[0], want[0])
    ok = want[0] >= 0
    assert np.array_equal(got[1][ok], want[1][ok])
