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
