"""Multi-rank slab EDT host logic under gloo, world sizes 2 and 3,
on CPU: the slab partition, the fused pass-2 exchange addressing and the
all-to-all splits, with the oracle standing in for the kernels.  The assembled
j-slabs must equal the single-grid EDT bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2407_02363_b200.slab import SlabEDT, even_split
from tests.slab_oracle_backend import OracleBackend

CASES = [((13, 11, 9), 0.08, 1), ((16, 16, 16), 0.02, 2), ((7, 20, 5), 0.3, 3), ((9, 9, 33), 0.0, 4)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for dims, p, seed in CASES:
            occ = (np.random.default_rng(seed).random(dims) < p).astype(np.uint8)
            ok = True
            for chunks in (1, 3, 16):   # pipelined exchange: slice groups (more groups than slices too)
                slab_edt = SlabEDT(dims, exchange="nccl", backend=OracleBackend(), device=torch.device("cpu"),
                                   chunks=chunks)
                i0, i1 = slab_edt.i_starts[rank], slab_edt.i_starts[rank + 1]
                for rep in range(2):   # buffers reused across calls
                    site = slab_edt(torch.from_numpy(occ[i0:i1].copy())).clone()
                    parts = [None] * world
                    dist.all_gather_object(parts, site.numpy())
                    full = np.concatenate(parts, axis=1)
                    ok = ok and bool(np.array_equal(full, O.pba_edt_site(occ)))
                # sphere queries routed to the row owner (engine.py:212-221)
                vs, origin = 0.05, np.array([-0.3, 0.2, -0.1])
                rng = np.random.default_rng(seed + 100)
                lo, hi = origin - 0.2, origin + np.array(dims) * vs + 0.2   # some centres outside
                centers = rng.uniform(lo, hi, size=(25, 3))
                lin, world_pt, dd = slab_edt.site_world(centers, origin, vs)
                rl, rw, rd = O.site_world(O.pba_edt_site(occ), vs, origin, centers)
                okq = np.array_equal(lin, rl) and np.array_equal(world_pt[rl >= 0], rw[rl >= 0]) and \
                    np.allclose(dd[rl >= 0], rd[rl >= 0], rtol=1e-6) and bool(np.all(np.isinf(dd[rl < 0])))
                ok = ok and okq
            if rank == 0:
                q.put((dims, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_gloo_matches_single_grid(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, q), nprocs=world, join=True)
    results = [q.get(timeout=60) for _ in CASES]
    for dims, ok in results:
        assert ok, dims


def test_even_split():
    assert even_split(10, 3) == [0, 4, 7, 10]
    assert even_split(1024, 8)[-1] == 1024
    assert even_split(5, 5) == [0, 1, 2, 3, 4, 5]
