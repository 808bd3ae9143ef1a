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
            slab_edt = SlabEDT(dims, exchange="nccl", backend=OracleBackend(), device=torch.device("cpu"))
            i0, i1 = slab_edt.i_starts[rank], slab_edt.i_starts[rank + 1]
            site = slab_edt(torch.from_numpy(occ[i0:i1].copy())).clone()
            parts = [None] * world
            dist.all_gather_object(parts, site.numpy())
            if rank == 0:
                full = np.concatenate(parts, axis=1)
                q.put((dims, bool(np.array_equal(full, O.pba_edt_site(occ)))))
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
