"""One large grid across G GPUs: slab decomposition along the slow axis i
(1024^3 on 2/4/8 B200).

Rank r owns the i-slab [i0_r, i1_r) of the occupancy.  Passes 1 (along k)
and 2 (along j) are local to a slab (edt.py:168-317 never mix slices).  Pass 3
(along i, edt.py:320-420) needs every slice of a column, so the pass-2 codes
are transposed from i-slabs to j-slabs: rank q receives rows j in
[j0_q, j1_q) of every slice, i.e. a (nx, nyl_q, nz) array, and runs pass 3
on it with global coordinates.  The result stays j-sliced (no transpose
back): rank q holds site[:, j0_q:j1_q, :] with global flat indices.

The exchange is fused into pass 2's epilogue (vx_edt_pass12_scatter): each
code row is stored straight to its destination, so there is no separate pack
pass.  Two transports:
  * "nccl": the destination is this rank's all-to-all send block for q, and one
    NCCL all_to_all_single over NVLink moves the blocks (the baseline);
  * "p2p":  the destination is rank q's receive buffer itself, mapped into this
    process over NVLink (torch symmetric memory); a barrier replaces the
    collective, and the transfer overlaps pass-2 compute tile by tile.
Bytes crossing NVLink per rank: 4 B x nxl x (ny - nyl) x nz each way.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def even_split(n: int, parts: int) -> list[int]:
    """Start offsets (len parts+1) of an as-even-as-possible split of n."""
    base, extra = divmod(int(n), int(parts))
    starts = [0]
    for q in range(parts):
        starts.append(starts[-1] + base + (1 if q < extra else 0))
    return starts


class CudaBackend:
    """libvx on torch CUDA tensors (the product path)."""

    def __init__(self, ctx=None):
        self.ctx = ctx or _lib.default_context()
        self.L = _lib.load()

    def pass12_scatter(self, occ_slab, dims, dst_ptrs, j_starts, x_base: int):
        nx, ny, nz = dims
        nxl = int(occ_slab.shape[0])
        ptrs = (ctypes.c_void_p * len(dst_ptrs))(*[int(p) for p in dst_ptrs])
        js = (ctypes.c_int * len(j_starts))(*[int(v) for v in j_starts])
        _lib.check(self.L.vx_edt_pass12_scatter(
            self.ctx.handle, ctypes.c_void_p(occ_slab.data_ptr()), nx, ny, nz, nxl,
            len(dst_ptrs), ptrs, js, int(x_base), None, 0))

    def pass3(self, s2_jslab, site_jslab, dims, j0: int):
        nx, ny, nz = dims
        nyl = int(s2_jslab.shape[1])
        _lib.check(self.L.vx_edt_pass3_device(
            self.ctx.handle, ctypes.c_void_p(s2_jslab.data_ptr()), nx, ny, nz, int(j0), nyl,
            ctypes.c_void_p(site_jslab.data_ptr()), None, 0))

    def stream(self):
        import torch
        return torch.cuda.ExternalStream(self.ctx.stream_handle())

    def synchronize(self):
        """Wait for the library stream (and torch's, which carries the copies
        and collectives) so the next stage sees all writes."""
        import torch
        self.ctx.synchronize()
        torch.cuda.synchronize()


class SlabEDT:
    """Exact EDT of a (nx, ny, nz) grid held as i-slabs by the ranks of a
    torch.distributed group.  Call with this rank's occupancy slab
    (uint8, (i1-i0, ny, nz)); returns its j-slab of the site array (int32,
    (nx, j1-j0, nz), global flat indices)."""

    def __init__(self, dims, group=None, exchange: str = "nccl", backend=None, device=None):
        import torch
        import torch.distributed as dist
        self.dims = tuple(int(d) for d in dims)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.exchange = exchange
        self.backend = backend or CudaBackend()
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else
            torch.device("cpu"))
        nx, ny, nz = self.dims
        if self.world > nx or self.world > ny:
            raise ValueError("more ranks than slices along i or j")
        self.i_starts = even_split(nx, self.world)
        self.j_starts = even_split(ny, self.world)
        r = self.rank
        self.nxl = self.i_starts[r + 1] - self.i_starts[r]
        self.nyl = self.j_starts[r + 1] - self.j_starts[r]
        # receive buffer (this rank's pass-3 input) and send blocks
        self.recv = torch.empty((nx, self.nyl, nz), dtype=torch.int32, device=self.device)
        self.site = torch.empty((nx, self.nyl, nz), dtype=torch.int32, device=self.device)
        self._symm = None
        if exchange == "nccl":
            self.send = torch.empty(self.nxl * ny * nz, dtype=torch.int32, device=self.device)
            self.in_splits = [self.nxl * (self.j_starts[q + 1] - self.j_starts[q]) * nz
                              for q in range(self.world)]
            self.out_splits = [(self.i_starts[q + 1] - self.i_starts[q]) * self.nyl * nz
                               for q in range(self.world)]
        else:
            self._setup_p2p()

    # -- p2p transport: peers' receive buffers mapped over NVLink --------------
    def _setup_p2p(self):
        import torch
        import torch.distributed._symmetric_memory as symm_mem
        nx, ny, nz = self.dims
        maxl = max(self.j_starts[q + 1] - self.j_starts[q] for q in range(self.world))
        buf = symm_mem.empty(nx * maxl * nz, dtype=torch.int32, device=self.device)
        import torch.distributed as dist
        hdl = symm_mem.rendezvous(buf, self.group if self.group is not None else dist.group.WORLD)
        self._symm = (buf, hdl)
        self.recv = buf[: nx * self.nyl * nz].view(nx, self.nyl, nz)
        self.peer_ptrs = []
        for q in range(self.world):
            nyl_q = self.j_starts[q + 1] - self.j_starts[q]
            peer = hdl.get_buffer(q, (nx * nyl_q * nz,), torch.int32)
            self.peer_ptrs.append(peer.data_ptr())

    def destinations(self):
        """(dst pointers, x_base) for this rank's pass-2 epilogue."""
        nz = self.dims[2]
        if self.exchange == "nccl":
            base = self.send.data_ptr()
            ptrs = [base + 4 * self.nxl * self.j_starts[q] * nz for q in range(self.world)]
            return ptrs, 0
        return self.peer_ptrs, self.i_starts[self.rank]

    def __call__(self, occ_slab):
        import torch
        import torch.distributed as dist
        if tuple(occ_slab.shape) != (self.nxl, self.dims[1], self.dims[2]):
            raise ValueError(f"rank {self.rank} expects a slab of shape "
                             f"{(self.nxl, self.dims[1], self.dims[2])}")
        ptrs, x_base = self.destinations()
        if self.exchange == "p2p":
            # every peer is done reading its receive buffer (the previous
            # call's pass 3) before anyone's pass-2 epilogue writes into it;
            # the barrier kernel runs on the library stream, so it is ordered
            # after this rank's pass 3 and before its pass 2
            with torch.cuda.stream(self.backend.stream()):
                self._symm[1].barrier()
        self.backend.pass12_scatter(occ_slab, self.dims, ptrs, self.j_starts, x_base)
        if self.exchange == "nccl":
            self.backend.synchronize()
            if self.world > 1:
                dist.all_to_all_single(self.recv.view(-1), self.send, self.out_splits,
                                       self.in_splits, group=self.group)
            else:
                self.recv.view(-1).copy_(self.send)
            self.backend.synchronize()
        else:
            # the peers' NVLink stores into this rank's buffer have landed
            # once every rank's pass 2 is past this barrier; pass 3 is queued
            # behind it on the same (library) stream
            with torch.cuda.stream(self.backend.stream()):
                self._symm[1].barrier()
        self.backend.pass3(self.recv, self.site, self.dims, self.j_starts[self.rank])
        self.backend.synchronize()
        return self.site


def emulate_ranks(occ, world: int, exchange: str = "p2p", backend=None):
    """Run the slab pipeline for `world` virtual ranks inside one process on
    one GPU (sequentially: no rank waits on another).  Exercises exactly the
    addressing each transport uses; returns the assembled site array.
    occ: torch uint8 (nx, ny, nz) on the backend's device."""
    import torch
    nx, ny, nz = (int(d) for d in occ.shape)
    be = backend or CudaBackend()
    i_starts, j_starts = even_split(nx, world), even_split(ny, world)
    nyl = [j_starts[q + 1] - j_starts[q] for q in range(world)]
    recv = [torch.empty((nx, nyl[q], nz), dtype=torch.int32, device=occ.device) for q in range(world)]
    for r in range(world):
        i0, i1 = i_starts[r], i_starts[r + 1]
        slab = occ[i0:i1].contiguous()
        if exchange == "p2p":
            be.pass12_scatter(slab, (nx, ny, nz), [t.data_ptr() for t in recv], j_starts, i0)
        else:   # send blocks, then the all-to-all as block copies
            send = torch.empty((i1 - i0) * ny * nz, dtype=torch.int32, device=occ.device)
            ptrs = [send.data_ptr() + 4 * (i1 - i0) * j_starts[q] * nz for q in range(world)]
            be.pass12_scatter(slab, (nx, ny, nz), ptrs, j_starts, 0)
            be.synchronize()
            for q in range(world):
                off = (i1 - i0) * j_starts[q] * nz
                blk = send[off: off + (i1 - i0) * nyl[q] * nz].view(i1 - i0, nyl[q], nz)
                recv[q][i0:i1].copy_(blk)
            be.synchronize()
        be.synchronize()
    out = torch.empty((nx, ny, nz), dtype=torch.int32, device=occ.device)
    for q in range(world):
        site = torch.empty_like(recv[q])
        be.pass3(recv[q], site, (nx, ny, nz), j_starts[q])
        be.synchronize()
        out[:, j_starts[q]:j_starts[q + 1]] = site
    be.synchronize()
    return out


__all__ = ["SlabEDT", "emulate_ranks", "even_split", "CudaBackend"]
