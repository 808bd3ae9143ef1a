"""One large grid across G GPUs: slab decomposition along the slow axis i
(1024^3 on 2/4/8 B200).

Rank r owns the i-slab [i0_r, i1_r) of the occupancy.  Passes 1 (along k)
and 2 (along j) are local to a slab (edt.py:168-317 never mix slices).  Pass 3
(along i, edt.py:320-420) needs every slice of a column, so the pass-2 codes
are transposed from i-slabs to j-slabs: rank q receives rows j in
[j0_q, j1_q) of every slice, i.e. a (nx, nyl_q, nz) array, and runs pass 3
on it with global coordinates.  The result stays j-sliced (no transpose
back): rank q holds site[:, j0_q:j1_q, :] with global flat indices.  Sphere
queries (engine.py:212-221) go to the rank that owns a centre's row j
(site_world: every rank answers its rows, one small all-gather).

The exchange is fused into pass 2's epilogue (vx_edt_pass12_scatter): each
code row is stored straight to its destination, so there is no pack pass.
Rows a rank keeps are stored into its own receive buffer.  Two transports:
  * "nccl": the destinations are this rank's send blocks, and NCCL
    send/recv moves them.  The slab is processed in `chunks` slice groups:
    chunk c's sends and receives are issued (grouped, on the library stream,
    no host synchronisation) as soon as its pass 2 is queued, so NVLink
    carries chunk c while pass 2 computes chunk c+1; pass 3 waits on the
    receives on the same stream;
  * "p2p":  the destinations are the peers' receive buffers themselves,
    mapped into this process over NVLink (torch symmetric memory); the
    transfer overlaps pass-2 compute tile by tile and a barrier on the
    library stream replaces the collective.
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

    def site_world_slab(self, site_jslab, dims, j0: int, centers, origin, voxel_size: float):
        nx, ny, nz = dims
        c = np.ascontiguousarray(centers, np.float64).reshape(-1, 3)
        s = c.shape[0]
        lin = np.empty(s, np.int32)
        world = np.empty((s, 3), np.float64)
        dist = np.empty(s, np.float64)
        org = np.ascontiguousarray(origin, np.float64).reshape(3)
        _lib.check(self.L.vx_site_world_slab(
            self.ctx.handle, ctypes.c_void_p(site_jslab.data_ptr()), nx, ny, nz, int(j0),
            int(site_jslab.shape[1]), _lib.ptr(org), float(voxel_size), _lib.ptr(c), s,
            _lib.ptr(lin), _lib.ptr(world), _lib.ptr(dist)))
        return lin, world, dist

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
    (nx, j1-j0, nz), global flat indices), ordered before later work on the
    caller's current stream."""

    def __init__(self, dims, group=None, exchange: str = "nccl", backend=None, device=None,
                 chunks: int | None = None):
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
        # slice groups of the pipelined exchange (the same split rule on every rank)
        self.chunks = max(1, int(chunks if chunks is not None else (4 if self.world > 1 else 1)))
        self.c_starts = [even_split(self.i_starts[q + 1] - self.i_starts[q], self.chunks)
                         for q in range(self.world)]
        # receive buffer (this rank's pass-3 input) and send blocks
        self.recv = torch.empty((nx, self.nyl, nz), dtype=torch.int32, device=self.device)
        self.site = torch.empty((nx, self.nyl, nz), dtype=torch.int32, device=self.device)
        self._symm = None
        if exchange == "nccl":
            # chunk-major send blocks: chunk c, destination q -> [slices of c][nyl_q][nz]
            self.send = torch.empty(max(1, self.nxl * ny * nz), dtype=torch.int32, device=self.device)
        else:
            self._setup_p2p()

    # -- p2p transport: peers' receive buffers mapped over NVLink --------------
    def _setup_p2p(self):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        nx, ny, nz = self.dims
        maxl = max(self.j_starts[q + 1] - self.j_starts[q] for q in range(self.world))
        buf = symm_mem.empty(nx * maxl * nz, dtype=torch.int32, device=self.device)
        hdl = symm_mem.rendezvous(buf, self.group if self.group is not None else dist.group.WORLD)
        self._symm = (buf, hdl)
        self.recv = buf[: nx * self.nyl * nz].view(nx, self.nyl, nz)
        self.peer_ptrs = []
        for q in range(self.world):
            nyl_q = self.j_starts[q + 1] - self.j_starts[q]
            peer = hdl.get_buffer(q, (nx * nyl_q * nz,), torch.int32)
            self.peer_ptrs.append(peer.data_ptr())

    def _send_block(self, c: int, q: int):
        """(offset, count) of chunk c's block for destination q in self.send."""
        ny, nz = self.dims[1], self.dims[2]
        cs = self.c_starts[self.rank]
        n_c = cs[c + 1] - cs[c]
        return cs[c] * ny * nz + n_c * self.j_starts[q] * nz, n_c * (self.j_starts[q + 1] - self.j_starts[q]) * nz

    def destinations(self, c: int = 0):
        """(dst pointers, x_base) of chunk c's pass-2 epilogue: send blocks
        (nccl) or peer receive buffers (p2p); this rank's own rows always go
        straight into its receive buffer."""
        nz = self.dims[2]
        r = self.rank
        x0 = self.i_starts[r] + self.c_starts[r][c]
        if self.exchange == "p2p":
            ptrs = [p + 4 * x0 * (self.j_starts[q + 1] - self.j_starts[q]) * nz
                    for q, p in enumerate(self.peer_ptrs)]
            return ptrs, 0
        own = self.recv.data_ptr() + 4 * x0 * self.nyl * nz
        base = self.send.data_ptr()
        return [own if q == r else base + 4 * self._send_block(c, q)[0] for q in range(self.world)], 0

    def _exchange_ops(self, c: int):
        """Chunk c's NCCL sends (this rank's rows for q) and receives (q's
        chunk-c slices of this rank's rows, straight into recv)."""
        import torch.distributed as dist
        nz = self.dims[2]
        ops = []
        for q in range(self.world):
            if q == self.rank:
                continue
            off, cnt = self._send_block(c, q)
            if cnt:
                ops.append(dist.P2POp(dist.isend, self.send[off:off + cnt], q, self.group))
            cq = self.c_starts[q]
            x0, x1 = self.i_starts[q] + cq[c], self.i_starts[q] + cq[c + 1]
            if (x1 - x0) * self.nyl * nz:
                ops.append(dist.P2POp(dist.irecv, self.recv[x0:x1].view(-1), q, self.group))
        return ops

    def __call__(self, occ_slab):
        import contextlib

        import torch
        import torch.distributed as dist
        if tuple(occ_slab.shape) != (self.nxl, self.dims[1], self.dims[2]):
            raise ValueError(f"rank {self.rank} expects a slab of shape "
                             f"{(self.nxl, self.dims[1], self.dims[2])}")
        cuda = self.device.type == "cuda"
        lib = self.backend.stream() if cuda else None
        caller = torch.cuda.current_stream(self.device) if cuda else None
        if cuda:   # the occupancy was produced on the caller's stream
            lib.wait_stream(caller)
        with torch.cuda.stream(lib) if cuda else contextlib.nullcontext():
            if self.exchange == "p2p":
                # every peer is done reading its receive buffer (the previous
                # call's pass 3) before anyone's pass-2 epilogue writes into it
                self._symm[1].barrier()
                ptrs, x_base = self.destinations(0)
                self.backend.pass12_scatter(occ_slab, self.dims, ptrs, self.j_starts, x_base)
                self._symm[1].barrier()   # the peers' NVLink stores have landed
            else:
                reqs = []
                cs = self.c_starts[self.rank]
                for c in range(self.chunks):
                    if cs[c + 1] > cs[c]:
                        ptrs, x_base = self.destinations(c)
                        self.backend.pass12_scatter(occ_slab[cs[c]:cs[c + 1]], self.dims, ptrs,
                                                    self.j_starts, x_base)
                    if self.world > 1:
                        ops = self._exchange_ops(c)
                        if ops:   # queued behind chunk c's pass 2 on this stream
                            reqs += dist.batch_isend_irecv(ops)
                for rq in reqs:   # the library stream waits for the transfers
                    rq.wait()
            self.backend.pass3(self.recv, self.site, self.dims, self.j_starts[self.rank])
        if cuda:
            caller.wait_stream(lib)
        else:
            self.backend.synchronize()
        return self.site

    def site_world(self, centers, origin, voxel_size: float):
        """_site_world (engine.py:212-221) plus the tasks.py:102-104 distance
        for every centre on the j-sliced field: each rank answers the centres
        whose clipped row j it holds (vx_site_world_slab), one all-gather of
        (S, 5) values picks the owner's answer.  Returns (lin int32 (S,),
        world (S,3), dist (S,)) on every rank, as engine.site_world does on a
        whole field (lin -1 / NaN / inf where there is no site)."""
        import torch
        import torch.distributed as dist
        if self.device.type == "cuda":
            torch.cuda.current_stream(self.device).synchronize()
        lin, world, dist_ = self.backend.site_world_slab(self.site, self.dims, self.j_starts[self.rank],
                                                         centers, origin, voxel_size)
        mine = np.concatenate([lin.astype(np.float64)[:, None], world, dist_[:, None]], axis=1)
        if self.world == 1:
            allv = [mine]
        else:
            t = torch.from_numpy(np.ascontiguousarray(mine)).to(self.device)
            parts = [torch.empty_like(t) for _ in range(self.world)]
            dist.all_gather(parts, t, group=self.group)
            allv = [p_.cpu().numpy() for p_ in parts]
        s = lin.shape[0]
        out_lin = np.full(s, -2, np.int32)
        out_world = np.empty((s, 3), np.float64)
        out_dist = np.empty(s, np.float64)
        for v in allv:
            own = v[:, 0] != -2
            out_lin[own] = v[own, 0].astype(np.int32)
            out_world[own] = v[own, 1:4]
            out_dist[own] = v[own, 4]
        return out_lin, out_world, out_dist


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
