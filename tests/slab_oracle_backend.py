"""Test-only backend for paper_2407_02363_b200.slab: the same pass interface
as CudaBackend, computed by the CPU oracle (oracle/) on CPU tensors, so the
multi-rank host logic (partitioning, fused-epilogue addressing, all-to-all
splits) runs under gloo on CPU.  Never used by the product."""
import ctypes

import numpy as np

from oracle import oracle as O


def _bits(v: int) -> int:
    b = 0
    while v > 0:
        b += 1
        v >>= 1
    return b


def _view(ptr: int, count: int) -> np.ndarray:
    return np.ctypeslib.as_array((ctypes.c_int32 * count).from_address(int(ptr)))


class OracleBackend:
    def pass12_scatter(self, occ_slab, dims, dst_ptrs, j_starts, x_base):
        nx, ny, nz = dims
        slab = occ_slab.numpy()
        zb = _bits(nz - 1)
        s1 = O.line_nearest_sites(slab)
        s2y, s2z = O.slice_transform(s1)
        codes = np.where(s2y >= 0, (s2y.astype(np.int64) << zb) | s2z, -1).astype(np.int32)
        nxl = slab.shape[0]
        for q in range(len(dst_ptrs)):
            j0, j1 = j_starts[q], j_starts[q + 1]
            nyl = j1 - j0
            if nyl == 0:
                continue
            cnt = (int(x_base) + nxl) * nyl * nz
            dst = _view(dst_ptrs[q], cnt).reshape(int(x_base) + nxl, nyl, nz)
            dst[int(x_base):int(x_base) + nxl] = codes[:, j0:j1, :]

    def pass3(self, s2_jslab, site_jslab, dims, j0):
        nx, ny, nz = dims
        zb = _bits(nz - 1)
        c = s2_jslab.numpy()
        valid = c != -1
        s2y = np.where(valid, c.view(np.uint32) >> zb, -1).astype(np.int32)
        s2z = np.where(valid, c & ((1 << zb) - 1), -1).astype(np.int32)
        site_jslab.numpy()[...] = O.column_transform_slab(s2y, s2z, j0, ny)

    def site_world_slab(self, site_jslab, dims, j0, centers, origin, voxel_size):
        """engine.py:212-221 on a j-slab (numpy): lin -2 for rows not held."""
        nx, ny, nz = dims
        site = site_jslab.numpy()
        nyl = site.shape[1]
        c = np.asarray(centers, np.float64).reshape(-1, 3)
        org = np.asarray(origin, np.float64)
        idx = np.clip(np.floor((c - org) / voxel_size).astype(np.int64), 0, np.array(dims) - 1)
        s = c.shape[0]
        lin = np.full(s, -2, np.int32)
        world = np.full((s, 3), np.nan)
        dist = np.full(s, np.nan)
        for q in range(s):
            i, j, k = idx[q]
            if not (j0 <= j < j0 + nyl):
                continue
            v = int(site[i, j - j0, k])
            lin[q] = v
            if v < 0:
                dist[q] = np.inf
                continue
            si, sj, sk = v // (ny * nz), (v // nz) % ny, v % nz
            world[q] = org + (np.array([si, sj, sk], np.float64) + 0.5) * voxel_size
            dist[q] = np.linalg.norm(world[q] - c[q])
        return lin, world, dist

    def synchronize(self):
        pass
