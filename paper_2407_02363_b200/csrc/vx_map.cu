// Map-side kernels: device-resident log-odds grid (voxarm grids.py).
//
//   K0 k_reset     VoxelGrid.clear             grids.py:146-147 (sparse: only
//                  voxels touched since the last clear; dense on overflow)
//   K1 k_scatter   insert_point_cloud          grids.py:149-188 (k_neighbors=0)
//      k_finalize  the bincount/clip epilogue  grids.py:185-187
//   K2 k_stamp     insert_voxel_set            grids.py:190-203 (many link
//                  voxel sets, one launch; per-set FK transform)
//      k_occupancy occupancy_mask              grids.py:207-208
//
// Float semantics follow numpy exactly: float64 discretisation with IEEE
// division and floor (grids.py:137); hits counted as integers and applied as
// clip(cell + f32(count) * f32(hit)) in float32 (grids.py:185-187, NEP 50
// weak-scalar promotion) -- never per-point float atomics; the float32
// threshold compare (numpy casts the python-float logit to float32).  The
// rigid transform of voxel-set centres is evaluated as numpy's OpenBLAS dgemm
// does on this image: fma(c2, r2, fma(c1, r1, c0*r0)) + t.
#include "vx_internal.cuh"

#include <algorithm>

namespace vx {
namespace {

constexpr float kLMin = -2.0f;  // grids.py:18
constexpr float kLMax = 3.5f;   // grids.py:19

__device__ __forceinline__ float clip_logodds(float c) {
    // np.clip semantics: NaN propagates
    if (c < kLMin) return kLMin;
    if (c > kLMax) return kLMax;
    return c;
}

// floor((p - origin) / vs) per axis; -1 when outside [0, dims)  (grids.py:134-139)
__device__ __forceinline__ long long discretize(double px, double py, double pz, const GridGeom &g) {
    const double fx = floor(__ddiv_rn(__dsub_rn(px, g.ox), g.vs));
    const double fy = floor(__ddiv_rn(__dsub_rn(py, g.oy), g.vs));
    const double fz = floor(__ddiv_rn(__dsub_rn(pz, g.oz), g.vs));
    if (!(fx >= 0.0) || !(fx < (double)g.nx)) return -1;
    if (!(fy >= 0.0) || !(fy < (double)g.ny)) return -1;
    if (!(fz >= 0.0) || !(fz < (double)g.nz)) return -1;
    return ((long long)fx * g.ny + (long long)fy) * g.nz + (long long)fz;
}

// warp-aggregated counter add (one atomic per warp)
__device__ __forceinline__ void warp_sum(unsigned long long *dst, int v) {
    const int t = __reduce_add_sync(VX_FULL_MASK, (unsigned)v);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(dst, (unsigned long long)t);
}

__device__ __forceinline__ void warp_count(unsigned long long *dst, bool pred) {
    const unsigned m = __ballot_sync(VX_FULL_MASK, pred);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(dst, (unsigned long long)__popc(m));
}

// true in exactly one thread of the last block to finish: it commits the
// grid's counters once every block has read them (saves a 1-thread launch)
__device__ __forceinline__ bool last_block(DevCounters *ctr) {
    __shared__ bool is_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(&ctr->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && is_last) {
        ctr->done = 0u;
        __threadfence();
        return true;
    }
    return false;
}

__device__ __forceinline__ void reset_body(const ResetArgs &r, long long tid, long long nth) {
    const bool dense = r.dense || r.ctr->overflow;
    if (dense) {
        const long long n4 = r.n >> 2;  // cells are 16-byte aligned (cudaMalloc)
        float4 *c4 = reinterpret_cast<float4 *>(r.cells);
        uint32_t *o4 = reinterpret_cast<uint32_t *>(r.occ);
        for (long long v = tid; v < n4; v += nth) {
            c4[v] = make_float4(0.f, 0.f, 0.f, 0.f);
            o4[v] = 0u;
        }
        for (long long v = (n4 << 2) + tid; v < r.n; v += nth) {
            r.cells[v] = 0.f;
            r.occ[v] = 0;
        }
    } else {
        const int cnt = r.ctr->touched;
        for (long long t = tid; t < cnt; t += nth) {
            const int v = r.touched[t];
            r.cells[v] = 0.f;
            r.occ[v] = 0;
        }
    }
    if (last_block(r.ctr)) {   // commit
        r.ctr->touched = 0;
        r.ctr->pending = 0;
        r.ctr->overflow = 0;
        r.ctr->dirty = 1;
    }
}

__global__ void k_reset(ResetArgs r) {
    reset_body(r, (long long)blockIdx.x * blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
}

// the camera tick's resets in one launch: blockIdx.y picks the grid (each
// commits in its own last block); block (0, 0) also zeroes up to three small
// buffers (slice flags, per-link OOB counters, insert stats) that would
// otherwise be memset nodes of their own
// Block (0, 1) also copies `cp` (the camera tick's per-step arguments, read
// straight from the host-mapped staging slot, so the tick needs no H2D copy
// of its own; the graph node's source pointer is updated per tick).
__global__ void k_reset2(ResetArgs a, ResetArgs b, ZeroSpan z0, ZeroSpan z1, ZeroSpan z2, CopySpan cp) {
    if (blockIdx.x == 0 && blockIdx.y == 0) {
        for (const ZeroSpan &z : {z0, z1, z2})
            for (size_t i = threadIdx.x; i < z.bytes; i += blockDim.x) static_cast<unsigned char *>(z.p)[i] = 0;
    }
    if (blockIdx.x == 0 && blockIdx.y == 1 && cp.bytes) {
        const uint4 *src = static_cast<const uint4 *>(cp.src);
        uint4 *dst = static_cast<uint4 *>(cp.dst);
        for (size_t i = threadIdx.x; i < cp.bytes / 16; i += blockDim.x) dst[i] = src[i];
    }
    reset_body(blockIdx.y ? b : a, (long long)blockIdx.x * blockDim.x + threadIdx.x,
               (long long)gridDim.x * blockDim.x);
}

// clip untouched voxels (only needed after host writes put cells out of
// range): grids.py:187 clips every voxel whenever any point was inserted
__global__ void k_dense_clip(float *__restrict__ cells, const uint32_t *__restrict__ counts,
                             long long n, const DevCounters *__restrict__ ctr) {
    if (ctr->inserted == 0) return;
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nth)
        if (counts[v] == 0) cells[v] = clip_logodds(__fadd_rn(cells[v], 0.0f));
}

// VX_SCATTER_U points per thread per trip, their loads, mask lookups and
// count atomics issued back to back: the per-point chain (point load ->
// mask load -> returning atomic) is latency-bound, and one wave of CTAs with
// U independent chains per thread beats two waves of single chains
#ifndef VX_SCATTER_U
#define VX_SCATTER_U 2
#endif
__global__ void __launch_bounds__(256, 4)
k_scatter(const double *__restrict__ pts, long long npts,
          const long long *__restrict__ npts_dev, GridGeom g,
          const float *__restrict__ mask_cells, float thr,
          uint32_t *__restrict__ counts, int32_t *__restrict__ touched,
          DevCounters *__restrict__ ctr, int capacity, const uint8_t *__restrict__ keep) {
    constexpr int U = VX_SCATTER_U;
    const long long n = npts_dev ? *npts_dev : npts;
    // pts == nullptr: npts_dev heads a device block {count, cloud pointer}
    // (the camera tick's staged arguments, so its graph needs no cloud copy)
    if (!pts) pts = *reinterpret_cast<const double *const *>(npts_dev + 1);
    const int base = ctr->touched;
    __shared__ int s_cnt, s_base;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    // uniform trip count so the warp-aggregated counters see full warps
    const long long trips = (n + nth * U - 1) / (nth * U);
    for (long long it = 0; it < trips; ++it) {
        bool oob[U], skip[U], ins[U], first[U];
        long long lin[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = start + (it * U + u) * nth;
            oob[u] = skip[u] = ins[u] = first[u] = false;
            lin[u] = -2;
            if (p < n && (!keep || keep[p])) {   // outliers were removed before discretising (grids.py:166-170)
                const double x = pts[3 * p], y = pts[3 * p + 1], z = pts[3 * p + 2];
                lin[u] = discretize(x, y, z, g);
                oob[u] = lin[u] < 0;                                 // grids.py:171
            }
        }
        float mv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            mv[u] = (mask_cells && lin[u] >= 0) ? mask_cells[lin[u]] : 0.0f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (lin[u] < 0) continue;
            if (mask_cells && mv[u] > thr) {
                skip[u] = true;                                      // grids.py:178-182
            } else {
                ins[u] = true;
                first[u] = atomicAdd(&counts[lin[u]], 1u) == 0u;     // first touch
            }
        }
        // first touches join the touched list with one global atomic per block
        // (a per-warp atomic on the one counter serialised ~10k requests)
        unsigned fm[U];
        int wofs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            fm[u] = __ballot_sync(VX_FULL_MASK, first[u]);
            wofs[u] = 0;
            if (lane == 0 && fm[u]) wofs[u] = atomicAdd(&s_cnt, __popc(fm[u]));
            wofs[u] = __shfl_sync(VX_FULL_MASK, wofs[u], 0);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_base = s_cnt ? atomicAdd(&ctr->pending, s_cnt) : 0;
            s_cnt = 0;
        }
        __syncthreads();
        int ns = 0, nk = 0, ni = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (first[u]) {
                const int slot = base + s_base + wofs[u] + __popc(fm[u] & ((1u << lane) - 1u));
                if (slot < capacity) touched[slot] = (int32_t)lin[u];
                else ctr->overflow = 1;
            }
            ns += oob[u]; nk += skip[u]; ni += ins[u];
        }
        __syncthreads();   // s_base is rewritten next iteration
        warp_sum(&ctr->oob, ns);
        warp_sum(&ctr->skipped, nk);
        warp_sum(&ctr->inserted, ni);
    }
}

// fresh: the grid was reset before this insert, so its cells are all +0.0f
// and the scatter counted hits in the cells' own bits (counts == cells): one
// random read and one write fewer per touched voxel.  0.0f + f32(c) * hit is
// exactly f32(c) * hit, so the result equals the general path's.
__device__ __forceinline__ bool apply_hits(float *cells, uint8_t *occ, uint32_t *counts,
                                           long long v, float hit, float occ_thr, bool fresh) {
    const uint32_t c = counts[v];
    if (fresh) {
        const float cell = clip_logodds(__fmul_rn((float)c, hit));
        cells[v] = cell;
        occ[v] = cell > occ_thr ? 1 : 0;
        return cell > occ_thr;
    }
    counts[v] = 0u;
    // np.clip(flat + hits * hit, L_MIN, L_MAX): f32 multiply, f32 add (no fma)
    const float h = __fmul_rn((float)c, hit);
    const float cell = clip_logodds(__fadd_rn(cells[v], h));
    cells[v] = cell;
    occ[v] = cell > occ_thr ? 1 : 0;
    return cell > occ_thr;
}

__global__ void k_finalize(float *__restrict__ cells, uint8_t *__restrict__ occ,
                           uint32_t *__restrict__ counts, const int32_t *__restrict__ touched,
                           DevCounters *__restrict__ ctr, long long n, float hit,
                           float occ_thr, int capacity, int fresh, uint8_t *__restrict__ sflag,
                           long long plane, int nx, int *__restrict__ xs, int *__restrict__ hdr,
                           int *__restrict__ m_mirror) {
    // sflag (fresh grids only): every occupied voxel is one of this insert's,
    // so the EDT's occupied-slice flags are set here (per-CTA bitmap, one
    // store per slice and CTA) and need no pass over the touched list
    __shared__ unsigned bits[1024];
    const bool local = sflag && nx <= 32768;
    if (local)
        for (int w = threadIdx.x; w < (nx + 31) / 32; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    auto mark = [&](long long v) {
        if (!sflag) return;
        const int i = (int)(v / plane);
        if (local) atomicOr(&bits[i >> 5], 1u << (i & 31));
        else sflag[i] = 1;
    };
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (ctr->overflow) {  // the touched list is incomplete: scan every voxel
        for (long long v = tid; v < n; v += nth)
            if (counts[v] && apply_hits(cells, occ, counts, v, hit, occ_thr, fresh != 0)) mark(v);
    } else {
        const int base = ctr->touched, cnt = ctr->pending;
        for (long long t = tid; t < cnt; t += nth) {
            const int v = touched[base + t];
            VX_ASSERT(v >= 0 && v < n, "finalize voxel");
            if (apply_hits(cells, occ, counts, v, hit, occ_thr, fresh != 0)) mark(v);
        }
    }
    if (local) {
        __syncthreads();
        for (int w = threadIdx.x; w < (nx + 31) / 32; w += blockDim.x)
            for (unsigned b = bits[w]; b; b &= b - 1) sflag[w * 32 + __ffs(b) - 1] = 1;
    }
    // last block: commit; with xs it also builds the EDT's occupied-slice list
    // from the finished flags (what k_slice_list would do in a launch of its own)
    __shared__ bool is_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(&ctr->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    if (threadIdx.x == 0) {   // commit
        ctr->done = 0u;
        __threadfence();
        const long long t = (long long)ctr->touched + ctr->pending;
        ctr->touched = t > capacity ? capacity : (int)t;
        ctr->pending = 0;
        if (ctr->inserted) ctr->dirty = 1;
    }
    if (!xs) return;
    __threadfence();
    __shared__ int wsum[32];
    __shared__ int base_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    for (int c0 = 0; c0 < nx; c0 += blockDim.x) {   // ascending slice indices
        const int x = c0 + threadIdx.x;
        const int f = (x < nx && __ldcg(sflag + x)) ? 1 : 0;
        const unsigned fm = __ballot_sync(VX_FULL_MASK, f);
        if (lane == 0) wsum[warp] = __popc(fm);
        __syncthreads();
        int wbase = 0, tot = 0;
        for (int q = 0; q < nwarps; ++q) {
            if (q < warp) wbase += wsum[q];
            tot += wsum[q];
        }
        const int base = base_s;
        if (f) xs[base + wbase + __popc(fm & ((1u << lane) - 1u))] = x;
        __syncthreads();
        if (threadIdx.x == 0) base_s = base + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        hdr[0] = base_s;
        hdr[32] = hdr[33] = 0;   // the one-warp pass 3's tile counters (vx_edt.cu k_pass3_stream)
        if (m_mirror) *(volatile int *)m_mirror = base_s;   // host-mapped hint
    }
}

__global__ void k_stamp(const int32_t *__restrict__ ijk, const long long *__restrict__ offsets,
                        int nsets, const double *__restrict__ set_origin,
                        const double *__restrict__ set_vs, const double *__restrict__ T,
                        GridGeom g, float *__restrict__ cells, uint8_t *__restrict__ occ,
                        float value, float occ_thr, int32_t *__restrict__ touched,
                        DevCounters *__restrict__ ctr, unsigned long long *__restrict__ oob_per_set,
                        int capacity, long long total) {
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += nth) {
        int s = 0;
        while (s + 1 < nsets && q >= offsets[s + 1]) ++s;
        const double vs = set_vs[s];
        // VoxelSet.centers(): origin + (idx + 0.5) * vs   (grids.py:87-88)
        double c[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
            c[a] = __dadd_rn(set_origin[3 * s + a],
                             __dmul_rn(__dadd_rn((double)ijk[3 * q + a], 0.5), vs));
        double p[3];
        if (T) {
            const double *M = T + 16 * s;  // row-major 4x4; c @ R.T + t  (grids.py:198)
#pragma unroll
            for (int a = 0; a < 3; ++a)
                p[a] = __dadd_rn(__fma_rn(c[2], M[4 * a + 2],
                                          __fma_rn(c[1], M[4 * a + 1], __dmul_rn(c[0], M[4 * a]))),
                                 M[4 * a + 3]);
        } else {
            p[0] = c[0]; p[1] = c[1]; p[2] = c[2];
        }
        const long long lin = discretize(p[0], p[1], p[2], g);
        if (lin < 0) {
            atomicAdd(&oob_per_set[s], 1ull);
            continue;
        }
        // grids.py:202.  Only a voxel whose cell was +0.0f joins the touched
        // list: any other value is already on it (a grid whose list is
        // incomplete resets densely anyway), so repeated stamps of one voxel
        // (several link voxels per cell, links overlapping) append it once.
        const float old = atomicExch(&cells[lin], value);
        occ[lin] = value > occ_thr ? 1 : 0;
        // one touched-list atomic per warp (lanes that took `continue` are inactive)
        const unsigned am = __activemask();
        const unsigned fm = __ballot_sync(am, __float_as_uint(old) == 0u);
        const int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
        int wbase = 0;
        if (lane == leader && fm) wbase = atomicAdd(&ctr->touched, __popc(fm));
        wbase = __shfl_sync(am, wbase, leader);
        if (fm & (1u << lane)) {
            const int slot = wbase + __popc(fm & ((1u << lane) - 1u));
            if (slot < capacity) touched[slot] = (int32_t)lin;
            else ctr->overflow = 1;
        }
    }
    if (last_block(ctr)) {   // commit
        if (ctr->touched > capacity) ctr->touched = capacity;
        ctr->dirty = 1;
    }
}

__global__ void k_stamp_commit(DevCounters *ctr, int capacity) {
    if (ctr->touched > capacity) ctr->touched = capacity;
    ctr->dirty = 1;
}

__global__ void k_occupancy(const float *__restrict__ cells, uint8_t *__restrict__ out, long long n,
                            float thr) {
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += nth)
        out[v] = cells[v] > thr ? 1 : 0;                              // grids.py:207-208
}

// Occupancy-set digest (the engine's memo key, engine.py:259-268, without the
// N-byte copy and blake2b): two order-independent 64-bit sums of mixed voxel
// indices plus the count, so any traversal order gives the same digest.  From
// the touched list (unique first touches since the last clear) when it covers
// every occupied voxel: O(K); otherwise over the whole occupancy array.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ void digest_add(unsigned long long *out, bool occ, long long v) {
    unsigned long long a = occ ? mix64((unsigned long long)v) : 0ull;
    unsigned long long b = occ ? mix64((unsigned long long)v ^ 0xD6E8FEB86659FD93ull) : 0ull;
    unsigned c = occ ? 1u : 0u;
    for (int d = 16; d; d >>= 1) {   // warp sums, one atomic per warp and word
        a += __shfl_xor_sync(VX_FULL_MASK, a, d);
        b += __shfl_xor_sync(VX_FULL_MASK, b, d);
        c += __shfl_xor_sync(VX_FULL_MASK, c, d);
    }
    if ((threadIdx.x & 31) == 0 && c) {
        atomicAdd(out, a);
        atomicAdd(out + 1, b);
        atomicAdd(out + 2, (unsigned long long)c);
    }
}

__global__ void k_occ_digest(const uint8_t *__restrict__ occ, long long n, const int32_t *__restrict__ touched,
                             const DevCounters *__restrict__ ctr, int use_list, unsigned long long *__restrict__ out) {
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (use_list && !ctr->overflow) {
        const long long cnt = ctr->touched;
        const long long trips = (cnt + nth - 1) / nth;   // uniform trip count: full warps
        for (long long it = 0; it < trips; ++it) {
            const long long t = tid + it * nth;
            const int v = t < cnt ? touched[t] : -1;
            digest_add(out, v >= 0 && occ[v] != 0, v);
        }
    } else {
        const long long trips = (n + nth - 1) / nth;
        for (long long it = 0; it < trips; ++it) {
            const long long v = tid + it * nth;
            digest_add(out, v < n && occ[v] != 0, v);
        }
    }
}

unsigned grid_for(long long work, int block) {
    long long g = (work + block - 1) / block;
    const long long cap = (long long)num_sms() * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace

cudaError_t launch_reset(float *cells, uint8_t *occ, int32_t *touched, DevCounters *ctr, int64_t n,
                         int capacity, bool dense, cudaStream_t st) {
    (void)capacity;
    // the sparse count is only known on the device: size for the dense case
    // when asked, otherwise for a persistent grid-stride sweep
    const unsigned g = dense ? grid_for(n / 4 + 1, 256) : (unsigned)(num_sms() * 4);
    k_reset<<<g, 256, 0, st>>>(ResetArgs{cells, occ, touched, ctr, n, dense ? 1 : 0});   // commits in its last block
    return cudaGetLastError();
}

cudaError_t launch_reset2(const ResetArgs &a, const ResetArgs &b, ZeroSpan z0, ZeroSpan z1, ZeroSpan z2,
                          cudaStream_t st, CopySpan cp) {
    const long long work = std::max(a.dense ? a.n / 4 + 1 : 0LL, b.dense ? b.n / 4 + 1 : 0LL);
    const unsigned g = work ? std::max(grid_for(work, 256), (unsigned)(num_sms() * 2)) : (unsigned)(num_sms() * 2);
    k_reset2<<<dim3(g, 2), 256, 0, st>>>(a, b, z0, z1, z2, cp);
    return cudaGetLastError();
}

cudaError_t launch_dense_clip(float *cells, const uint32_t *counts, int64_t n,
                              const DevCounters *ctr, cudaStream_t st) {
    k_dense_clip<<<grid_for(n, 256), 256, 0, st>>>(cells, counts, n, ctr);
    return cudaGetLastError();
}

cudaError_t launch_scatter(const double *pts, int64_t npts, const int64_t *npts_dev, GridGeom g,
                           const float *mask_cells, float thr, uint32_t *counts, int32_t *touched,
                           DevCounters *ctr, int capacity, cudaStream_t st, const uint8_t *keep) {
    if (npts <= 0 && !npts_dev) return cudaSuccess;
    k_scatter<<<grid_for((npts + VX_SCATTER_U - 1) / VX_SCATTER_U, 256), 256, 0, st>>>(pts, npts, (const long long *)npts_dev, g,
                                                   mask_cells, thr, counts, touched, ctr, capacity, keep);
    return cudaGetLastError();
}

cudaError_t launch_finalize(float *cells, uint8_t *occ, uint32_t *counts, int32_t *touched,
                            DevCounters *ctr, int64_t n, int capacity, int64_t max_new, float hit,
                            float occ_thr, cudaStream_t st, bool fresh, uint8_t *sflag, long long plane,
                            int nx, int *xs, int *hdr, int *m_mirror) {
    // grid-stride over the new touched entries (<= max_new; a dense overflow
    // sweep loops): few blocks, so the last-block commit's atomic is cheap
    const long long work = n < max_new ? n : max_new;
    const unsigned gf = (unsigned)std::min<long long>(grid_for(work, 256), 2LL * num_sms());
    k_finalize<<<gf, 256, 0, st>>>(cells, occ, counts, touched, ctr, n, hit, occ_thr, capacity, fresh ? 1 : 0,
                                   sflag, plane, nx, sflag ? xs : nullptr, hdr, m_mirror);
    return cudaGetLastError();
}

cudaError_t launch_stamp(const int32_t *ijk, const int64_t *offsets, int nsets,
                         const double *set_origin, const double *set_vs, const double *T,
                         GridGeom g, float *cells, uint8_t *occ, float value, float occ_thr,
                         int32_t *touched, DevCounters *ctr, unsigned long long *oob_per_set,
                         int capacity, int64_t total, cudaStream_t st) {
    if (total > 0)   // commits in its last block
        k_stamp<<<grid_for(total, 256), 256, 0, st>>>(ijk, (const long long *)offsets, nsets,
                                                      set_origin, set_vs, T, g, cells, occ, value,
                                                      occ_thr, touched, ctr, oob_per_set, capacity,
                                                      total);
    else
        k_stamp_commit<<<1, 1, 0, st>>>(ctr, capacity);
    return cudaGetLastError();
}

cudaError_t launch_occ_digest(const uint8_t *occ, int64_t n, const int32_t *touched, const DevCounters *ctr,
                              bool use_list, unsigned long long *out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, 3 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    k_occ_digest<<<(unsigned)(num_sms() * 4), 256, 0, st>>>(occ, n, touched, ctr, use_list ? 1 : 0, out);
    return cudaGetLastError();
}

cudaError_t launch_occupancy(const float *cells, uint8_t *out, int64_t n, float thr,
                             cudaStream_t st) {
    k_occupancy<<<grid_for(n, 256), 256, 0, st>>>(cells, out, n, thr);
    return cudaGetLastError();
}

}  // namespace vx
