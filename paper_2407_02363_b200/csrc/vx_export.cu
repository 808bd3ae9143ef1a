// Field and grid export formats on the device:
//
//   k_sq_distance   DistanceField.sq_distance_grid   edt.py:123-135
//   k_dump_len/     DistanceField.dump_squared       edt.py:137-145
//   k_dump_write      (golden text, test_edt.py:248-253)
//   k_occ_count/    VoxelGrid.occupied_voxels        grids.py:210-212
//   k_occ_write       (np.argwhere: lexicographic = flat index order)
//
// All are HBM-bound byte/integer work.  The text dump is laid out by a
// per-line length pass and an exclusive scan, so every thread writes its own
// line at a known offset; occupied voxels are a stable stream compaction
// (per-chunk counts, scan, in-order write).
#include "vx_internal.cuh"

namespace vx {
namespace {

__device__ __forceinline__ long long sq_of(int32_t s, int i, int j, int k, int ny, int nz) {
    if (s == -1) return -1;   // NO_SITE
    const unsigned us = (unsigned)s, plane = (unsigned)ny * (unsigned)nz;
    const int si = (int)(us / plane);
    const unsigned r = us - (unsigned)si * plane;
    const int sj = (int)(r / (unsigned)nz), sk = (int)(r - (unsigned)sj * (unsigned)nz);
    const long long di = i - si, dj = j - sj, dk = k - sk;
    return di * di + dj * dj + dk * dk;
}

// one block row = one (i, j) line; threads across k (coalesced)
__global__ void k_sq_distance(const int32_t *__restrict__ site, int nx, int ny, int nz,
                              long long *__restrict__ out) {
    const long long rows = (long long)nx * ny;
    for (long long row = blockIdx.y; row < rows; row += gridDim.y) {
        const int i = (int)(row / ny), j = (int)(row - (long long)i * ny);
        const int32_t *src = site + row * nz;
        long long *dst = out + row * nz;
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nz; k += gridDim.x * blockDim.x)
            dst[k] = sq_of(src[k], i, j, k, ny, nz);
    }
}

__device__ __forceinline__ int ndigits(long long v) {   // v >= -1
    if (v < 0) return 2;   // "-1"
    int d = 1;
    while (v >= 10) {
        v /= 10;
        ++d;
    }
    return d;
}

__device__ __forceinline__ int header_len(int k) { return 8 + ndigits(k) + 1; }   // "slice k=" k "\n"

// thread per text line (j, k); threads across k so the site reads coalesce
__global__ void k_dump_len(const int32_t *__restrict__ site, int nx, int ny, int nz,
                           long long *__restrict__ len) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (k >= nz) return;
    long long n = nx;   // nx - 1 separators + the newline
    for (int i = 0; i < nx; ++i) n += ndigits(sq_of(site[((long long)i * ny + j) * nz + k], i, j, k, ny, nz));
    if (j == 0) n += header_len(k);
    len[(long long)k * ny + j] = n;
}

__device__ __forceinline__ char *put_int(char *p, long long v) {
    if (v < 0) {
        p[0] = '-';
        p[1] = '1';
        return p + 2;
    }
    char t[20];
    int n = 0;
    do {
        t[n++] = (char)('0' + v % 10);
        v /= 10;
    } while (v);
    while (n) *p++ = t[--n];
    return p;
}

__global__ void k_dump_write(const int32_t *__restrict__ site, int nx, int ny, int nz,
                             const long long *__restrict__ off, char *__restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (k >= nz) return;
    char *p = out + off[(long long)k * ny + j];
    if (j == 0) {
        const char h[8] = {'s', 'l', 'i', 'c', 'e', ' ', 'k', '='};
        for (int c = 0; c < 8; ++c) p[c] = h[c];
        p = put_int(p + 8, k);
        *p++ = '\n';
    }
    for (int i = 0; i < nx; ++i) {
        if (i) *p++ = ' ';
        p = put_int(p, sq_of(site[((long long)i * ny + j) * nz + k], i, j, k, ny, nz));
    }
    *p = '\n';
}

// exclusive scan of m int64 values into off[0..m], off[m] = total (one CTA)
__global__ void __launch_bounds__(1024) k_scan64(const long long *__restrict__ in, long long m,
                                                 long long *__restrict__ off) {
    __shared__ long long wsum[32];
    __shared__ long long base_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    for (long long c0 = 0; c0 < m; c0 += blockDim.x) {
        const long long idx = c0 + threadIdx.x;
        const long long v = idx < m ? in[idx] : 0;
        long long x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            long long w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += y;
            }
            wsum[lane] = w;   // inclusive over warps
        }
        __syncthreads();
        const long long base = base_s;
        const long long excl = base + (warp ? wsum[warp - 1] : 0) + x - v;
        if (idx < m) off[idx] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) base_s = base + wsum[(blockDim.x >> 5) - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) off[m] = base_s;
}

constexpr int kOccThreads = 256, kOccPer = 16, kOccChunk = kOccThreads * kOccPer;

__device__ __forceinline__ unsigned occ16(const uint8_t *__restrict__ occ, long long v0, long long n) {
    unsigned bits = 0;
    if (v0 + kOccPer <= n) {
        const uint4 q = *reinterpret_cast<const uint4 *>(occ + v0);
        const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int a = 0; a < 16; ++a) bits |= (((w[a >> 2] >> (8 * (a & 3))) & 0xffu) != 0u ? 1u : 0u) << a;
    } else {
        for (int a = 0; v0 + a < n; ++a) bits |= (occ[v0 + a] ? 1u : 0u) << a;
    }
    return bits;
}

__global__ void __launch_bounds__(kOccThreads) k_occ_count(const uint8_t *__restrict__ occ, long long n,
                                                          long long *__restrict__ cnt) {
    __shared__ int ws[kOccThreads / 32];
    const long long v0 = (long long)blockIdx.x * kOccChunk + (long long)threadIdx.x * kOccPer;
    int c = v0 < n ? __popc(occ16(occ, v0, n)) : 0;
#pragma unroll
    for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < kOccThreads / 32; ++w) t += ws[w];
        cnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kOccThreads) k_occ_write(const uint8_t *__restrict__ occ, long long n, int ny,
                                                          int nz, const long long *__restrict__ off,
                                                          long long *__restrict__ out) {
    __shared__ int ws[kOccThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long v0 = (long long)blockIdx.x * kOccChunk + (long long)threadIdx.x * kOccPer;
    const unsigned bits = v0 < n ? occ16(occ, v0, n) : 0u;
    const int c = __popc(bits);
    int x = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    long long pos = off[blockIdx.x] + x - c;
    for (int w = 0; w < warp; ++w) pos += ws[w];
    const long long plane = (long long)ny * nz;
    for (unsigned b = bits; b; b &= b - 1) {
        const long long v = v0 + __ffs(b) - 1;
        const long long i = v / plane, r = v - i * plane, j = r / nz;
        out[3 * pos] = i;
        out[3 * pos + 1] = j;
        out[3 * pos + 2] = r - j * nz;
        ++pos;
    }
}

}  // namespace

cudaError_t launch_sq_distance(const int32_t *site, int nx, int ny, int nz, long long *out, cudaStream_t st) {
    const int bx = nz >= 256 ? 256 : ((nz + 31) / 32) * 32;
    const long long rows = (long long)nx * ny;
    dim3 grid((unsigned)((nz + bx - 1) / bx), (unsigned)(rows < 65535 ? rows : 65535));
    k_sq_distance<<<grid, bx, 0, st>>>(site, nx, ny, nz, out);
    return cudaGetLastError();
}

size_t dump_scratch_bytes(int ny, int nz) { return (size_t)(2 * (long long)ny * nz + 1) * 8; }

// lengths + scan into scratch (dump_scratch_bytes); *total_dev = off[m]
cudaError_t launch_dump_layout(const int32_t *site, int nx, int ny, int nz, void *scratch, cudaStream_t st) {
    long long *len = (long long *)scratch, *off = len + (long long)ny * nz;
    dim3 grid((unsigned)((nz + 127) / 128), (unsigned)ny);
    k_dump_len<<<grid, 128, 0, st>>>(site, nx, ny, nz, len);
    k_scan64<<<1, 1024, 0, st>>>(len, (long long)ny * nz, off);
    return cudaGetLastError();
}

const long long *dump_total_ptr(void *scratch, int ny, int nz) {
    return (const long long *)scratch + 2 * (long long)ny * nz;
}

cudaError_t launch_dump_write(const int32_t *site, int nx, int ny, int nz, const void *scratch, char *out,
                              cudaStream_t st) {
    const long long *off = (const long long *)scratch + (long long)ny * nz;
    dim3 grid((unsigned)((nz + 127) / 128), (unsigned)ny);
    k_dump_write<<<grid, 128, 0, st>>>(site, nx, ny, nz, off, out);
    return cudaGetLastError();
}

size_t occ_scratch_bytes(long long n) {
    const long long nb = (n + kOccChunk - 1) / kOccChunk;
    return (size_t)(2 * nb + 1) * 8;
}

// per-chunk counts + scan; the total lands at occ_total_ptr
// brute_force_edt (edt.py:487-508): per voxel the minimum over every occupied
// voxel, ties to the lexicographically smallest (the sites arrive in flat-index
// order from the compaction, and only a strictly smaller distance replaces the
// current best).  O(N x sites): meant for the reference's test sizes (<= ~48^3).
// Sites are staged through shared memory in blocks of 1024.
__global__ void __launch_bounds__(256) k_brute_force(const long long *__restrict__ sites, long long nsites, int nx,
                                                     int ny, int nz, int32_t *__restrict__ out) {
    __shared__ int3 s[1024];
    const long long n = (long long)nx * ny * nz;
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int i = (int)(v / ((long long)ny * nz)), j = (int)((v / nz) % ny), k = (int)(v % nz);
    long long best = -1;
    long long bl = -1;
    for (long long b0 = 0; b0 < nsites; b0 += 1024) {
        const int nb = (int)min(1024LL, nsites - b0);
        __syncthreads();
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            const long long *q = sites + 3 * (b0 + t);
            s[t] = make_int3((int)q[0], (int)q[1], (int)q[2]);
        }
        __syncthreads();
        if (v < n) {
            for (int t = 0; t < nb; ++t) {
                const long long di = i - s[t].x, dj = j - s[t].y, dk = k - s[t].z;
                const long long d = di * di + dj * dj + dk * dk;
                if (best < 0 || d < best) {
                    best = d;
                    bl = ((long long)s[t].x * ny + s[t].y) * nz + s[t].z;
                }
            }
        }
    }
    if (v < n) out[v] = (int32_t)bl;   // -1 (NO_SITE) when there is no site
}

cudaError_t launch_brute_force(const long long *sites, long long nsites, int nx, int ny, int nz, int32_t *out,
                               cudaStream_t st) {
    const long long n = (long long)nx * ny * nz;
    if (n == 0) return cudaSuccess;
    k_brute_force<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sites, nsites, nx, ny, nz, out);
    return cudaGetLastError();
}

cudaError_t launch_occ_layout(const uint8_t *occ, long long n, void *scratch, cudaStream_t st) {
    const long long nb = (n + kOccChunk - 1) / kOccChunk;
    long long *cnt = (long long *)scratch, *off = cnt + nb;
    k_occ_count<<<(unsigned)nb, kOccThreads, 0, st>>>(occ, n, cnt);
    k_scan64<<<1, 1024, 0, st>>>(cnt, nb, off);
    return cudaGetLastError();
}

const long long *occ_total_ptr(void *scratch, long long n) {
    const long long nb = (n + kOccChunk - 1) / kOccChunk;
    return (const long long *)scratch + 2 * nb;
}

cudaError_t launch_occ_write(const uint8_t *occ, long long n, int ny, int nz, const void *scratch,
                             long long *out, cudaStream_t st) {
    const long long nb = (n + kOccChunk - 1) / kOccChunk;
    const long long *off = (const long long *)scratch + nb;
    k_occ_write<<<(unsigned)nb, kOccThreads, 0, st>>>(occ, n, ny, nz, off, out);
    return cudaGetLastError();
}

}  // namespace vx
