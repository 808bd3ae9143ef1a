// Statistical outlier filter on the GPU (voxarm grids.py:224-240,
// statistical_outlier_filter; used by insert_point_cloud when k_neighbors > 0,
// grids.py:166-169).
//
// Reference: cKDTree(pts).query(pts, k+1) -> dists; mean_knn = dists[:, 1:]
// .mean(axis=1); cutoff = mean_knn.mean() + m * mean_knn.std(); keep
// mean_knn <= cutoff; clouds with <= k points pass through.
//
// Here: exact kNN on a uniform hash grid (counting sort by cell; each point
// searches Chebyshev rings of cells until the (k+1)-th distance is inside the
// searched cube), distances sqrt((dx*dx + dy*dy) + dz*dz) as cKDTree computes
// them, and every sum in numpy's own order -- the row mean over the k sorted
// distances and the two global means use numpy's pairwise summation
// (8 accumulators per <=128-element leaf, halves rounded to multiples of 8),
// evaluated bottom-up over the same tree -- so the survivor set equals the
// reference's bit for bit (verified against numpy/scipy, tests/test_outlier_gpu.py).
#include "vx_internal.cuh"

#include <cmath>
#include <map>
#include <mutex>
#include <vector>

namespace vx {
namespace {

constexpr int kMaxK = 31;  // k + 1 <= 32 distances per point

__device__ __forceinline__ double dist3(const double *a, const double *b) {
    const double dx = __dsub_rn(a[0], b[0]), dy = __dsub_rn(a[1], b[1]), dz = __dsub_rn(a[2], b[2]);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// numpy pairwise_sum for n <= 128 (one leaf): 8 accumulators, then the rest
__device__ __forceinline__ double pw_leaf(const double *a, int n, int stride) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[(long long)i * stride]);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[(long long)j * stride];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[(long long)(i + j) * stride]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[(long long)i * stride]);
    return res;
}

struct Box {
    double lo[3];
    double h;        // cell edge
    int dim[3];
};

__global__ void k_cell_of(const double *__restrict__ pts, long long n, Box b, int *__restrict__ cell,
                          int *__restrict__ count) {
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth) {
        int c[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            int v = (int)floor((pts[3 * i + a] - b.lo[a]) / b.h);
            c[a] = min(max(v, 0), b.dim[a] - 1);
        }
        const int id = (c[0] * b.dim[1] + c[1]) * b.dim[2] + c[2];
        cell[i] = id;
        atomicAdd(&count[id], 1);
    }
}

// exclusive scan of count[0..m) into start[0..m] (single CTA, chunked)
__global__ void __launch_bounds__(1024) k_scan(const int *__restrict__ count, int m, int *__restrict__ start) {
    __shared__ int wsum[32];
    __shared__ int base_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    for (int c0 = 0; c0 < m; c0 += blockDim.x) {
        const int i = c0 + threadIdx.x;
        const int v = i < m ? count[i] : 0;
        int x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(VX_FULL_MASK, x, d);
            if (lane >= d) x += o;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        int wb = 0, tot = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
            if (q < warp) wb += wsum[q];
            tot += wsum[q];
        }
        const int base = base_s;
        if (i < m) start[i] = base + wb + x - v;
        __syncthreads();
        if (threadIdx.x == 0) base_s = base + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) start[m] = base_s;
}

__global__ void k_scatter_cells(const int *__restrict__ cell, long long n, const int *__restrict__ start,
                                int *__restrict__ fill, int *__restrict__ order) {
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth) {
        const int c = cell[i];
        order[start[c] + atomicAdd(&fill[c], 1)] = (int)i;
    }
}

// exact kNN: the K = k+1 smallest distances of point i to all points
// (itself included), then mean_knn = pairwise(sorted[1..k]) / k
template <int KM>
__global__ void __launch_bounds__(128) k_knn(const double *__restrict__ pts, long long n, Box b, int K,
                                             const int *__restrict__ start, const int *__restrict__ order,
                                             const int *__restrict__ cell, double *__restrict__ mean_knn) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    const int id = cell[i];
    const int cz = id % b.dim[2], cy = (id / b.dim[2]) % b.dim[1], cx = id / (b.dim[2] * b.dim[1]);
    const int c0[3] = {cx, cy, cz};
    double best[KM];
    int cnt = 0;
    // distance from p to the faces of its own cell (for the coverage bound)
    double face = 1e300;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double lo = b.lo[a] + c0[a] * b.h;
        face = fmin(face, fmin(p[a] - lo, lo + b.h - p[a]));
    }
    face = fmax(face, 0.0);
    const int rmax = max(b.dim[0], max(b.dim[1], b.dim[2]));
    for (int r = 0; r <= rmax; ++r) {
        // cells at Chebyshev distance exactly r from the home cell
        for (int dx = -r; dx <= r; ++dx) {
            const int x = c0[0] + dx;
            if (x < 0 || x >= b.dim[0]) continue;
            for (int dy = -r; dy <= r; ++dy) {
                const int y = c0[1] + dy;
                if (y < 0 || y >= b.dim[1]) continue;
                const bool edge = (dx == -r || dx == r || dy == -r || dy == r);
                for (int dz = -r; dz <= r; dz += (edge ? 1 : 2 * r > 0 ? 2 * r : 1)) {
                    const int z = c0[2] + dz;
                    if (z >= 0 && z < b.dim[2]) {
                        const int c = (x * b.dim[1] + y) * b.dim[2] + z;
                        for (int s = start[c]; s < start[c + 1]; ++s) {
                            const int j = order[s];
                            const double q[3] = {pts[3 * (long long)j], pts[3 * (long long)j + 1],
                                                 pts[3 * (long long)j + 2]};
                            const double d = dist3(p, q);
                            if (cnt < K) {
                                int t = cnt++;
                                while (t > 0 && best[t - 1] > d) { best[t] = best[t - 1]; --t; }
                                best[t] = d;
                            } else if (d < best[K - 1]) {
                                int t = K - 1;
                                while (t > 0 && best[t - 1] > d) { best[t] = best[t - 1]; --t; }
                                best[t] = d;
                            }
                        }
                    }
                    if (r == 0) break;
                }
            }
        }
        // every point outside the searched cube is farther than this
        // (with a relative margin so rounding can never admit an unseen point)
        const double covered = (face + (double)r * b.h) * (1.0 - 1e-12);
        if (cnt == K && best[K - 1] < covered) break;
    }
    // dists[:, 1:].mean(axis=1): numpy pairwise sum of the k sorted distances
    mean_knn[i] = __ddiv_rn(pw_leaf(best + 1, K - 1, 1), (double)(K - 1));
}

// numpy pairwise_sum over n doubles, bottom-up over the same tree: leaves
// (<= 128 elements) in parallel, then the internal nodes level by level.
struct PwTree {
    std::vector<int> leaf_start, leaf_len;    // leaves, left to right
    std::vector<int> node_l, node_r;          // internal nodes (ids >= nleaf), children ids
    std::vector<int> level_off;               // nodes grouped by height
    int root = 0;
};

int build_pw(PwTree &t, long long lo, long long n, std::vector<std::vector<int>> &levels,
             std::vector<int> &height, std::vector<int> &L, std::vector<int> &R) {
    if (n <= 128) {
        const int id = (int)t.leaf_start.size();
        t.leaf_start.push_back((int)lo);
        t.leaf_len.push_back((int)n);
        return -(id + 1);   // leaves encoded negative while building
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    const int a = build_pw(t, lo, n2, levels, height, L, R);
    const int b = build_pw(t, lo + n2, n - n2, levels, height, L, R);
    const int id = (int)L.size();
    L.push_back(a);
    R.push_back(b);
    const int ha = a < 0 ? 0 : height[a], hb = b < 0 ? 0 : height[b];
    height.push_back(std::max(ha, hb) + 1);
    return id;
}

__global__ void k_pw_leaves(const double *__restrict__ x, const double *__restrict__ sub, int square,
                            const int *__restrict__ ls, const int *__restrict__ ll, int nleaf,
                            double *__restrict__ val, double *__restrict__ tmp) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nleaf) return;
    const double *a = x + ls[l];
    if (square) {   // (x - mean)^2 as numpy's x = arr - mean; x = x * x
        double *t = tmp + ls[l];
        const double m = *sub;
        for (int q = 0; q < ll[l]; ++q) {
            const double d = __dsub_rn(a[q], m);
            t[q] = __dmul_rn(d, d);
        }
        a = t;
    }
    val[l] = pw_leaf(a, ll[l], 1);
}

// one CTA: internal nodes by height; node values after the nleaf leaf values
__global__ void __launch_bounds__(1024) k_pw_tree(double *__restrict__ val, int nleaf, const int *__restrict__ nl,
                                                  const int *__restrict__ nr, const int *__restrict__ loff,
                                                  int nlevels, long long n, double *__restrict__ out_mean) {
    for (int h = 0; h < nlevels; ++h) {
        for (int q = loff[h] + threadIdx.x; q < loff[h + 1]; q += blockDim.x) {
            const int a = nl[q], b = nr[q];
            val[nleaf + q] = __dadd_rn(val[a], val[b]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int root = nlevels ? nleaf + loff[nlevels] - 1 : 0;
        *out_mean = __ddiv_rn(val[root], (double)n);
    }
}

__global__ void k_keep(const double *__restrict__ mk, long long n, const double *__restrict__ stats, double m,
                       uint8_t *__restrict__ keep, unsigned long long *__restrict__ removed) {
    // cutoff = mean + m * std   (two numpy float64 scalar ops)
    const double cutoff = __dadd_rn(stats[0], __dmul_rn(m, __dsqrt_rn(stats[1])));
    const long long nth = (long long)gridDim.x * blockDim.x;
    unsigned long long rem = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth) {
        const bool k = mk[i] <= cutoff;
        keep[i] = k ? 1 : 0;
        rem += k ? 0 : 1;
    }
    for (int d = 16; d > 0; d >>= 1) rem += __shfl_down_sync(VX_FULL_MASK, rem, d);
    if ((threadIdx.x & 31) == 0 && rem) atomicAdd(removed, rem);
}

}  // namespace

struct PwPlan {
    int nleaf = 0, nnode = 0, nlevels = 0;
    int *d = nullptr;   // [ls nleaf][ll nleaf][nl nnode][nr nnode][loff nlevels+1]
};

// pairwise-tree plans cached per n (topology depends only on n)
static PwPlan pw_plan(long long n) {
    static std::mutex mu;
    static std::map<std::pair<long long, int>, PwPlan> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({n, dev});
    if (it != cache.end()) return it->second;
    PwTree t;
    std::vector<std::vector<int>> levels;
    std::vector<int> height, L, R;
    build_pw(t, 0, n, levels, height, L, R);
    const int nleaf = (int)t.leaf_start.size(), nnode = (int)L.size();
    int maxh = 0;
    for (int h : height) maxh = std::max(maxh, h);
    // order internal nodes by height; children ids: leaves 0..nleaf-1, nodes nleaf+pos
    std::vector<int> pos(nnode), loff(maxh + 1, 0);
    std::vector<std::vector<int>> byh(maxh + 1);
    for (int q = 0; q < nnode; ++q) byh[height[q] - 1 + 1 - 1].push_back(q);
    int p = 0;
    for (int h = 0; h < maxh; ++h) {
        loff[h] = p;
        for (int q : byh[h]) pos[q] = p++;
    }
    loff[maxh] = p;
    std::vector<int> host;
    host.insert(host.end(), t.leaf_start.begin(), t.leaf_start.end());
    host.insert(host.end(), t.leaf_len.begin(), t.leaf_len.end());
    auto child = [&](int c) { return c < 0 ? (-c - 1) : nleaf + pos[c]; };
    std::vector<int> nl(nnode), nr(nnode);
    for (int q = 0; q < nnode; ++q) {
        nl[pos[q]] = child(L[q]);
        nr[pos[q]] = child(R[q]);
    }
    host.insert(host.end(), nl.begin(), nl.end());
    host.insert(host.end(), nr.begin(), nr.end());
    host.insert(host.end(), loff.begin(), loff.end());
    PwPlan plan;
    plan.nleaf = nleaf;
    plan.nnode = nnode;
    plan.nlevels = maxh;
    if (cudaMalloc(&plan.d, host.size() * sizeof(int)) != cudaSuccess) return PwPlan{};
    cudaMemcpy(plan.d, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice);
    cache[{n, dev}] = plan;
    return plan;
}

constexpr int kMaxCellDim = 128;

size_t outlier_scratch_bytes(long long n) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const long long ncell = (long long)kMaxCellDim * kMaxCellDim * kMaxCellDim;
    return al(n * 4) * 2 + al((ncell + 1) * 4) * 3 + al(n * 8) * 2 + al((n / 32 + 64) * 2 * 8) + 256;
}

// per-block min/max of the cloud (the caller folds the <=148 partials)
__global__ void k_bounds(const double *__restrict__ pts, long long n, double *__restrict__ part) {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    const long long nth = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = fmin(lo[a], pts[3 * i + a]);
            hi[a] = fmax(hi[a], pts[3 * i + a]);
        }
#pragma unroll
    for (int a = 0; a < 3; ++a)
        for (int d = 16; d > 0; d >>= 1) {
            lo[a] = fmin(lo[a], __shfl_down_sync(VX_FULL_MASK, lo[a], d));
            hi[a] = fmax(hi[a], __shfl_down_sync(VX_FULL_MASK, hi[a], d));
        }
    __shared__ double sm[32][6];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; ++a) { sm[w][a] = lo[a]; sm[w][3 + a] = hi[a]; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
            for (int a = 0; a < 3; ++a) {
                sm[0][a] = fmin(sm[0][a], sm[q][a]);
                sm[0][3 + a] = fmax(sm[0][3 + a], sm[q][3 + a]);
            }
        for (int a = 0; a < 6; ++a) part[6 * blockIdx.x + a] = sm[0][a];
    }
}

cudaError_t cloud_bounds(const double *pts, long long n, double lo[3], double hi[3], void *scratch,
                         cudaStream_t st) {
    const int nb = 148;
    double *part = static_cast<double *>(scratch);
    k_bounds<<<nb, 256, 0, st>>>(pts, n, part);
    double h[nb * 6];
    cudaError_t e = cudaMemcpyAsync(h, part, sizeof h, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    for (int a = 0; a < 3; ++a) { lo[a] = 1e300; hi[a] = -1e300; }
    for (int b = 0; b < nb; ++b)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], h[6 * b + a]);
            hi[a] = std::max(hi[a], h[6 * b + 3 + a]);
        }
    return cudaSuccess;
}

cudaError_t outlier_filter(const double *pts, long long n, int k, double stdm, const double lo[3],
                           const double hi[3], uint8_t *keep, unsigned long long *removed, void *scratch,
                           size_t scratch_bytes, cudaStream_t st) {
    if (k < 1 || k > kMaxK) return cudaErrorInvalidValue;
    // cell edge: ~4 points per cell if the cloud filled its bounding box
    double ext[3], vol = 1.0;
    for (int a = 0; a < 3; ++a) {
        ext[a] = hi[a] - lo[a];
        vol *= std::max(ext[a], 1e-9);
    }
    double h = std::cbrt(vol / std::max(1.0, n / 4.0));
    const double emax = std::max(ext[0], std::max(ext[1], ext[2]));
    h = std::max(h, emax / (kMaxCellDim - 1));   // <= kMaxCellDim^3 cells
    if (!(h > 0.0)) h = 1.0;
    Box b;
    long long ncell = 1;
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = lo[a];
        b.dim[a] = std::max(1, std::min(kMaxCellDim, (int)std::floor(ext[a] / h) + 1));
        ncell *= b.dim[a];
    }
    b.h = h;
    if (outlier_scratch_bytes(n) > scratch_bytes) return cudaErrorInvalidValue;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    unsigned char *p = static_cast<unsigned char *>(scratch);
    int *cell = (int *)p; p += al(n * 4);
    int *order = (int *)p; p += al(n * 4);
    int *count = (int *)p; p += al((ncell + 1) * 4);
    int *start = (int *)p; p += al((ncell + 1) * 4);
    int *fill = (int *)p; p += al((ncell + 1) * 4);
    double *mk = (double *)p; p += al(n * 8);
    double *tmp = (double *)p; p += al(n * 8);
    double *val = (double *)p;
    cudaError_t e = cudaMemsetAsync(count, 0, (ncell + 1) * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(fill, 0, (ncell + 1) * 4, st);
    if (e != cudaSuccess) return e;
    const unsigned g = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
    k_cell_of<<<g, 256, 0, st>>>(pts, n, b, cell, count);
    k_scan<<<1, 1024, 0, st>>>(count, (int)ncell, start);
    k_scatter_cells<<<g, 256, 0, st>>>(cell, n, start, fill, order);
    const unsigned gk = (unsigned)((n + 127) / 128);
    if (k + 1 <= 16) k_knn<16><<<gk, 128, 0, st>>>(pts, n, b, k + 1, start, order, cell, mk);
    else k_knn<32><<<gk, 128, 0, st>>>(pts, n, b, k + 1, start, order, cell, mk);
    // global mean and variance in numpy's pairwise order
    const PwPlan plan = pw_plan(n);
    if (!plan.d) return cudaErrorMemoryAllocation;
    const int *ls = plan.d, *ll = plan.d + plan.nleaf, *nl = plan.d + 2 * plan.nleaf;
    const int *nr = nl + plan.nnode, *loff = nr + plan.nnode;
    double *stats = val + plan.nleaf + plan.nnode + 8;   // [mean, var]
    const unsigned gl = (unsigned)((plan.nleaf + 127) / 128);
    k_pw_leaves<<<gl, 128, 0, st>>>(mk, nullptr, 0, ls, ll, plan.nleaf, val, tmp);
    k_pw_tree<<<1, 1024, 0, st>>>(val, plan.nleaf, nl, nr, loff, plan.nlevels, n, stats);
    k_pw_leaves<<<gl, 128, 0, st>>>(mk, stats, 1, ls, ll, plan.nleaf, val, tmp);
    k_pw_tree<<<1, 1024, 0, st>>>(val, plan.nleaf, nl, nr, loff, plan.nlevels, n, stats + 1);
    k_keep<<<g, 256, 0, st>>>(mk, n, stats, stdm, keep, removed);
    return cudaGetLastError();
}

}  // namespace vx
