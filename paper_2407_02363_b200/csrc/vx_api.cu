// C-ABI layer of libvx.so (include/vx.h): contexts, device-resident grids and
// fields, host<->device staging, the camera-tick pipeline.  No CPU compute
// path exists here: every numeric result comes from the sm_100a kernels in
// vx_edt.cu / vx_map.cu / vx_query.cu.
#include "vx.h"
#include "vx_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace vx;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(e == cudaErrorMemoryAllocation ? VX_ENOMEM : VX_ECUDA, "%s: %s (%s)", what,
                cudaGetErrorString(e), cudaGetErrorName(e));
}

#define VX_CUDA(call)                                   \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

// growable device buffer
struct DevBuf {
    void *p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= n) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        size_t want = bytes + bytes / 8 + 256;
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) n = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

inline double logit(double p) { return std::log(p / (1.0 - p)); }  // grids.py:24-25

constexpr float kLMin = -2.0f, kLMax = 3.5f;
constexpr float kOccThr = 0.0f;  // float32(logit(0.5)): the cached occupancy threshold

}  // namespace

struct vx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    DevBuf scratch, staging, staging2, temp, outl, exp, exp_out;
    DevBuf slabhdr;   // slab mode: the windowed search's header (pass-1 counts, fall-backs)
    long long launches = 0;
    long long h2d = 0, d2h = 0;   // bytes moved by the ABI's own copies (vx_ctx_transfer_bytes)
};

struct vx_grid {
    vx_ctx *ctx = nullptr;
    GridGeom g{};
    long long n = 0;
    float *cells = nullptr;
    uint8_t *occ = nullptr;         // cells > 0 (threshold 0.5), kept in sync by the kernels
    uint32_t *counts = nullptr;     // bincount scratch, all zero between inserts
    int32_t *touched = nullptr;     // voxels written since the last clear (may repeat)
    DevCounters *ctr = nullptr;
    unsigned long long *set_oob = nullptr;
    int set_oob_cap = 0;
    int capacity = 0;
    bool sparse_ok = true;          // touched list covers every non-zero cell
    bool maybe_oor = false;         // host wrote cells outside [L_MIN, L_MAX] or NaN
    bool fresh = false;             // every cell is +0.0f (reset, nothing written since):
                                    // an insert may count hits in the cells themselves
};

struct vx_field {
    vx_ctx *ctx = nullptr;
    int nx = 0, ny = 0, nz = 0;
    int32_t *site = nullptr;
    bool owned = true;
};

// ----------------------------------------------------------------------------
extern "C" int vx_abi_version(void) { return VX_ABI_VERSION; }
extern "C" const char *vx_last_error(void) { return g_err.c_str(); }

extern "C" int vx_ctx_create(int device, vx_ctx **out) {
    if (!out) return fail(VX_EINVAL, "out is NULL");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(VX_ENODEV, "no CUDA device available (%s); libvx has no CPU fallback",
                    e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(VX_EINVAL, "device %d out of range", device);
    VX_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    VX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(VX_ENODEV, "device %d is sm_%d%d; libvx is built for sm_100a", device, prop.major,
                    prop.minor);
    vx_ctx *c = new vx_ctx;
    c->device = device;
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate");
    }
    *out = c;
    return VX_OK;
}

extern "C" int vx_ctx_destroy(vx_ctx *c) {
    if (!c) return VX_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->scratch.release();
    c->staging.release();
    c->staging2.release();
    c->temp.release();
    c->exp.release();
    c->exp_out.release();
    c->outl.release();
    c->slabhdr.release();
    cudaStreamDestroy(c->stream);
    delete c;
    return VX_OK;
}

extern "C" int vx_ctx_stream(vx_ctx *c, void **s) {
    if (!c || !s) return fail(VX_EINVAL, "NULL argument");
    *s = (void *)c->stream;
    return VX_OK;
}

extern "C" int vx_ctx_synchronize(vx_ctx *c) {
    if (!c) return fail(VX_EINVAL, "NULL ctx");
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

extern "C" int64_t vx_ctx_launches(const vx_ctx *c) { return c ? c->launches : 0; }

extern "C" int vx_host_alloc(size_t bytes, void **out) {
    if (!out) return fail(VX_EINVAL, "NULL out");
    VX_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
    return VX_OK;
}

extern "C" int vx_host_free(void *p) {
    if (p) VX_CUDA(cudaFreeHost(p));
    return VX_OK;
}

// ---- grids ------------------------------------------------------------------
static int check_geom(int nx, int ny, int nz, double vs) {
    if (nx <= 0 || ny <= 0 || nz <= 0)
        return fail(VX_EINVAL, "dims must be three positive integers, got (%d, %d, %d)", nx, ny, nz);
    if (!(vs > 0.0)) return fail(VX_EINVAL, "voxel_size must be > 0");
    if ((long long)nx * ny * nz >= (1LL << 31))
        return fail(VX_EINVAL, "grid too large for 32-bit voxel addressing");
    return VX_OK;
}

extern "C" int vx_grid_create(vx_ctx *ctx, int nx, int ny, int nz, double vs, const double origin[3],
                              vx_grid **out) {
    if (!ctx || !out) return fail(VX_EINVAL, "NULL argument");
    int rc = check_geom(nx, ny, nz, vs);
    if (rc) return rc;
    VX_CUDA(cudaSetDevice(ctx->device));
    vx_grid *g = new vx_grid;
    g->ctx = ctx;
    g->g = GridGeom{nx, ny, nz, vs, origin ? origin[0] : 0.0, origin ? origin[1] : 0.0,
                    origin ? origin[2] : 0.0};
    g->n = (long long)nx * ny * nz;
    g->capacity = (int)g->n;
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&g->cells, g->n * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&g->occ, (g->n + 15) & ~15LL);
    if (e == cudaSuccess) e = cudaMalloc(&g->counts, g->n * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&g->touched, g->n * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&g->ctr, sizeof(DevCounters));
    if (e == cudaSuccess) e = cudaMemsetAsync(g->cells, 0, g->n * sizeof(float), ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(g->occ, 0, (g->n + 15) & ~15LL, ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(g->counts, 0, g->n * sizeof(uint32_t), ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(g->ctr, 0, sizeof(DevCounters), ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        vx_grid_destroy(g);
        return cuda_fail(e, "vx_grid_create");
    }
    *out = g;
    return VX_OK;
}

extern "C" int vx_grid_destroy(vx_grid *g) {
    if (!g) return VX_OK;
    if (g->ctx) cudaStreamSynchronize(g->ctx->stream);
    cudaFree(g->cells);
    cudaFree(g->occ);
    cudaFree(g->counts);
    cudaFree(g->touched);
    cudaFree(g->ctr);
    cudaFree(g->set_oob);
    delete g;
    return VX_OK;
}

static int grid_clear_async(vx_grid *g) {
    cudaError_t e = launch_reset(g->cells, g->occ, g->touched, g->ctr, g->n, g->capacity,
                                 !g->sparse_ok, g->ctx->stream);
    g->ctx->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "reset");
    g->sparse_ok = true;
    g->maybe_oor = false;
    g->fresh = true;
    return VX_OK;
}

extern "C" int vx_grid_clear(vx_grid *g) {
    if (!g) return fail(VX_EINVAL, "NULL grid");
    return grid_clear_async(g);
}

static bool same_geometry(const vx_grid *a, const vx_grid *b) {  // grids.py:214-217
    return a->g.nx == b->g.nx && a->g.ny == b->g.ny && a->g.nz == b->g.nz && a->g.vs == b->g.vs &&
           a->g.ox == b->g.ox && a->g.oy == b->g.oy && a->g.oz == b->g.oz;
}

// sflag (optional, zeroed by the caller): on a fresh grid the finalize also
// flags the occupied i-slices for the EDT; *flags_done says whether it did
static int insert_device(vx_grid *g, const double *d_xyz, long long n, const long long *n_dev,
                         float hit, double thr, const vx_grid *mask, const uint8_t *keep = nullptr,
                         uint8_t *sflag = nullptr, bool *flags_done = nullptr, bool stats_zeroed = false,
                         const SparseRows *list = nullptr) {
    if (mask && !same_geometry(g, mask))
        return fail(VX_EINVAL, "robot_mask geometry does not match this grid");
    cudaStream_t st = g->ctx->stream;
    if (!stats_zeroed) VX_CUDA(cudaMemsetAsync(g->ctr, 0, 3 * sizeof(unsigned long long), st));
    const float thr32 = (float)logit(thr);  // numpy compares in float32
    // a fresh grid counts hits in its own (zero) cells: finalize then reads one
    // array per touched voxel instead of two and has no counts to clear
    // (not when the grid is its own robot mask: the scatter would read the
    // partly incremented counts as mask cells, grids.py:178-182 reads the
    // pre-insert cells)
    const bool fresh = g->fresh && !g->maybe_oor && mask != g;
    uint32_t *counts = fresh ? reinterpret_cast<uint32_t *>(g->cells) : g->counts;
    g->fresh = false;
    cudaError_t e = launch_scatter(d_xyz, n, (const int64_t *)n_dev, g->g, mask ? mask->cells : nullptr,
                                   thr32, counts, g->touched, g->ctr, g->capacity, st, keep);
    if (e != cudaSuccess) return cuda_fail(e, "scatter");
    g->ctx->launches += 1;
    if (g->maybe_oor) {
        e = launch_dense_clip(g->cells, g->counts, g->n, g->ctr, st);
        if (e != cudaSuccess) return cuda_fail(e, "dense_clip");
        g->ctx->launches += 1;
    }
    uint8_t *fl = fresh ? sflag : nullptr;
    // list (with the flags): finalize's last block also builds the occupied-slice list
    e = launch_finalize(g->cells, g->occ, counts, g->touched, g->ctr, g->n, g->capacity,
                        n > 0 ? n : 1, hit, kOccThr, st, fresh, fl, (long long)g->g.ny * g->g.nz, g->g.nx,
                        list ? const_cast<int *>(list->xs) : nullptr, list ? const_cast<int *>(list->hdr) : nullptr,
                        list ? list->m_mirror : nullptr);
    if (flags_done) *flags_done = fl != nullptr;
    if (e != cudaSuccess) return cuda_fail(e, "finalize");
    g->ctx->launches += 1;
    return VX_OK;
}

extern "C" int vx_grid_last_stats(vx_grid *g, vx_insert_stats *stats) {
    if (!g || !stats) return fail(VX_EINVAL, "NULL argument");
    DevCounters h;
    VX_CUDA(cudaMemcpyAsync(&h, g->ctr, sizeof h, cudaMemcpyDeviceToHost, g->ctx->stream));
    VX_CUDA(cudaStreamSynchronize(g->ctx->stream));
    stats->inserted = (int64_t)h.inserted;
    stats->outliers_removed = 0;
    stats->robot_skipped = (int64_t)h.skipped;
    stats->out_of_bounds = (int64_t)h.oob;
    return VX_OK;
}

extern "C" int vx_grid_insert_points_device(vx_grid *g, const double *d_xyz, int64_t n, float hit,
                                            double thr, const vx_grid *mask) {
    if (!g || (n > 0 && !d_xyz)) return fail(VX_EINVAL, "NULL argument");
    if (n < 0) return fail(VX_EINVAL, "negative point count");
    return insert_device(g, d_xyz, n, nullptr, hit, thr, mask);
}

extern "C" int vx_grid_insert_points(vx_grid *g, const double *xyz, int64_t n, float hit, double thr,
                                     const vx_grid *mask, vx_insert_stats *stats) {
    if (!g || (n > 0 && !xyz)) return fail(VX_EINVAL, "NULL argument");
    if (n < 0) return fail(VX_EINVAL, "negative point count");
    if (mask && !same_geometry(g, mask))
        return fail(VX_EINVAL, "robot_mask geometry does not match this grid");
    if (n == 0) {  // grids.py:163-164
        if (stats) *stats = vx_insert_stats{0, 0, 0, 0};
        return VX_OK;
    }
    vx_ctx *c = g->ctx;
    VX_CUDA(c->staging.ensure((size_t)n * 3 * sizeof(double)));
    VX_CUDA(cudaMemcpyAsync(c->staging.p, xyz, (size_t)n * 3 * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
    c->h2d += (long long)n * 24;
    int rc = insert_device(g, (const double *)c->staging.p, n, nullptr, hit, thr, mask);
    if (rc) return rc;
    vx_insert_stats s;
    rc = vx_grid_last_stats(g, &s);
    if (rc) return rc;
    if (s.inserted > 0) g->maybe_oor = false;  // the dense clip ran
    if (stats) *stats = s;
    return VX_OK;
}

// statistical_outlier_filter (grids.py:224-240) on device points: keep mask
// into outl scratch, removed count into *removed_host (syncs)
static int outlier_device(vx_ctx *c, const double *d_xyz, long long n, int k, double stdm, uint8_t **keep_out,
                          long long *removed_host) {
    if (k > 31) return fail(VX_EINVAL, "k_neighbors > 31 is not supported on the GPU");
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t need = al(n) + 256 + outlier_scratch_bytes(n) + 148 * 6 * 8 + 256;
    VX_CUDA(c->outl.ensure(need));
    unsigned char *p = (unsigned char *)c->outl.p;
    uint8_t *keep = p;
    unsigned long long *removed = (unsigned long long *)(p + al(n));
    void *scr = p + al(n) + 256;
    double lo[3], hi[3];
    VX_CUDA(cloud_bounds(d_xyz, n, lo, hi, (unsigned char *)scr + outlier_scratch_bytes(n), c->stream));
    VX_CUDA(cudaMemsetAsync(removed, 0, sizeof(unsigned long long), c->stream));
    cudaError_t e = outlier_filter(d_xyz, n, k, stdm, lo, hi, keep, removed, scr, outlier_scratch_bytes(n),
                                   c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "outlier_filter");
    c->launches += 9;
    unsigned long long rem = 0;
    VX_CUDA(cudaMemcpyAsync(&rem, removed, sizeof rem, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    *keep_out = keep;
    *removed_host = (long long)rem;
    return VX_OK;
}

extern "C" int vx_outlier_mask(vx_ctx *c, const double *xyz, int64_t n, int k_neighbors, double std_multiplier,
                               uint8_t *keep_host, int64_t *removed) {
    if (!c || (n > 0 && (!xyz || !keep_host))) return fail(VX_EINVAL, "NULL argument");
    if (k_neighbors < 0) return fail(VX_EINVAL, "k_neighbors must be >= 0");
    if (!(std_multiplier > 0.0)) return fail(VX_EINVAL, "std_multiplier must be > 0");
    if (n <= k_neighbors || n == 0 || k_neighbors == 0) {   // grids.py:233-234: pass through
        if (n > 0) std::memset(keep_host, 1, (size_t)n);
        if (removed) *removed = 0;
        return VX_OK;
    }
    VX_CUDA(c->staging.ensure((size_t)n * 24));
    VX_CUDA(cudaMemcpyAsync(c->staging.p, xyz, (size_t)n * 24, cudaMemcpyHostToDevice, c->stream));
    uint8_t *keep = nullptr;
    long long rem = 0;
    int rc = outlier_device(c, (const double *)c->staging.p, n, k_neighbors, std_multiplier, &keep, &rem);
    if (rc) return rc;
    VX_CUDA(cudaMemcpyAsync(keep_host, keep, (size_t)n, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    if (removed) *removed = rem;
    return VX_OK;
}

extern "C" int vx_grid_insert_points_ex(vx_grid *g, const double *xyz, int64_t n, float hit, double thr,
                                        const vx_grid *mask, int k_neighbors, double std_multiplier,
                                        vx_insert_stats *stats) {
    if (!g || (n > 0 && !xyz)) return fail(VX_EINVAL, "NULL argument");
    if (k_neighbors < 0) return fail(VX_EINVAL, "k_neighbors must be >= 0");
    if (!(std_multiplier > 0.0)) return fail(VX_EINVAL, "std_multiplier must be > 0");
    if (k_neighbors == 0 || n <= k_neighbors)
        return vx_grid_insert_points(g, xyz, n, hit, thr, mask, stats);
    if (mask && !same_geometry(g, mask))
        return fail(VX_EINVAL, "robot_mask geometry does not match this grid");
    vx_ctx *c = g->ctx;
    VX_CUDA(c->staging.ensure((size_t)n * 24));
    VX_CUDA(cudaMemcpyAsync(c->staging.p, xyz, (size_t)n * 24, cudaMemcpyHostToDevice, c->stream));
    c->h2d += (long long)n * 24;
    uint8_t *keep = nullptr;
    long long rem = 0;
    int rc = outlier_device(c, (const double *)c->staging.p, n, k_neighbors, std_multiplier, &keep, &rem);
    if (rc) return rc;
    rc = insert_device(g, (const double *)c->staging.p, n, nullptr, hit, thr, mask, keep);
    if (rc) return rc;
    vx_insert_stats s;
    rc = vx_grid_last_stats(g, &s);
    if (rc) return rc;
    s.outliers_removed = rem;
    if (s.inserted > 0) g->maybe_oor = false;
    if (stats) *stats = s;
    return VX_OK;
}

static int ensure_set_oob(vx_grid *g, int nsets) {
    if (g->set_oob_cap < nsets) {
        cudaFree(g->set_oob);
        g->set_oob = nullptr;
        VX_CUDA(cudaMalloc(&g->set_oob, sizeof(unsigned long long) * nsets));
        g->set_oob_cap = nsets;
    }
    return VX_OK;
}

// oob_zeroed: the per-set OOB counters were already cleared (camera tick)
static int stamp_sets(vx_grid *g, int nsets, const int32_t *d_ijk, const int64_t *d_offsets,
                      const double *d_origins, const double *d_vs, const double *d_T, float value,
                      int64_t total, bool oob_zeroed = false) {
    vx_ctx *c = g->ctx;
    g->fresh = false;   // stamped cells are no longer +0.0f
    int rc = ensure_set_oob(g, nsets);
    if (rc) return rc;
    if (!oob_zeroed) VX_CUDA(cudaMemsetAsync(g->set_oob, 0, sizeof(unsigned long long) * nsets, c->stream));
    cudaError_t e = launch_stamp(d_ijk, d_offsets, nsets, d_origins, d_vs, d_T, g->g, g->cells, g->occ,
                                 value, kOccThr, g->touched, g->ctr, g->set_oob, g->capacity, total,
                                 c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "stamp");
    c->launches += 1;
    return VX_OK;
}

extern "C" int vx_grid_insert_voxel_sets(vx_grid *g, int nsets, const int32_t *const *ijk,
                                         const int64_t *counts, const double *set_origins,
                                         const double *set_vs, const double *T, float value,
                                         int64_t *oob_out) {
    if (!g || nsets < 0 || (nsets && (!ijk || !counts || !set_origins || !set_vs)))
        return fail(VX_EINVAL, "NULL argument");
    if (nsets == 0) return VX_OK;
    vx_ctx *c = g->ctx;
    std::vector<int64_t> off(nsets + 1, 0);
    for (int s = 0; s < nsets; ++s) {
        if (counts[s] < 0) return fail(VX_EINVAL, "negative voxel count");
        if (!(set_vs[s] > 0.0)) return fail(VX_EINVAL, "voxel_size must be > 0");
        off[s + 1] = off[s] + counts[s];
    }
    const int64_t total = off[nsets];
    // one staging block: ijk | offsets | origins | vs | T
    const size_t b_ijk = ((size_t)total * 3 * sizeof(int32_t) + 15) & ~(size_t)15;
    const size_t b_off = (sizeof(int64_t) * (nsets + 1) + 15) & ~(size_t)15;
    const size_t b_org = sizeof(double) * 3 * nsets, b_vs = sizeof(double) * nsets;
    const size_t b_T = T ? sizeof(double) * 16 * nsets : 0;
    std::vector<unsigned char> host(b_ijk + b_off + b_org + b_vs + b_T);
    size_t pos = 0;
    for (int s = 0; s < nsets; ++s) {
        if (counts[s]) std::memcpy(host.data() + pos, ijk[s], counts[s] * 3 * sizeof(int32_t));
        pos += counts[s] * 3 * sizeof(int32_t);
    }
    std::memcpy(host.data() + b_ijk, off.data(), sizeof(int64_t) * (nsets + 1));
    std::memcpy(host.data() + b_ijk + b_off, set_origins, b_org);
    std::memcpy(host.data() + b_ijk + b_off + b_org, set_vs, b_vs);
    if (T) std::memcpy(host.data() + b_ijk + b_off + b_org + b_vs, T, b_T);
    VX_CUDA(c->staging2.ensure(host.size()));
    unsigned char *d = (unsigned char *)c->staging2.p;
    VX_CUDA(cudaMemcpyAsync(d, host.data(), host.size(), cudaMemcpyHostToDevice, c->stream));
    c->h2d += (long long)host.size();
    int rc = stamp_sets(g, nsets, (const int32_t *)d, (const int64_t *)(d + b_ijk),
                        (const double *)(d + b_ijk + b_off), (const double *)(d + b_ijk + b_off + b_org),
                        T ? (const double *)(d + b_ijk + b_off + b_org + b_vs) : nullptr, value, total);
    if (rc) return rc;
    std::vector<unsigned long long> oob(nsets);
    VX_CUDA(cudaMemcpyAsync(oob.data(), g->set_oob, sizeof(unsigned long long) * nsets,
                            cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    if (oob_out)
        for (int s = 0; s < nsets; ++s) oob_out[s] = (int64_t)oob[s];
    return VX_OK;
}

extern "C" int vx_grid_read_cells(vx_grid *g, float *out) {
    if (!g || !out) return fail(VX_EINVAL, "NULL argument");
    VX_CUDA(cudaMemcpyAsync(out, g->cells, g->n * sizeof(float), cudaMemcpyDeviceToHost, g->ctx->stream));
    g->ctx->d2h += g->n * 4;
    VX_CUDA(cudaStreamSynchronize(g->ctx->stream));
    return VX_OK;
}

extern "C" int vx_grid_write_cells(vx_grid *g, const float *in) {
    if (!g || !in) return fail(VX_EINVAL, "NULL argument");
    // cells an insert's dense clip would change outside the touched voxels
    // (grids.py:187 clips every voxel: out of range, NaN, and -0.0 -> +0.0)
    bool oor = false;
    for (long long v = 0; v < g->n && !oor; ++v)
        oor = !(in[v] >= kLMin && in[v] <= kLMax) || (in[v] == 0.0f && std::signbit(in[v]));
    VX_CUDA(cudaMemcpyAsync(g->cells, in, g->n * sizeof(float), cudaMemcpyHostToDevice, g->ctx->stream));
    g->ctx->h2d += g->n * 4;
    cudaError_t e = launch_occupancy(g->cells, g->occ, g->n, kOccThr, g->ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    g->ctx->launches += 1;
    g->sparse_ok = false;  // non-zero cells are no longer all on the touched list
    g->fresh = false;
    g->maybe_oor = g->maybe_oor || oor;
    VX_CUDA(cudaStreamSynchronize(g->ctx->stream));
    return VX_OK;
}

// device occupancy at `thr` (cached array when thr is the 0.5 default)
static int grid_occ_device(vx_grid *g, double thr, const uint8_t **out) {
    const float thr32 = (float)logit(thr);
    if (thr32 == kOccThr) {
        *out = g->occ;
        return VX_OK;
    }
    vx_ctx *c = g->ctx;
    VX_CUDA(c->temp.ensure(g->n));
    cudaError_t e = launch_occupancy(g->cells, (uint8_t *)c->temp.p, g->n, thr32, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy");
    c->launches += 1;
    *out = (const uint8_t *)c->temp.p;
    return VX_OK;
}

extern "C" int vx_grid_occupancy(vx_grid *g, double thr, uint8_t *out) {
    if (!g || !out) return fail(VX_EINVAL, "NULL argument");
    const uint8_t *d = nullptr;
    int rc = grid_occ_device(g, thr, &d);
    if (rc) return rc;
    VX_CUDA(cudaMemcpyAsync(out, d, g->n, cudaMemcpyDeviceToHost, g->ctx->stream));
    g->ctx->d2h += g->n;
    VX_CUDA(cudaStreamSynchronize(g->ctx->stream));
    return VX_OK;
}

// grids.py:210-212: np.argwhere(occupancy_mask) -- (K,3) int64, flat-index
// order.  host_out == NULL (or too small): *count only (VX_ERANGE if short).
extern "C" int vx_grid_occupied_voxels(vx_grid *g, double thr, int64_t *host_out, int64_t capacity,
                                       int64_t *count) {
    if (!g || !count) return fail(VX_EINVAL, "NULL argument");
    vx_ctx *c = g->ctx;
    const uint8_t *d = nullptr;
    int rc = grid_occ_device(g, thr, &d);
    if (rc) return rc;
    VX_CUDA(c->exp.ensure(occ_scratch_bytes(g->n)));
    cudaError_t e = launch_occ_layout(d, g->n, c->exp.p, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "occupied_voxels");
    c->launches += 2;
    long long total = 0;
    VX_CUDA(cudaMemcpyAsync(&total, occ_total_ptr(c->exp.p, g->n), 8, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    *count = total;
    if (!host_out) return VX_OK;
    if (capacity < total) return fail(VX_ERANGE, "capacity %lld < %lld occupied voxels", (long long)capacity, total);
    if (!total) return VX_OK;
    VX_CUDA(c->exp_out.ensure((size_t)total * 24));
    e = launch_occ_write(d, g->n, g->g.ny, g->g.nz, c->exp.p, (long long *)c->exp_out.p, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "occupied_voxels");
    c->launches += 1;
    VX_CUDA(cudaMemcpyAsync(host_out, c->exp_out.p, (size_t)total * 24, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

// ---- EDT ----------------------------------------------------------------------
static int check_edt_dims(int nx, int ny, int nz) {
    if (nx <= 0 || ny <= 0 || nz <= 0) return fail(VX_EINVAL, "occupancy must be a non-empty 3D array");
    if (nx > (1 << 20) || ny > (1 << 20) || nz > (1 << 20))   // edt.py:29, 459-460
        return fail(VX_EINVAL, "grid extent too large for integer-exact transform");
    if ((long long)nx * ny * nz >= (1LL << 31))
        return fail(VX_EINVAL, "grid too large for 32-bit site indices");
    return VX_OK;
}

static int field_new(vx_ctx *c, int nx, int ny, int nz, vx_field **out) {
    vx_field *f = new vx_field;
    f->ctx = c;
    f->nx = nx; f->ny = ny; f->nz = nz;
    cudaError_t e = cudaMalloc(&f->site, (size_t)nx * ny * nz * sizeof(int32_t));
    if (e != cudaSuccess) {
        delete f;
        return cuda_fail(e, "cudaMalloc(site)");
    }
    *out = f;
    return VX_OK;
}

static int edt_run(vx_ctx *c, const uint8_t *d_occ, int nx, int ny, int nz, int nscenes, int32_t *d_site,
                   void *scratch, size_t scratch_bytes) {
    EdtPlan p;
    if (!make_plan(nx, ny, nz, &p, 0)) return fail(VX_EINVAL, "bad EDT shape");
    const size_t need = scratch_bytes_for(p, nscenes);
    if (!scratch) {
        VX_CUDA(c->scratch.ensure(need));
        scratch = c->scratch.p;
    } else if (scratch_bytes < need) {
        return fail(VX_EINVAL, "EDT scratch too small: %zu < %zu", scratch_bytes, need);
    }
    cudaError_t e = edt_device_batched(d_occ, d_site, scratch, p, nscenes, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "edt");
    c->launches += 3;
    return VX_OK;
}

extern "C" size_t vx_edt_scratch_bytes(int nx, int ny, int nz, int nscenes) {
    EdtPlan p;
    if (!make_plan(nx, ny, nz, &p, 0) || nscenes <= 0) return 0;
    return scratch_bytes_for(p, nscenes);
}

extern "C" int vx_edt(vx_ctx *c, const uint8_t *occ, int nx, int ny, int nz, double vs, vx_field **out) {
    (void)vs;
    if (!c || !occ || !out) return fail(VX_EINVAL, "NULL argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    const size_t n = (size_t)nx * ny * nz;
    VX_CUDA(c->staging.ensure(n));
    VX_CUDA(cudaMemcpyAsync(c->staging.p, occ, n, cudaMemcpyHostToDevice, c->stream));
    c->h2d += (long long)n;
    vx_field *f = nullptr;
    rc = field_new(c, nx, ny, nz, &f);
    if (rc) return rc;
    rc = edt_run(c, (const uint8_t *)c->staging.p, nx, ny, nz, 1, f->site, nullptr, 0);
    if (rc) {
        vx_field_destroy(f);
        return rc;
    }
    *out = f;
    return VX_OK;
}

extern "C" int vx_edt_grid(vx_grid *g, double thr, vx_field **out) {
    if (!g || !out) return fail(VX_EINVAL, "NULL argument");
    const uint8_t *d = nullptr;
    int rc = grid_occ_device(g, thr, &d);
    if (rc) return rc;
    vx_field *f = nullptr;
    rc = field_new(g->ctx, g->g.nx, g->g.ny, g->g.nz, &f);
    if (rc) return rc;
    rc = edt_run(g->ctx, d, g->g.nx, g->g.ny, g->g.nz, 1, f->site, nullptr, 0);
    if (rc) {
        vx_field_destroy(f);
        return rc;
    }
    *out = f;
    return VX_OK;
}

// brute_force_edt (edt.py:487-508) on the GPU: site compaction in flat-index
// order, then an exhaustive minimum per voxel with lexicographic ties
extern "C" int vx_brute_force_edt(vx_ctx *c, const uint8_t *occ, int nx, int ny, int nz, vx_field **out) {
    if (!c || !occ || !out) return fail(VX_EINVAL, "NULL argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    const size_t n = (size_t)nx * ny * nz;
    VX_CUDA(c->staging.ensure(n));
    VX_CUDA(cudaMemcpyAsync(c->staging.p, occ, n, cudaMemcpyHostToDevice, c->stream));
    const uint8_t *d_occ = (const uint8_t *)c->staging.p;
    VX_CUDA(c->exp.ensure(occ_scratch_bytes((long long)n)));
    cudaError_t e = launch_occ_layout(d_occ, (long long)n, c->exp.p, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "brute_force_edt (layout)");
    long long total = 0;
    VX_CUDA(cudaMemcpyAsync(&total, occ_total_ptr(c->exp.p, (long long)n), 8, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    VX_CUDA(c->exp_out.ensure((size_t)std::max(total, 1LL) * 24));
    if (total) {
        e = launch_occ_write(d_occ, (long long)n, ny, nz, c->exp.p, (long long *)c->exp_out.p, c->stream);
        if (e != cudaSuccess) return cuda_fail(e, "brute_force_edt (sites)");
    }
    vx_field *f = nullptr;
    rc = field_new(c, nx, ny, nz, &f);
    if (rc) return rc;
    e = launch_brute_force((const long long *)c->exp_out.p, total, nx, ny, nz, f->site, c->stream);
    if (e != cudaSuccess) {
        vx_field_destroy(f);
        return cuda_fail(e, "brute_force_edt");
    }
    c->launches += 4;
    *out = f;
    return VX_OK;
}

extern "C" int vx_field_create(vx_ctx *c, int nx, int ny, int nz, vx_field **out) {
    if (!c || !out) return fail(VX_EINVAL, "NULL argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    return field_new(c, nx, ny, nz, out);
}

// pba_edt(grid.occupancy_mask(thr)) into an existing field (a pooled buffer:
// no allocation per call); the data never leaves the device
extern "C" int vx_edt_grid_into(vx_grid *g, double thr, vx_field *f) {
    if (!g || !f) return fail(VX_EINVAL, "NULL argument");
    if (f->nx != g->g.nx || f->ny != g->g.ny || f->nz != g->g.nz || !f->owned)
        return fail(VX_EINVAL, "field dims (%d, %d, %d) do not match the grid (%d, %d, %d)", f->nx, f->ny, f->nz,
                    g->g.nx, g->g.ny, g->g.nz);
    const uint8_t *d = nullptr;
    int rc = grid_occ_device(g, thr, &d);
    if (rc) return rc;
    return edt_run(g->ctx, d, g->g.nx, g->g.ny, g->g.nz, 1, f->site, nullptr, 0);
}

// engine.py:259-268's memo key without the N-byte copy: a digest of the
// occupied-voxel set at `thr` computed on the device (O(touched voxels) when
// the grid's touched list covers its occupancy); 16 bytes come back.  Equal
// occupancy => equal digest; unequal occupancy collides with probability
// ~2^-64, as a 128-bit blake2b of the mask does at ~2^-128.
extern "C" int vx_grid_occupancy_digest(vx_grid *g, double thr, uint64_t digest[2]) {
    if (!g || !digest) return fail(VX_EINVAL, "NULL argument");
    vx_ctx *c = g->ctx;
    const uint8_t *d = nullptr;
    int rc = grid_occ_device(g, thr, &d);
    if (rc) return rc;
    const bool list = d == g->occ && g->sparse_ok;
    // the sums go to a buffer that does not hold the occupancy (temp does when
    // thr is not the cached 0.5)
    DevBuf &accb = d == (const uint8_t *)c->temp.p ? c->exp : c->temp;
    VX_CUDA(accb.ensure(64));
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(accb.p);
    cudaError_t e = launch_occ_digest(d, g->n, g->touched, g->ctr, list, acc, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy digest");
    c->launches += 1;
    unsigned long long h[3];
    VX_CUDA(cudaMemcpyAsync(h, acc, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    c->d2h += sizeof h;
    VX_CUDA(cudaStreamSynchronize(c->stream));
    digest[0] = h[0] ^ (h[2] * 0x9E3779B97F4A7C15ull);
    digest[1] = h[1] + h[2];
    return VX_OK;
}

// _site_world (engine.py:212-221) for s centres on up to two fields in one
// round trip: outputs [field a's s results, field b's s results]
extern "C" int vx_fields_site_world(vx_field *a, vx_field *b, const double origin[3], double vs,
                                    const double *centers, int64_t s, int32_t *lin, double *world, double *dist) {
    if (!a || !origin || (s > 0 && (!centers || !lin || !world || !dist))) return fail(VX_EINVAL, "NULL argument");
    if (b && (b->nx != a->nx || b->ny != a->ny || b->nz != a->nz)) return fail(VX_EINVAL, "field dims differ");
    if (s <= 0) return VX_OK;
    vx_ctx *c = a->ctx;
    const int nf = b ? 2 : 1;
    const size_t bc = (size_t)s * 3 * sizeof(double);
    const size_t bl = ((size_t)nf * s * 4 + 15) & ~(size_t)15;
    VX_CUDA(c->temp.ensure(bc + bl + nf * bc + (size_t)nf * s * 8));
    unsigned char *d = (unsigned char *)c->temp.p;
    VX_CUDA(cudaMemcpyAsync(d, centers, bc, cudaMemcpyHostToDevice, c->stream));
    c->h2d += (long long)bc;
    GridGeom g{a->nx, a->ny, a->nz, vs, origin[0], origin[1], origin[2]};
    int32_t *dl = (int32_t *)(d + bc);
    double *dw = (double *)(d + bc + bl), *dd = (double *)(d + bc + bl + nf * bc);
    for (int q = 0; q < nf; ++q) {
        cudaError_t e = launch_site_world((q ? b : a)->site, g, (const double *)d, (int)s, dl + q * s,
                                          dw + (size_t)q * s * 3, dd + (size_t)q * s, c->stream);
        if (e != cudaSuccess) return cuda_fail(e, "site_world");
        c->launches += 1;
    }
    VX_CUDA(cudaMemcpyAsync(lin, dl, (size_t)nf * s * 4, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaMemcpyAsync(world, dw, (size_t)nf * bc, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaMemcpyAsync(dist, dd, (size_t)nf * s * 8, cudaMemcpyDeviceToHost, c->stream));
    c->d2h += (long long)nf * s * (4 + 24 + 8);
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

// slab mode: _site_world on this rank's j-slab (device site
// array (nx, nyl, nz) holding rows j0.., global flat indices); centres whose
// row another rank holds come back with lin -2 (the caller gathers)
extern "C" int vx_site_world_slab(vx_ctx *c, const int32_t *d_site, int nx, int ny, int nz, int j0, int nyl,
                                  const double origin[3], double vs, const double *centers, int64_t s,
                                  int32_t *lin, double *world, double *dist) {
    if (!c || !d_site || !origin || (s > 0 && (!centers || !lin || !world || !dist)))
        return fail(VX_EINVAL, "NULL argument");
    if (j0 < 0 || nyl < 0 || j0 + nyl > ny) return fail(VX_EINVAL, "bad j-slab [%d, %d) of %d", j0, j0 + nyl, ny);
    if (s <= 0) return VX_OK;
    const size_t bc = (size_t)s * 3 * sizeof(double);
    const size_t bl = ((size_t)s * 4 + 15) & ~(size_t)15;
    VX_CUDA(c->temp.ensure(bc + bl + bc + (size_t)s * 8));
    unsigned char *d = (unsigned char *)c->temp.p;
    VX_CUDA(cudaMemcpyAsync(d, centers, bc, cudaMemcpyHostToDevice, c->stream));
    c->h2d += (long long)bc;
    GridGeom g{nx, ny, nz, vs, origin[0], origin[1], origin[2]};
    cudaError_t e = launch_site_world(d_site, g, (const double *)d, (int)s, (int32_t *)(d + bc),
                                      (double *)(d + bc + bl), (double *)(d + bc + bl + bc), c->stream, j0, nyl);
    if (e != cudaSuccess) return cuda_fail(e, "site_world_slab");
    c->launches += 1;
    VX_CUDA(cudaMemcpyAsync(lin, d + bc, (size_t)s * 4, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaMemcpyAsync(world, d + bc + bl, bc, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaMemcpyAsync(dist, d + bc + bl + bc, (size_t)s * 8, cudaMemcpyDeviceToHost, c->stream));
    c->d2h += (long long)s * 36;
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

extern "C" int vx_ctx_transfer_bytes(const vx_ctx *c, int64_t out[2]) {
    if (!c || !out) return fail(VX_EINVAL, "NULL argument");
    out[0] = c->h2d;
    out[1] = c->d2h;
    return VX_OK;
}

extern "C" int vx_line_nearest_sites(vx_ctx *c, const uint8_t *occ, int nx, int ny, int nz, int32_t *s1) {
    if (!c || !occ || !s1) return fail(VX_EINVAL, "NULL argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    const size_t n = (size_t)nx * ny * nz;
    VX_CUDA(c->staging.ensure(n));
    VX_CUDA(c->temp.ensure(n * 4 + 16));
    VX_CUDA(cudaMemcpyAsync(c->staging.p, occ, n, cudaMemcpyHostToDevice, c->stream));
    cudaError_t e = launch_pass1((const uint8_t *)c->staging.p, (int32_t *)c->temp.p, nx, ny, nz, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "pass1");
    c->launches += 1;
    VX_CUDA(cudaMemcpyAsync(s1, c->temp.p, n * 4, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

extern "C" int vx_field_destroy(vx_field *f) {
    if (!f) return VX_OK;
    if (f->owned) {
        if (f->ctx) cudaStreamSynchronize(f->ctx->stream);
        cudaFree(f->site);
        delete f;
    }
    return VX_OK;
}

extern "C" int vx_field_dims(const vx_field *f, int dims[3]) {
    if (!f || !dims) return fail(VX_EINVAL, "NULL argument");
    dims[0] = f->nx; dims[1] = f->ny; dims[2] = f->nz;
    return VX_OK;
}

extern "C" int vx_field_read_site(vx_field *f, int32_t *out) {
    if (!f || !out) return fail(VX_EINVAL, "NULL argument");
    const size_t n = (size_t)f->nx * f->ny * f->nz;
    VX_CUDA(cudaMemcpyAsync(out, f->site, n * 4, cudaMemcpyDeviceToHost, f->ctx->stream));
    f->ctx->d2h += (long long)n * 4;
    VX_CUDA(cudaStreamSynchronize(f->ctx->stream));
    return VX_OK;
}

// edt.py:123-135: squared voxel distance, int64, -1 where there is no site
extern "C" int vx_field_sq_distance(vx_field *f, int64_t *out, int out_on_device) {
    if (!f || !out) return fail(VX_EINVAL, "NULL argument");
    vx_ctx *c = f->ctx;
    const size_t n = (size_t)f->nx * f->ny * f->nz;
    long long *d = (long long *)out;
    if (!out_on_device) {
        VX_CUDA(c->exp_out.ensure(n * 8));
        d = (long long *)c->exp_out.p;
    }
    cudaError_t e = launch_sq_distance(f->site, f->nx, f->ny, f->nz, d, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "sq_distance");
    c->launches += 1;
    if (!out_on_device) VX_CUDA(cudaMemcpyAsync(out, d, n * 8, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

// edt.py:137-145: the golden text of dump_squared.  buf == NULL (or too
// small): *nbytes only (VX_ERANGE if short).  No terminating NUL.
extern "C" int vx_field_dump_squared(vx_field *f, char *buf, int64_t capacity, int64_t *nbytes) {
    if (!f || !nbytes) return fail(VX_EINVAL, "NULL argument");
    if (f->ny > 65535) return fail(VX_EINVAL, "dump_squared: ny %d > 65535", f->ny);
    vx_ctx *c = f->ctx;
    VX_CUDA(c->exp.ensure(dump_scratch_bytes(f->ny, f->nz)));
    cudaError_t e = launch_dump_layout(f->site, f->nx, f->ny, f->nz, c->exp.p, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "dump_squared");
    c->launches += 2;
    long long total = 0;
    VX_CUDA(cudaMemcpyAsync(&total, dump_total_ptr(c->exp.p, f->ny, f->nz), 8, cudaMemcpyDeviceToHost,
                            c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    *nbytes = total;
    if (!buf) return VX_OK;
    if (capacity < total) return fail(VX_ERANGE, "capacity %lld < %lld bytes", (long long)capacity, total);
    VX_CUDA(c->exp_out.ensure((size_t)total));
    e = launch_dump_write(f->site, f->nx, f->ny, f->nz, c->exp.p, (char *)c->exp_out.p, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "dump_squared");
    c->launches += 1;
    VX_CUDA(cudaMemcpyAsync(buf, c->exp_out.p, (size_t)total, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

extern "C" int vx_field_site_at(vx_field *f, int64_t i, int64_t j, int64_t k, int32_t *out) {
    if (!f || !out) return fail(VX_EINVAL, "NULL argument");
    if (!(0 <= i && i < f->nx && 0 <= j && j < f->ny && 0 <= k && k < f->nz))
        return fail(VX_ERANGE, "voxel (%lld, %lld, %lld) outside grid (%d, %d, %d)", (long long)i,
                    (long long)j, (long long)k, f->nx, f->ny, f->nz);
    const size_t off = ((size_t)i * f->ny + j) * f->nz + k;
    VX_CUDA(cudaMemcpyAsync(out, f->site + off, 4, cudaMemcpyDeviceToHost, f->ctx->stream));
    f->ctx->d2h += 4;
    VX_CUDA(cudaStreamSynchronize(f->ctx->stream));
    return VX_OK;
}

extern "C" int vx_field_site_world(vx_field *f, const double origin[3], double vs, const double *centers,
                                   int64_t s, int32_t *lin, double *world, double *dist) {
    if (!f || !origin || (s > 0 && (!centers || !lin || !world || !dist)))
        return fail(VX_EINVAL, "NULL argument");
    if (s <= 0) return VX_OK;
    vx_ctx *c = f->ctx;
    const size_t bc = (size_t)s * 3 * sizeof(double);
    const size_t bl = ((size_t)s * 4 + 15) & ~(size_t)15;
    VX_CUDA(c->temp.ensure(bc + bl + bc + (size_t)s * 8));
    unsigned char *d = (unsigned char *)c->temp.p;
    VX_CUDA(cudaMemcpyAsync(d, centers, bc, cudaMemcpyHostToDevice, c->stream));
    GridGeom g{f->nx, f->ny, f->nz, vs, origin[0], origin[1], origin[2]};
    cudaError_t e = launch_site_world(f->site, g, (const double *)d, (int)s, (int32_t *)(d + bc),
                                      (double *)(d + bc + bl), (double *)(d + bc + bl + bc), c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "site_world");
    c->launches += 1;
    VX_CUDA(cudaMemcpyAsync(lin, d + bc, (size_t)s * 4, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaMemcpyAsync(world, d + bc + bl, bc, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaMemcpyAsync(dist, d + bc + bl + bc, (size_t)s * 8, cudaMemcpyDeviceToHost, c->stream));
    VX_CUDA(cudaStreamSynchronize(c->stream));
    return VX_OK;
}

// ---- device-pointer entry points -------------------------------------------------
extern "C" int vx_edt_device(vx_ctx *c, const uint8_t *d_occ, int nx, int ny, int nz, int nscenes,
                             int32_t *d_site, void *d_scratch, size_t scratch_bytes) {
    if (!c || !d_occ || !d_site || nscenes <= 0) return fail(VX_EINVAL, "bad argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    return edt_run(c, d_occ, nx, ny, nz, nscenes, d_site, d_scratch, scratch_bytes);
}

extern "C" int vx_edt_s2_bytes(int nx, int ny, int nz) {
    EdtPlan p;
    if (!make_plan(nx, ny, nz, &p, 0)) return 0;
    return p.s2_wide ? 8 : 4;
}

extern "C" int vx_edt_pass12_device(vx_ctx *c, const uint8_t *d_occ, int nx, int ny, int nz, int nxl,
                                    void *d_s2, void *d_scratch, size_t scratch_bytes) {
    if (!c || !d_occ || !d_s2 || nxl < 0 || nxl > nx) return fail(VX_EINVAL, "bad argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    EdtPlan p;
    make_plan(nx, ny, nz, &p, 0);
    const size_t s1b = ((size_t)nxl * ny * nz * 4 + 255) & ~(size_t)255;
    const size_t need = s1b + p.gstack_bytes;
    if (!d_scratch) {
        VX_CUDA(c->scratch.ensure(need));
        d_scratch = c->scratch.p;
    } else if (scratch_bytes < need) {
        return fail(VX_EINVAL, "scratch too small");
    }
    int32_t *s1 = (int32_t *)d_scratch;
    cudaError_t e = launch_pass1(d_occ, s1, nxl, ny, nz, c->stream, nullptr, p.s1_16);
    if (e == cudaSuccess) e = launch_pass2(s1, d_s2, (unsigned char *)d_scratch + s1b, p, nxl, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "pass12");
    c->launches += 2;
    return VX_OK;
}

// slab-mode calls have no occupied-slice list, only the search header
static int slab_rows(vx_ctx *c, SparseRows *sp) {
    if (!c->slabhdr.p) {
        VX_CUDA(c->slabhdr.ensure(256));
        VX_CUDA(cudaMemsetAsync(c->slabhdr.p, 0, c->slabhdr.n, c->stream));
    }
    *sp = SparseRows{};
    sp->sflag = nullptr;
    sp->xs = nullptr;
    sp->hdr = nullptr;
    sp->fails = static_cast<int *>(c->slabhdr.p);
    return VX_OK;
}

extern "C" int vx_edt_pass12_scatter(vx_ctx *c, const uint8_t *d_occ, int nx, int ny, int nz, int nxl,
                                     int nranks, void *const *dst, const int *j_starts, long long x_base,
                                     void *d_scratch, size_t scratch_bytes) {
    if (!c || !d_occ || !dst || !j_starts || nxl < 0 || nxl > nx || nranks < 1 || nranks > kMaxRanks)
        return fail(VX_EINVAL, "bad argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    if (j_starts[0] != 0 || j_starts[nranks] != ny) return fail(VX_EINVAL, "j_starts must cover 0..ny");
    ScatterTab tab{};
    tab.nranks = nranks;
    tab.x_base = x_base;
    for (int q = 0; q < nranks; ++q) {
        if (j_starts[q + 1] < j_starts[q]) return fail(VX_EINVAL, "j_starts must be non-decreasing");
        tab.dst[q] = dst[q];
        tab.j_start[q] = j_starts[q];
    }
    tab.j_start[nranks] = ny;
    EdtPlan p;
    make_plan(nx, ny, nz, &p, 0);
    if (p.s2_wide) return fail(VX_EINVAL, "slab exchange needs 32-bit pass-2 codes");
    const size_t s1b = ((size_t)nxl * ny * nz * 4 + 255) & ~(size_t)255;
    const size_t need = s1b + p.gstack_bytes;
    if (!d_scratch) {
        VX_CUDA(c->scratch.ensure(need));
        d_scratch = c->scratch.p;
    } else if (scratch_bytes < need) {
        return fail(VX_EINVAL, "scratch too small");
    }
    int32_t *s1 = (int32_t *)d_scratch;
    SparseRows sp;
    if ((rc = slab_rows(c, &sp))) return rc;
    cudaError_t e = launch_pass1(d_occ, s1, nxl, ny, nz, c->stream, &sp, p.s1_16);
    if (e != cudaSuccess) return cuda_fail(e, "pass12_scatter (pass 1)");
    e = launch_pass2_scatter(s1, tab, (unsigned char *)d_scratch + s1b, p, nxl, c->stream, &sp);
    if (e != cudaSuccess) return cuda_fail(e, "pass12_scatter (pass 2)");
    c->launches += 2;
    return VX_OK;
}

extern "C" int vx_edt_pass3_device(vx_ctx *c, const void *d_s2, int nx, int ny, int nz, int j0, int nyl,
                                   int32_t *d_site, void *d_scratch, size_t scratch_bytes) {
    if (!c || !d_s2 || !d_site || j0 < 0 || nyl < 0 || j0 + nyl > ny) return fail(VX_EINVAL, "bad argument");
    int rc = check_edt_dims(nx, ny, nz);
    if (rc) return rc;
    EdtPlan p;
    make_plan(nx, ny, nz, &p, 0);
    if (p.gstack_bytes) {
        if (!d_scratch) {
            VX_CUDA(c->scratch.ensure(p.gstack_bytes));
            d_scratch = c->scratch.p;
        } else if (scratch_bytes < p.gstack_bytes) {
            return fail(VX_EINVAL, "scratch too small");
        }
    }
    SparseRows sp;
    if ((rc = slab_rows(c, &sp))) return rc;
    cudaError_t e = launch_pass3(d_s2, d_site, d_scratch, p, 1, j0, nyl, c->stream, &sp);
    if (e != cudaSuccess) return cuda_fail(e, "pass3");
    c->launches += 1;
    return VX_OK;
}

// ---- camera-tick pipeline (engine.py:233-280) ----------------------------------------
struct vx_cycle {
    vx_ctx *ctx = nullptr;
    vx_grid *env = nullptr, *self = nullptr, *mask = nullptr;
    vx_field env_f, self_f;
    int nlinks = 0, nself = 0;
    int64_t total_all = 0, total_self = 0, max_points = 0;
    int max_spheres = 0;
    // device tables: all links, then the self-obstacle subset
    unsigned char *tab = nullptr;
    int32_t *ijk_all = nullptr, *ijk_self = nullptr;
    int64_t *off_all = nullptr, *off_self = nullptr;
    double *org_all = nullptr, *org_self = nullptr, *vs_all = nullptr, *vs_self = nullptr;
    double *T_all = nullptr, *T_self = nullptr;
    std::vector<int> self_links;
    // per-step buffers
    double *d_pts = nullptr, *d_centers = nullptr;
    int32_t *d_lin = nullptr;
    double *d_world = nullptr, *d_dist = nullptr;
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    // K7 avoidance rows (tasks.py:88-123), enabled by vx_cycle_set_avoidance
    int av_s = 0, av_nj = 0;
    double av_kappa = 0.0, av_offset = -1.0;
    double *d_av_par = nullptr;   // radius[s], buffer[s]
    int *d_av_link = nullptr;
    double *d_frames = nullptr, *h_frames = nullptr;   // origins[nj*3], axes[nj*3] (pinned)
    double *d_J = nullptr, *d_act = nullptr, *d_ref = nullptr, *d_val = nullptr;
    int *d_flag = nullptr;
    EdtPlan plan{};
    std::vector<double> last_self_T;
    bool self_valid = false;
    int last_s = 0;
    int self_recomputed = 0;
    // CUDA graph of the per-tick sequence (mask/env reset, stamp, scatter,
    // EDT, gather); the cloud size is read from d_npts on the device
    bool use_graph = true;
    long long *d_npts = nullptr, *h_npts = nullptr;  // device / pinned host point count
    // per-step arguments staged in one H2D copy: {npts, cloud pointer | pad |
    // link frames (nlinks x 4x4) | sphere centres}; kStage pinned host slots
    // let the host run up to kStage ticks ahead of the device
    static constexpr int kStage = 8;
    unsigned char *d_stage = nullptr, *h_stage[kStage] = {};
    cudaEvent_t ev_stage[kStage] = {};
    size_t stage_bytes = 0;
    int stage_slot = 0, nstage = kStage;
    // occupied-slice count of the last env EDT (host-mapped, written by the
    // device) -> which pass-3 kernels the next tick launches
    int *h_m = nullptr, *d_m = nullptr;
    int p3_mode = 0, g_mode = -1;
    int m_hint = -1;   // previous tick's occupied-slice count (dense scenes: windowed search)
    int captures = 0, last_graph = 0;   // vx_cycle_info
    unsigned char *h_out = nullptr, *d_out = nullptr;   // packed results (host-mapped)
    // vx_cycle_prefetch: the next cloud is uploaded on a copy stream into one
    // of two device slots while the current tick computes
    cudaStream_t cst = nullptr;
    double *d_pb[2] = {nullptr, nullptr};
    cudaEvent_t ev_up[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
    unsigned long long pf_ticket[2] = {0, 0};   // 0 = slot empty or consumed
    long long pf_n[2] = {-1, -1};
    unsigned long long pf_issued = 0;
    int pf_next = 0;
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;   // kept while gexec lives (its reset node is updated per tick)
    // the graph's reset node copies the per-step block from the host-mapped
    // staging slot of the tick: its CopySpan source is set before each launch
    cudaGraphNode_t g_reset = nullptr;
    cudaKernelNodeParams g_reset_kp = {};
    ResetArgs g_ra = {}, g_rb = {};
    ZeroSpan g_z[3] = {};
    CopySpan g_cp = {};
    unsigned char *d_hstage[kStage] = {};   // device views of h_stage (mapped)
    bool capturing = false;
    int g_s = -1;
    float g_hit = 0.f;
    double g_thr = 0.0;
    long long g_kernels = 0;
    // per-phase CUDA-event timing (vx_cycle_profile)
    static constexpr int kRing = 64;
    bool profiling = false;
    cudaEvent_t ev[kRing][VX_CYCLE_PHASES + 1] = {};
    int ring_n = 0;      // steps recorded since the last reset
    int ring_used = 0;   // event sets created
    void mark(int phase) {
        if (profiling && ring_n < kRing) cudaEventRecord(ev[ring_n][phase], ctx->stream);
    }
};
static void drop_graph(vx_cycle *cy);

static void av_free(vx_cycle *cy);

extern "C" int vx_cycle_create(vx_ctx *c, int nx, int ny, int nz, double vs, const double origin[3],
                               int nlinks, const int32_t *const *link_ijk, const int64_t *link_counts,
                               const double *link_origins, double link_vs, const int32_t *self_links,
                               int n_self, int64_t max_points, int max_spheres, vx_cycle **out) {
    if (!c || !out || nlinks < 0 || n_self < 0 || max_points < 0 || max_spheres < 0)
        return fail(VX_EINVAL, "bad argument");
    int rc = check_geom(nx, ny, nz, vs);
    if (rc) return rc;
    for (int s = 0; s < n_self; ++s)
        if (self_links[s] < 0 || self_links[s] >= nlinks) return fail(VX_EINVAL, "bad self link index");
    vx_cycle *cy = new vx_cycle;
    cy->ctx = c;
    cy->nlinks = nlinks;
    cy->nself = n_self;
    cy->self_links.assign(self_links, self_links + n_self);
    cy->max_points = max_points;
    cy->max_spheres = max_spheres;
    auto bail = [&](int code) {
        vx_cycle_destroy(cy);
        return code;
    };
    if ((rc = vx_grid_create(c, nx, ny, nz, vs, origin, &cy->env))) return bail(rc);
    if ((rc = vx_grid_create(c, nx, ny, nz, vs, origin, &cy->self))) return bail(rc);
    if ((rc = vx_grid_create(c, nx, ny, nz, vs, origin, &cy->mask))) return bail(rc);
    // link tables
    std::vector<int64_t> off_all(nlinks + 1, 0), off_self(n_self + 1, 0);
    for (int l = 0; l < nlinks; ++l) off_all[l + 1] = off_all[l] + link_counts[l];
    for (int s = 0; s < n_self; ++s) off_self[s + 1] = off_self[s] + link_counts[self_links[s]];
    cy->total_all = off_all[nlinks];
    cy->total_self = off_self[n_self];
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_ia = al(cy->total_all * 12), b_is = al(cy->total_self * 12);
    const size_t b_oa = al(8 * (nlinks + 1)), b_os = al(8 * (n_self + 1));
    const size_t b_ga = al(24 * nlinks + 8), b_gs = al(24 * n_self + 8);
    const size_t b_va = al(8 * nlinks + 8), b_vs = al(8 * n_self + 8);
    const size_t b_Ta = al(128 * nlinks + 8), b_Ts = al(128 * n_self + 8);
    const size_t tab_bytes = b_ia + b_is + b_oa + b_os + b_ga + b_gs + b_va + b_vs + b_Ta + b_Ts;
    std::vector<unsigned char> h(tab_bytes, 0);
    size_t p = 0;
    auto place = [&](size_t bytes) { size_t q = p; p += bytes; return q; };
    const size_t o_ia = place(b_ia), o_is = place(b_is), o_oa = place(b_oa), o_os = place(b_os);
    const size_t o_ga = place(b_ga), o_gs = place(b_gs), o_va = place(b_va), o_vs = place(b_vs);
    const size_t o_Ta = place(b_Ta), o_Ts = place(b_Ts);
    for (int l = 0; l < nlinks; ++l) {
        if (link_counts[l]) std::memcpy(&h[o_ia + off_all[l] * 12], link_ijk[l], link_counts[l] * 12);
        std::memcpy(&h[o_ga + 24 * l], link_origins + 3 * l, 24);
        std::memcpy(&h[o_va + 8 * l], &link_vs, 8);
    }
    for (int s = 0; s < n_self; ++s) {
        const int l = self_links[s];
        if (link_counts[l]) std::memcpy(&h[o_is + off_self[s] * 12], link_ijk[l], link_counts[l] * 12);
        std::memcpy(&h[o_gs + 24 * s], link_origins + 3 * l, 24);
        std::memcpy(&h[o_vs + 8 * s], &link_vs, 8);
    }
    std::memcpy(&h[o_oa], off_all.data(), 8 * (nlinks + 1));
    std::memcpy(&h[o_os], off_self.data(), 8 * (n_self + 1));
    cudaError_t e = cudaMalloc(&cy->tab, tab_bytes);
    if (e == cudaSuccess) e = cudaMemcpy(cy->tab, h.data(), tab_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cycle tables"));
    cy->ijk_all = (int32_t *)(cy->tab + o_ia); cy->ijk_self = (int32_t *)(cy->tab + o_is);
    cy->off_all = (int64_t *)(cy->tab + o_oa); cy->off_self = (int64_t *)(cy->tab + o_os);
    cy->org_all = (double *)(cy->tab + o_ga); cy->org_self = (double *)(cy->tab + o_gs);
    cy->vs_all = (double *)(cy->tab + o_va); cy->vs_self = (double *)(cy->tab + o_vs);
    cy->T_all = (double *)(cy->tab + o_Ta); cy->T_self = (double *)(cy->tab + o_Ts);
    // per-step buffers
    const size_t S = (size_t)(max_spheres > 0 ? max_spheres : 1);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_pts, (size_t)(max_points > 0 ? max_points : 1) * 24);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_centers, S * 24);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_lin, 2 * S * 4);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_world, 2 * S * 24);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_dist, 2 * S * 8);
    if (e == cudaSuccess) e = cudaHostAlloc(&cy->h_npts, sizeof(long long), cudaHostAllocPortable);
    cy->stage_bytes = (64 + (size_t)nlinks * 128 + S * 24 + 15) & ~(size_t)15;
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_stage, cy->stage_bytes);
    if (const char *ev = getenv("VX_STAGE_SLOTS")) cy->nstage = std::max(1, std::min(vx_cycle::kStage, atoi(ev)));
    for (int b = 0; b < vx_cycle::kStage && e == cudaSuccess; ++b) {
        e = cudaHostAlloc(&cy->h_stage[b], cy->stage_bytes, cudaHostAllocMapped | cudaHostAllocPortable);
        if (e == cudaSuccess) e = cudaHostGetDevicePointer((void **)&cy->d_hstage[b], cy->h_stage[b], 0);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cy->ev_stage[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) {   // the graph reads frames, centres and the count from the staged block
        cy->d_npts = reinterpret_cast<long long *>(cy->d_stage);
        cy->T_all = reinterpret_cast<double *>(cy->d_stage + 64);
        cudaFree(cy->d_centers);
        cy->d_centers = reinterpret_cast<double *>(cy->d_stage + 64 + (size_t)nlinks * 128);
    }
    if (e == cudaSuccess) e = cudaHostAlloc(&cy->h_m, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaSuccess)
        e = cudaHostAlloc(&cy->h_out, 64 + 8 + S * 2 * 36, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&cy->d_out, cy->h_out, 0);
    // vx_cycle_prefetch slots, copy stream and events (allocated up front so
    // the first prefetch does not allocate)
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cy->cst, cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaMalloc(&cy->d_pb[b], (size_t)std::max<int64_t>(max_points, 1) * 24);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cy->ev_up[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cy->ev_used[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(cy->ev_used[b], c->stream);
    }
    if (e == cudaSuccess) {
        *cy->h_m = -1;
        e = cudaHostGetDevicePointer(&cy->d_m, cy->h_m, 0);
    }
    for (vx_field *f : {&cy->env_f, &cy->self_f}) {
        f->ctx = c;
        f->nx = nx; f->ny = ny; f->nz = nz;
        f->owned = false;
        if (e == cudaSuccess) e = cudaMalloc(&f->site, (size_t)nx * ny * nz * 4);
    }
    if (e != cudaSuccess) return bail(cuda_fail(e, "cycle buffers"));
    make_plan(nx, ny, nz, &cy->plan, 0);
    cy->scratch_bytes = scratch_bytes_for(cy->plan, 1);
    e = cudaMalloc(&cy->scratch, cy->scratch_bytes);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cycle scratch"));
    *out = cy;
    return VX_OK;
}

extern "C" int vx_cycle_destroy(vx_cycle *cy) {
    if (!cy) return VX_OK;
    if (cy->ctx) cudaStreamSynchronize(cy->ctx->stream);
    vx_grid_destroy(cy->env);
    vx_grid_destroy(cy->self);
    vx_grid_destroy(cy->mask);
    cudaFree(cy->tab);
    cudaFree(cy->d_pts);
    if (!cy->d_stage) cudaFree(cy->d_centers);   // else it lives in d_stage
    cudaFree(cy->d_stage);
    for (int b = 0; b < vx_cycle::kStage; ++b) {
        if (cy->h_stage[b]) cudaFreeHost(cy->h_stage[b]);
        if (cy->ev_stage[b]) cudaEventDestroy(cy->ev_stage[b]);
    }
    cudaFree(cy->d_lin);
    cudaFree(cy->d_world);
    cudaFree(cy->d_dist);
    av_free(cy);
    if (cy->h_npts) cudaFreeHost(cy->h_npts);
    if (cy->h_m) cudaFreeHost(cy->h_m);
    if (cy->h_out) cudaFreeHost(cy->h_out);
    for (int b = 0; b < 2; ++b) {
        cudaFree(cy->d_pb[b]);
        if (cy->ev_up[b]) cudaEventDestroy(cy->ev_up[b]);
        if (cy->ev_used[b]) cudaEventDestroy(cy->ev_used[b]);
    }
    if (cy->cst) cudaStreamDestroy(cy->cst);
    drop_graph(cy);
    cudaFree(cy->env_f.site);
    cudaFree(cy->self_f.site);
    cudaFree(cy->scratch);
    for (int r = 0; r < cy->ring_used; ++r)
        for (int q = 0; q <= VX_CYCLE_PHASES; ++q)
            if (cy->ev[r][q]) cudaEventDestroy(cy->ev[r][q]);
    delete cy;
    return VX_OK;
}

// src: the grid whose occupancy this is; when its touched list covers every
// occupied voxel the slice flags come from that list
// flags_ready: the occupied-slice flags were set by the insert's finalize
static cudaError_t edt_passes(vx_cycle *cy, const vx_grid *src, int32_t *site, bool marks,
                              bool flags_ready = false, bool list_ready = false) {
    const uint8_t *occ = src->occ;
    unsigned char *base = static_cast<unsigned char *>(cy->scratch);
    const EdtPlan &p = cy->plan;
    const size_t n = (size_t)p.nx * p.ny * p.nz;
    const size_t s1b = (n * 4 + 255) & ~(size_t)255;
    const size_t s2b = (n * (p.s2_wide ? 8 : 4) + 255) & ~(size_t)255;
    int32_t *s1 = reinterpret_cast<int32_t *>(base);
    void *s2 = base + s1b, *gs = base + s1b + s2b;
    cudaStream_t st = cy->ctx->stream;
    const bool sparse = sparse_ok(p, 1);
    SparseRows sp{};
    cudaError_t e = cudaSuccess;
    if (sparse) {
        sp = sparse_rows_at(base + s1b + s2b + p.gstack_bytes, p);
        if (src == cy->env) {   // the per-tick map: feed and use the count hint
            sp.m_mirror = cy->d_m;
            sp.p3_mode = cy->p3_mode;
            sp.m_hint = cy->m_hint;
        }
        if (list_ready) {
            // the insert's finalize built the list (and the host-mapped hint)
        } else if (flags_ready) {
            e = launch_slice_list_only(p, sp, st);
            cy->ctx->launches += 1;
        } else {
            if (src->sparse_ok) e = launch_slice_list_touched(src->touched, src->ctr, occ, p, sp, st);
            else e = launch_slice_list(occ, p, sp, st);
            cy->ctx->launches += 2;
        }
    }
    if (e == cudaSuccess) e = launch_pass1(occ, s1, p.nx, p.ny, p.nz, st, sparse ? &sp : nullptr, p.s1_16);
    if (marks) cy->mark(5);
    if (e == cudaSuccess) e = launch_pass2(s1, s2, gs, p, p.nx, st, sparse ? &sp : nullptr);
    if (marks) cy->mark(6);
    // sparse path: s1 is dead by pass 3 and is the spill slab of its column stacks
    if (e == cudaSuccess) e = launch_pass3(s2, site, sparse ? (void *)s1 : gs, p, 1, 0, p.ny, st, sparse ? &sp : nullptr);
    if (marks) cy->mark(7);
    cy->ctx->launches += 3;
    return e;
}

// engine.py:236-254 and 272-280: mask <- all links; env <- cloud minus mask;
// EDT of env; the per-sphere gather on both fields.  n_dev (graph mode): the
// point count is read on the device and npts only sizes the launch.
static void drop_graph(vx_cycle *cy) {
    if (cy->gexec) cudaGraphExecDestroy(cy->gexec);
    if (cy->graph) cudaGraphDestroy(cy->graph);
    cy->gexec = nullptr;
    cy->graph = nullptr;
    cy->g_reset = nullptr;
}

static int cycle_main_seq(vx_cycle *cy, const double *d_pts, long long npts, const long long *n_dev,
                          float hit, double thr, int s, bool marks) {
    vx_ctx *c = cy->ctx;
    cudaStream_t st = c->stream;
    int rc;
    // the env EDT's occupied-slice flags come out of the (fresh-grid) finalize
    // (and, from its last block, the occupied-slice list and the host-mapped hint)
    uint8_t *sflag = nullptr;
    SparseRows sp_env{};
    if (sparse_ok(cy->plan, 1)) {
        const EdtPlan &p = cy->plan;
        const size_t nv = (size_t)p.nx * p.ny * p.nz;
        const size_t s1b = (nv * 4 + 255) & ~(size_t)255, s2b = (nv * (p.s2_wide ? 8 : 4) + 255) & ~(size_t)255;
        sp_env = sparse_rows_at(static_cast<unsigned char *>(cy->scratch) + s1b + s2b + p.gstack_bytes, p);
        sp_env.m_mirror = cy->d_m;
        sflag = const_cast<uint8_t *>(sp_env.sflag);
    }
    // one launch resets the mask and env grids and zeroes the slice flags, the
    // mask's per-link OOB counters and the env insert stats
    if (cy->nlinks && (rc = ensure_set_oob(cy->mask, cy->nlinks))) return rc;
    {
        const ResetArgs ra{cy->mask->cells, cy->mask->occ, cy->mask->touched, cy->mask->ctr, cy->mask->n,
                           cy->mask->sparse_ok ? 0 : 1};
        const ResetArgs rb{cy->env->cells, cy->env->occ, cy->env->touched, cy->env->ctr, cy->env->n,
                           cy->env->sparse_ok ? 0 : 1};
        const ZeroSpan z0{sflag, sflag ? (size_t)cy->plan.nx : 0},
            z1{cy->mask->set_oob, cy->nlinks ? (size_t)cy->nlinks * 8 : 0},
            z2{cy->env->ctr, 3 * sizeof(unsigned long long)};
        // captured into the graph: the node also fetches the staged block
        // (source slot set per tick by cycle_step)
        const CopySpan cp = cy->capturing ? CopySpan{cy->d_stage, cy->d_hstage[0], cy->stage_bytes}
                                          : CopySpan{nullptr, nullptr, 0};
        cudaError_t e = launch_reset2(ra, rb, z0, z1, z2, st, cp);
        if (e != cudaSuccess) return cuda_fail(e, "reset");
        if (cy->capturing) {   // the node just added: the capture's only dependency now
            cudaStreamCaptureStatus cs;
            const cudaGraphNode_t *deps = nullptr;
            size_t ndeps = 0;
            e = cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &ndeps);
            if (e != cudaSuccess || ndeps != 1) return cuda_fail(e != cudaSuccess ? e : cudaErrorUnknown, "capture info");
            cy->g_reset = deps[0];
            e = cudaGraphKernelNodeGetParams(cy->g_reset, &cy->g_reset_kp);
            if (e != cudaSuccess) return cuda_fail(e, "reset node params");
            cy->g_ra = ra; cy->g_rb = rb;
            cy->g_z[0] = z0; cy->g_z[1] = z1; cy->g_z[2] = z2;
            cy->g_cp = cp;
        }
        c->launches += 1;
        for (vx_grid *g : {cy->mask, cy->env}) {   // as grid_clear_async
            g->sparse_ok = true;
            g->maybe_oor = false;
            g->fresh = true;
        }
    }
    if (cy->nlinks && (rc = stamp_sets(cy->mask, cy->nlinks, cy->ijk_all, cy->off_all, cy->org_all, cy->vs_all,
                                       cy->T_all, kLMax, cy->total_all, true)))
        return rc;
    if (marks) cy->mark(3);
    bool flags_ready = sflag != nullptr;   // no points: the zeroed flags are right
    bool list_ready = false;
    if ((npts || n_dev) && (rc = insert_device(cy->env, d_pts, npts, n_dev, hit, thr, cy->mask, nullptr, sflag,
                                               &flags_ready, true, sflag ? &sp_env : nullptr)))
        return rc;
    if (npts || n_dev) list_ready = flags_ready;
    if (marks) cy->mark(4);
    cudaError_t e = edt_passes(cy, cy->env, cy->env_f.site, marks, flags_ready, list_ready);
    if (e != cudaSuccess) return cuda_fail(e, "edt(env)");
    const GridGeom g = cy->env->g;
    e = launch_gather_pack(cy->env_f.site, cy->self_f.site, g, cy->d_centers, s, cy->d_lin, cy->d_world,
                           cy->d_dist, cy->env->ctr, cy->d_out, st);
    if (e != cudaSuccess) return cuda_fail(e, "site_world");
    c->launches += 1;
    if (cy->av_s && s == cy->av_s) {
        e = launch_avoidance_rows(cy->d_world, cy->d_dist, cy->d_lin, cy->d_centers, s, cy->d_av_par,
                                  cy->d_av_par + s, cy->d_av_link, cy->d_frames, cy->d_frames + 3 * cy->av_nj,
                                  cy->av_nj, cy->av_kappa, cy->av_offset, cy->d_J, cy->d_act, cy->d_ref,
                                  cy->d_val, cy->d_flag, st);
        if (e != cudaSuccess) return cuda_fail(e, "avoidance_rows");
        c->launches += 1;
    }
    if (marks) cy->mark(8);
    return VX_OK;
}

static int cycle_step(vx_cycle *cy, const double *pts, const double *d_pts_in, int64_t npts,
                      const double *link_T, float hit, double thr, const double *centers, int s, int sync,
                      unsigned long long ticket = 0) {
    // a cloud staged by vx_cycle_prefetch: the tick reads that device slot
    int pf_slot = -1;
    if (cy && ticket) {
        for (int b = 0; b < 2; ++b)
            if (cy->pf_ticket[b] == ticket) pf_slot = b;
        if (pf_slot < 0)
            return fail(VX_EINVAL, "prefetch ticket %llu is not staged (already consumed or overwritten)",
                        ticket);
        npts = cy->pf_n[pf_slot];
    }
    if (!cy || npts < 0 || npts > cy->max_points || s < 0 || s > cy->max_spheres ||
        (npts && !pts && !d_pts_in && pf_slot < 0) || (s && !centers) || (cy->nlinks && !link_T))
        return fail(VX_EINVAL, "bad argument (npts %lld of max %lld, spheres %d of max %d)",
                    (long long)npts, (long long)cy->max_points, s, cy->max_spheres);
    vx_ctx *c = cy->ctx;
    cudaStream_t st = c->stream;
    int rc;
    if (cy->profiling && cy->ring_n < vx_cycle::kRing && cy->ring_n >= cy->ring_used) {
        for (int q = 0; q <= VX_CYCLE_PHASES; ++q) VX_CUDA(cudaEventCreate(&cy->ev[cy->ring_n][q]));
        cy->ring_used = cy->ring_n + 1;
    }
    cy->mark(0);
    if (pf_slot >= 0) {
        VX_CUDA(cudaStreamWaitEvent(st, cy->ev_up[pf_slot], 0));
        d_pts_in = cy->d_pb[pf_slot];
        cy->pf_ticket[pf_slot] = 0;   // consumed
        cy->pf_n[pf_slot] = -1;
    }
    // H2D: the cloud (unless staged by prefetch or already on the device),
    // then one copy of the per-step block {count, cloud pointer, frames, centres}
    std::vector<double> Ts(16 * cy->nself);
    for (int q = 0; q < cy->nself; ++q) std::memcpy(&Ts[16 * q], link_T + 16 * cy->self_links[q], 128);
    const double *d_pts = d_pts_in ? d_pts_in : cy->d_pts;
    if (npts && !d_pts_in) VX_CUDA(cudaMemcpyAsync(cy->d_pts, pts, (size_t)npts * 24, cudaMemcpyHostToDevice, st));
    const bool graph_path = cy->use_graph && !cy->profiling;
    int stage_b = 0;
    {
        const int b = cy->stage_slot;
        stage_b = b;
        cy->stage_slot = (b + 1) % cy->nstage;
        VX_CUDA(cudaEventSynchronize(cy->ev_stage[b]));   // its previous copy has been read
        unsigned char *h = cy->h_stage[b];
        const long long n64 = npts;
        std::memcpy(h, &n64, 8);
        std::memcpy(h + 8, &d_pts, sizeof(d_pts));
        if (cy->nlinks) std::memcpy(h + 64, link_T, (size_t)128 * cy->nlinks);
        if (s) std::memcpy(h + 64 + (size_t)128 * cy->nlinks, centers, (size_t)s * 24);
        const size_t bytes = 64 + (size_t)128 * cy->nlinks + (size_t)s * 24;
        if (!graph_path) {   // the graph's reset node reads the mapped slot itself
            VX_CUDA(cudaMemcpyAsync(cy->d_stage, h, bytes, cudaMemcpyHostToDevice, st));
            VX_CUDA(cudaEventRecord(cy->ev_stage[b], st));
        }
    }
    if (cy->av_s && s == cy->av_s)
        VX_CUDA(cudaMemcpyAsync(cy->d_frames, cy->h_frames, (size_t)cy->av_nj * 48, cudaMemcpyHostToDevice, st));
    cy->mark(1);
    // self map: memo on the self-obstacle transforms (engine.py:259-268 skips
    // the EDT when the occupancy is unchanged; equal transforms => equal
    // occupancy, since the stamp is deterministic)
    cy->self_recomputed = 0;
    if (!cy->self_valid || Ts != cy->last_self_T) {
        if (cy->nself) VX_CUDA(cudaMemcpyAsync(cy->T_self, Ts.data(), 128 * cy->nself, cudaMemcpyHostToDevice, st));
        if ((rc = grid_clear_async(cy->self))) return rc;
        if (cy->nself && (rc = stamp_sets(cy->self, cy->nself, cy->ijk_self, cy->off_self, cy->org_self,
                                          cy->vs_self, cy->T_self, kLMax, cy->total_self)))
            return rc;
        cudaError_t e = edt_passes(cy, cy->self, cy->self_f.site, false);
        if (e != cudaSuccess) return cuda_fail(e, "edt(self)");
        cy->last_self_T = Ts;
        cy->self_valid = true;
        cy->self_recomputed = 1;
    }
    cy->mark(2);
    if (graph_path) {
        // the graph reads the cloud pointer and its size from the staged block
        cy->m_hint = *(volatile int *)cy->h_m;
        cy->p3_mode = pass3_mode_hint(cy->plan, cy->m_hint);
        // the kernels the capture contains follow both hints
        const int gmode = cy->p3_mode * 2 + (ring_hint_on(cy->plan, cy->m_hint) ? 1 : 0);
        // reset modes from the grids' state before this tick (a capture below
        // runs cycle_main_seq, which already marks the grids as reset)
        const int dense_mask = cy->mask->sparse_ok ? 0 : 1, dense_env = cy->env->sparse_ok ? 0 : 1;
        if (!cy->gexec || cy->g_s != s || cy->g_hit != hit || cy->g_thr != thr || cy->g_mode != gmode) {
            drop_graph(cy);
            const long long l0 = c->launches;
            VX_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
            cy->capturing = true;
            rc = cycle_main_seq(cy, nullptr, cy->max_points, cy->d_npts, hit, thr, s, false);
            cy->capturing = false;
            cudaGraph_t graph = nullptr;
            cudaError_t ce = cudaStreamEndCapture(st, &graph);
            if (rc) {
                if (graph) cudaGraphDestroy(graph);
                return rc;
            }
            if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
            ce = cudaGraphInstantiate(&cy->gexec, graph, 0);
            cy->graph = graph;
            if (ce != cudaSuccess) {
                drop_graph(cy);
                return cuda_fail(ce, "cudaGraphInstantiate");
            }
            cy->captures += 1;
            cy->g_kernels = c->launches - l0;
            c->launches = l0;
            cy->g_s = s;
            cy->g_mode = gmode;
            cy->g_hit = hit;
            cy->g_thr = thr;
        }
        {   // this tick's staging slot -> the reset node's copy source.  The
            // reset mode follows the grids' current state: host writes since
            // the last tick (vx_grid_write_cells on cycle grids) leave cells
            // outside the touched list, so that tick's reset must be dense (it
            // also makes the captured fresh-grid insert valid again).
            cy->g_ra.dense = dense_mask;
            cy->g_rb.dense = dense_env;
            CopySpan cp = cy->g_cp;
            cp.src = cy->d_hstage[stage_b];
            void *args[] = {&cy->g_ra, &cy->g_rb, &cy->g_z[0], &cy->g_z[1], &cy->g_z[2], &cp};
            cudaKernelNodeParams kp = cy->g_reset_kp;
            kp.kernelParams = args;
            kp.extra = nullptr;
            VX_CUDA(cudaGraphExecKernelNodeSetParams(cy->gexec, cy->g_reset, &kp));
        }
        VX_CUDA(cudaGraphLaunch(cy->gexec, st));
        for (vx_grid *g : {cy->mask, cy->env}) {   // host state after the replayed tick (as cycle_main_seq)
            g->sparse_ok = true;
            g->maybe_oor = false;
            g->fresh = false;
        }
        VX_CUDA(cudaEventRecord(cy->ev_stage[stage_b], st));   // the graph read the slot
        c->launches += cy->g_kernels;
        if (pf_slot >= 0) VX_CUDA(cudaEventRecord(cy->ev_used[pf_slot], st));   // the tick read the slot
    } else {
        cy->m_hint = *(volatile int *)cy->h_m;
        cy->p3_mode = pass3_mode_hint(cy->plan, cy->m_hint);
        if ((rc = cycle_main_seq(cy, d_pts, npts, nullptr, hit, thr, s, true))) return rc;
        if (pf_slot >= 0) VX_CUDA(cudaEventRecord(cy->ev_used[pf_slot], st));
    }
    if (cy->profiling && cy->ring_n < vx_cycle::kRing) cy->ring_n++;
    cy->last_s = s;
    cy->last_graph = graph_path ? 1 : 0;
    if (sync) VX_CUDA(cudaStreamSynchronize(st));
    return VX_OK;
}

extern "C" int vx_cycle_step(vx_cycle *cy, const double *pts, int64_t npts, const double *link_T, float hit,
                             double thr, const double *centers, int s, int sync) {
    return cycle_step(cy, pts, nullptr, npts, link_T, hit, thr, centers, s, sync);
}

extern "C" int vx_cycle_step_device(vx_cycle *cy, const double *d_pts, int64_t npts, const double *link_T,
                                    float hit, double thr, const double *centers, int s, int sync) {
    return cycle_step(cy, nullptr, d_pts, npts, link_T, hit, thr, centers, s, sync);
}

// Stage a later tick's cloud (pinned host memory) on a copy stream while the
// current tick computes.  The upload is asynchronous: the host buffer must
// stay unchanged until the tick that consumes the ticket (vx_cycle_step_staged)
// has completed.  Two slots: a third prefetch
// overwrites the oldest unconsumed one, whose ticket then fails loudly.
extern "C" int vx_cycle_prefetch(vx_cycle *cy, const double *pts, int64_t npts, uint64_t *ticket) {
    if (!cy || !ticket || npts < 0 || npts > cy->max_points || (npts && !pts))
        return fail(VX_EINVAL, "bad argument (npts %lld of max %lld)", (long long)npts,
                    (long long)(cy ? cy->max_points : 0));
    const int b = cy->pf_next;
    cy->pf_next ^= 1;
    VX_CUDA(cudaStreamWaitEvent(cy->cst, cy->ev_used[b], 0));   // the tick that read slot b is past it
    if (npts) VX_CUDA(cudaMemcpyAsync(cy->d_pb[b], pts, (size_t)npts * 24, cudaMemcpyHostToDevice, cy->cst));
    VX_CUDA(cudaEventRecord(cy->ev_up[b], cy->cst));
    cy->pf_ticket[b] = ++cy->pf_issued;
    cy->pf_n[b] = npts;
    *ticket = cy->pf_ticket[b];
    return VX_OK;
}

extern "C" int vx_cycle_step_staged(vx_cycle *cy, uint64_t ticket, const double *link_T, float hit, double thr,
                                    const double *centers, int s, int sync) {
    if (!ticket) return fail(VX_EINVAL, "ticket 0 is never issued");
    return cycle_step(cy, nullptr, nullptr, 0, link_T, hit, thr, centers, s, sync, ticket);
}

extern "C" int vx_cycle_use_graph(vx_cycle *cy, int enable) {
    if (!cy) return fail(VX_EINVAL, "NULL cycle");
    VX_CUDA(cudaStreamSynchronize(cy->ctx->stream));
    cy->use_graph = enable != 0;
    return VX_OK;
}

extern "C" int vx_cycle_profile(vx_cycle *cy, int enable) {
    if (!cy) return fail(VX_EINVAL, "NULL cycle");
    VX_CUDA(cudaStreamSynchronize(cy->ctx->stream));
    cy->profiling = enable != 0;
    cy->ring_n = 0;
    return VX_OK;
}

extern "C" int vx_cycle_phase_ms(vx_cycle *cy, double *ms, int *nsteps) {
    if (!cy || !ms) return fail(VX_EINVAL, "NULL argument");
    VX_CUDA(cudaStreamSynchronize(cy->ctx->stream));
    for (int q = 0; q < VX_CYCLE_PHASES; ++q) ms[q] = 0.0;
    for (int r = 0; r < cy->ring_n; ++r)
        for (int q = 0; q < VX_CYCLE_PHASES; ++q) {
            float t = 0.f;
            VX_CUDA(cudaEventElapsedTime(&t, cy->ev[r][q], cy->ev[r][q + 1]));
            ms[q] += t;
        }
    if (cy->ring_n)
        for (int q = 0; q < VX_CYCLE_PHASES; ++q) ms[q] /= cy->ring_n;
    if (nsteps) *nsteps = cy->ring_n;
    return VX_OK;
}

extern "C" int vx_cycle_wait(vx_cycle *cy, vx_cycle_result *res, int32_t *lin, double *world, double *dist) {
    if (!cy) return fail(VX_EINVAL, "NULL cycle");
    VX_CUDA(cudaStreamSynchronize(cy->ctx->stream));
    // the tick packed its results into host-mapped memory (k_pack_results)
    const int s = cy->last_s;
    const unsigned char *o = cy->h_out;
    if (s && lin) std::memcpy(lin, o + 64, (size_t)2 * s * 4);
    const unsigned char *ow = o + 64 + (((size_t)2 * s * 4 + 7) & ~(size_t)7);
    if (s && world) std::memcpy(world, ow, (size_t)2 * s * 24);
    if (s && dist) std::memcpy(dist, ow + (size_t)2 * s * 24, (size_t)2 * s * 8);
    if (res) {
        const long long *h = reinterpret_cast<const long long *>(o);
        res->stats = vx_insert_stats{(int64_t)h[0], 0, (int64_t)h[1], (int64_t)h[2]};
        res->self_recomputed = cy->self_recomputed;
    }
    return VX_OK;
}

static void av_free(vx_cycle *cy) {
    cudaFree(cy->d_av_par);
    cudaFree(cy->d_av_link);
    cudaFree(cy->d_frames);
    cudaFreeHost(cy->h_frames);
    cudaFree(cy->d_J);
    cudaFree(cy->d_act);
    cudaFree(cy->d_ref);
    cudaFree(cy->d_val);
    cudaFree(cy->d_flag);
    cy->d_av_par = cy->d_frames = cy->h_frames = cy->d_J = cy->d_act = cy->d_ref = cy->d_val = nullptr;
    cy->d_av_link = cy->d_flag = nullptr;
    cy->av_s = cy->av_nj = 0;
}

extern "C" int vx_cycle_set_avoidance(vx_cycle *cy, int s, const double *radius, const double *buffer,
                                      const int32_t *link_index, int n_joints, double kappa,
                                      double x_star_offset) {
    if (!cy || s < 0 || s > cy->max_spheres || n_joints < 0 || (s && (!radius || !buffer || !link_index)))
        return fail(VX_EINVAL, "bad argument (spheres %d of max %d, joints %d)", s,
                    cy ? cy->max_spheres : 0, n_joints);
    for (int q = 0; q < s; ++q) {
        if (!(buffer[q] > 0)) return fail(VX_EINVAL, "buffer b must be > 0 (sphere %d)", q);
        if (link_index[q] < 0 || link_index[q] >= n_joints)
            return fail(VX_EINVAL, "link index %d out of range (sphere %d)", link_index[q], q);
    }
    if (!(kappa > 0)) return fail(VX_EINVAL, "kappa must be > 0");
    cudaStream_t st = cy->ctx->stream;
    VX_CUDA(cudaStreamSynchronize(st));
    av_free(cy);
    drop_graph(cy);
    if (!s) return VX_OK;
    const int nj = n_joints > 0 ? n_joints : 1;
    cudaError_t e = cudaMalloc(&cy->d_av_par, (size_t)2 * s * 8);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_av_link, (size_t)s * 4);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_frames, (size_t)nj * 48);
    if (e == cudaSuccess) e = cudaMallocHost(&cy->h_frames, (size_t)nj * 48);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_J, (size_t)2 * s * nj * 8);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_act, (size_t)2 * s * 8);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_ref, (size_t)2 * s * 8);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_val, (size_t)2 * s * 8);
    if (e == cudaSuccess) e = cudaMalloc(&cy->d_flag, (size_t)2 * s * 4);
    if (e != cudaSuccess) {
        av_free(cy);
        return cuda_fail(e, "cudaMalloc(avoidance)");
    }
    std::memset(cy->h_frames, 0, (size_t)nj * 48);
    VX_CUDA(cudaMemcpy(cy->d_av_par, radius, (size_t)s * 8, cudaMemcpyHostToDevice));
    VX_CUDA(cudaMemcpy(cy->d_av_par + s, buffer, (size_t)s * 8, cudaMemcpyHostToDevice));
    VX_CUDA(cudaMemcpy(cy->d_av_link, link_index, (size_t)s * 4, cudaMemcpyHostToDevice));
    cy->av_s = s;
    cy->av_nj = n_joints;
    cy->av_kappa = kappa;
    cy->av_offset = x_star_offset > 0 ? x_star_offset : -1.0;
    return VX_OK;
}

extern "C" int vx_cycle_set_joint_frames(vx_cycle *cy, const double *origins, const double *axes) {
    if (!cy || !cy->av_s) return fail(VX_EINVAL, "avoidance rows not enabled (vx_cycle_set_avoidance)");
    if (cy->av_nj && (!origins || !axes)) return fail(VX_EINVAL, "NULL joint frames");
    // the previous step's H2D reads h_frames: wait for it before overwriting
    VX_CUDA(cudaStreamSynchronize(cy->ctx->stream));
    std::memcpy(cy->h_frames, origins, (size_t)cy->av_nj * 24);
    std::memcpy(cy->h_frames + 3 * cy->av_nj, axes, (size_t)cy->av_nj * 24);
    return VX_OK;
}

extern "C" int vx_cycle_rows(vx_cycle *cy, double *J, double *act, double *ref, double *val, int32_t *flag) {
    if (!cy || !cy->av_s) return fail(VX_EINVAL, "avoidance rows not enabled (vx_cycle_set_avoidance)");
    if (cy->last_s != cy->av_s)
        return fail(VX_EINVAL, "last step had %d spheres, avoidance set for %d", cy->last_s, cy->av_s);
    cudaStream_t st = cy->ctx->stream;
    const size_t r = (size_t)2 * cy->av_s;
    if (J && cy->av_nj) VX_CUDA(cudaMemcpyAsync(J, cy->d_J, r * cy->av_nj * 8, cudaMemcpyDeviceToHost, st));
    if (act) VX_CUDA(cudaMemcpyAsync(act, cy->d_act, r * 8, cudaMemcpyDeviceToHost, st));
    if (ref) VX_CUDA(cudaMemcpyAsync(ref, cy->d_ref, r * 8, cudaMemcpyDeviceToHost, st));
    if (val) VX_CUDA(cudaMemcpyAsync(val, cy->d_val, r * 8, cudaMemcpyDeviceToHost, st));
    if (flag) VX_CUDA(cudaMemcpyAsync(flag, cy->d_flag, r * 4, cudaMemcpyDeviceToHost, st));
    VX_CUDA(cudaStreamSynchronize(st));
    return VX_OK;
}

extern "C" int vx_cycle_info(vx_cycle *cy, int32_t info[4]) {
    if (!cy || !info) return fail(VX_EINVAL, "NULL argument");
    VX_CUDA(cudaStreamSynchronize(cy->ctx->stream));
    info[0] = cy->p3_mode;
    info[1] = cy->last_graph;
    info[2] = cy->captures;
    info[3] = *(volatile int *)cy->h_m;
    return VX_OK;
}

extern "C" int vx_cycle_fields(vx_cycle *cy, vx_field **env, vx_field **self_field) {
    if (!cy) return fail(VX_EINVAL, "NULL cycle");
    if (env) *env = &cy->env_f;
    if (self_field) *self_field = &cy->self_f;
    return VX_OK;
}

extern "C" int vx_cycle_grids(vx_cycle *cy, vx_grid **env, vx_grid **self_grid, vx_grid **mask) {
    if (!cy) return fail(VX_EINVAL, "NULL cycle");
    if (env) *env = cy->env;
    if (self_grid) *self_grid = cy->self;
    if (mask) *mask = cy->mask;
    return VX_OK;
}
