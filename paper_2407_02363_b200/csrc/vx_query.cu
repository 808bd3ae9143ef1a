// K6: per-sphere nearest-obstacle gather.
//
// SimEngine._site_world (voxarm engine.py:212-221) for every bounding-sphere
// centre at once, plus the distance x = ||O - C|| that tasks.py:102-104
// computes from it:
//   idx  = clip(floor((c - origin) / vs), 0, dims - 1)      (engine.py:217-218)
//   site = field.site[idx]; None when NO_SITE               (engine.py:219-221)
//   O    = origin + (site_index + 0.5) * vs                  (engine.py:221)
// One thread per centre; the site lookup is the only grid access.
#include "vx_internal.cuh"

#include <math.h>
#include <math_constants.h>
#include <climits>

namespace vx {
namespace {

__device__ __forceinline__ long long clip_index(double f, int n) {
    // numpy: floor(...).astype(int64) then clip; out-of-range floats cast to
    // INT64_MIN (x86 cvttsd2si), which the clip maps to 0
    long long v;
    if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0)) v = LLONG_MIN;
    else v = (long long)f;
    if (v < 0) v = 0;
    if (v > n - 1) v = n - 1;
    return v;
}

// j0 / nyl: the site array holds rows j0 .. j0 + nyl - 1 of every slice (a
// slab-mode j-slab, global flat indices); a centre whose row is not held
// gets lin = -2 (another rank owns it)
__device__ __forceinline__ void site_world_one(const int32_t *__restrict__ site, const GridGeom &g,
                                               const double *__restrict__ centers, int q, int32_t *out_lin,
                                               double *out_world, double *out_dist, int j0 = 0, int nyl = -1) {
    const double cx = centers[3 * q], cy = centers[3 * q + 1], cz = centers[3 * q + 2];
    const long long i = clip_index(floor(__ddiv_rn(__dsub_rn(cx, g.ox), g.vs)), g.nx);
    const long long j = clip_index(floor(__ddiv_rn(__dsub_rn(cy, g.oy), g.vs)), g.ny);
    const long long k = clip_index(floor(__ddiv_rn(__dsub_rn(cz, g.oz), g.vs)), g.nz);
    if (nyl < 0) nyl = g.ny;
    if (j < j0 || j >= (long long)j0 + nyl) {
        out_lin[q] = -2;
        out_world[3 * q] = out_world[3 * q + 1] = out_world[3 * q + 2] = CUDART_NAN;
        out_dist[q] = CUDART_NAN;
        return;
    }
    const int32_t lin = site[(i * nyl + (j - j0)) * g.nz + k];
    out_lin[q] = lin;
    if (lin < 0) {
        out_world[3 * q] = out_world[3 * q + 1] = out_world[3 * q + 2] = CUDART_NAN;
        out_dist[q] = CUDART_INF;
        return;
    }
    const long long plane = (long long)g.ny * g.nz;
    const long long si = lin / plane, sj = (lin / g.nz) % g.ny, sk = lin % g.nz;
    const double ox = __dadd_rn(g.ox, __dmul_rn(__dadd_rn((double)si, 0.5), g.vs));
    const double oy = __dadd_rn(g.oy, __dmul_rn(__dadd_rn((double)sj, 0.5), g.vs));
    const double oz = __dadd_rn(g.oz, __dmul_rn(__dadd_rn((double)sk, 0.5), g.vs));
    out_world[3 * q] = ox;
    out_world[3 * q + 1] = oy;
    out_world[3 * q + 2] = oz;
    const double dx = ox - cx, dy = oy - cy, dz = oz - cz;
    out_dist[q] = sqrt(dx * dx + dy * dy + dz * dz);
}

__global__ void k_site_world(const int32_t *__restrict__ site, GridGeom g,
                             const double *__restrict__ centers, int s,
                             int32_t *__restrict__ out_lin, double *__restrict__ out_world,
                             double *__restrict__ out_dist, int j0, int nyl) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= s) return;
    site_world_one(site, g, centers, q, out_lin, out_world, out_dist, j0, nyl);
}

// the camera tick's gather: both maps in one launch (row r = map * s +
// sphere), device copies for the avoidance rows, and the packed host-mapped
// result block {inserted, skipped, oob | lin[2s] | world[2s*3] | dist[2s]}
__global__ void k_gather_pack(const int32_t *__restrict__ site_env, const int32_t *__restrict__ site_self,
                              GridGeom g, const double *__restrict__ centers, int s,
                              int32_t *__restrict__ lin, double *__restrict__ world, double *__restrict__ dist,
                              const DevCounters *__restrict__ ctr, unsigned char *__restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r == 0) {
        long long *hdr = reinterpret_cast<long long *>(out);
        hdr[0] = (long long)ctr->inserted;
        hdr[1] = (long long)ctr->skipped;
        hdr[2] = (long long)ctr->oob;
    }
    if (r >= 2 * s) return;
    const int m = r >= s ? 1 : 0, q = r - m * s;
    site_world_one(m ? site_self : site_env, g, centers, q, lin + m * s, world + 3 * m * s, dist + m * s);
    int32_t *ol = reinterpret_cast<int32_t *>(out + 64);
    double *ow = reinterpret_cast<double *>(out + 64 + (((size_t)2 * s * 4 + 7) & ~(size_t)7));
    double *od = ow + (size_t)6 * s;
    ol[r] = lin[r];
    ow[3 * r] = world[3 * r];
    ow[3 * r + 1] = world[3 * r + 1];
    ow[3 * r + 2] = world[3 * r + 2];
    od[r] = dist[r];
}

}  // namespace

cudaError_t launch_gather_pack(const int32_t *site_env, const int32_t *site_self, GridGeom g,
                               const double *centers, int s, int32_t *lin, double *world, double *dist,
                               const DevCounters *ctr, unsigned char *out, cudaStream_t st) {
    k_gather_pack<<<(2 * s + 127) / 128 + (s ? 0 : 1), 128, 0, st>>>(site_env, site_self, g, centers, s, lin,
                                                                     world, dist, ctr, out);
    return cudaGetLastError();
}

cudaError_t launch_site_world(const int32_t *site, GridGeom g, const double *centers, int s,
                              int32_t *out_lin, double *out_world, double *out_dist,
                              cudaStream_t st, int j0, int nyl) {
    if (s <= 0) return cudaSuccess;
    k_site_world<<<(s + 127) / 128, 128, 0, st>>>(site, g, centers, s, out_lin, out_world, out_dist, j0, nyl);
    return cudaGetLastError();
}

}  // namespace vx

// ---------------------------------------------------------------------------
// K7: avoidance rows, the consumer of K6 fused on the
// device: voxarm tasks.py:88-123 (_distance_rows) per sphere and map --
//   x = |O - C|, act = activation_sigmoid(x, r, b) (tasks.py:21-32),
//   ref = kappa * (r + offset - x), offset = cfg or 2b,
//   J_row = (-(O - C)/x) . position_jacobian(q, link, C)   (robot.py:560-578:
//   column j <= link is axis_j x (C - origin_j)).
// flag: 0 no site (inert row), 1 row built, 2 x <= 1e-12 (the host applies
// the held-direction rule of tasks.py:111-119).
// ---------------------------------------------------------------------------
namespace vx {
namespace {

__global__ void k_avoidance_rows(const double *__restrict__ world, const double *__restrict__ dist,
                                 const int32_t *__restrict__ lin, const double *__restrict__ centers,
                                 int s, const double *__restrict__ radius, const double *__restrict__ buffer,
                                 const int *__restrict__ link, const double *__restrict__ origins,
                                 const double *__restrict__ axes, int nj, double kappa, double offset,
                                 double *__restrict__ J, double *__restrict__ act, double *__restrict__ ref,
                                 double *__restrict__ val, int *__restrict__ flag) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;   // row = map * s + sphere
    if (r >= 2 * s) return;
    const int q = r % s;
    double *Jr = J + (size_t)r * nj;
    for (int j = 0; j < nj; ++j) Jr[j] = 0.0;
    if (lin[r] < 0) {   // no site: inert row (tasks.py:100-101)
        act[r] = 0.0;
        ref[r] = 0.0;
        val[r] = CUDART_INF;
        flag[r] = 0;
        return;
    }
    const double c[3] = {centers[3 * q], centers[3 * q + 1], centers[3 * q + 2]};
    const double d[3] = {world[3 * r] - c[0], world[3 * r + 1] - c[1], world[3 * r + 2] - c[2]};
    const double x = dist[r];
    const double rad = radius[q], b = buffer[q];
    val[r] = x;
    double a;
    if (x <= rad) a = 1.0;
    else if (x >= rad + b) a = 0.0;
    else a = 0.5 * (cos((x - rad) * CUDART_PI / b) + 1.0);
    const double off = offset >= 0.0 ? offset : 2.0 * b;
    ref[r] = kappa * (rad + off - x);
    if (!(x > 1e-12)) {
        act[r] = 1.0;
        flag[r] = 2;
        return;
    }
    act[r] = a;
    flag[r] = 1;
    const double u[3] = {-d[0] / x, -d[1] / x, -d[2] / x};
    const int kmax = min(link[q] + 1, nj);
    for (int j = 0; j < kmax; ++j) {
        const double *o = origins + 3 * j, *ax = axes + 3 * j;
        const double rx = c[0] - o[0], ry = c[1] - o[1], rz = c[2] - o[2];
        const double cx = ax[1] * rz - ax[2] * ry;
        const double cy = ax[2] * rx - ax[0] * rz;
        const double cz = ax[0] * ry - ax[1] * rx;
        Jr[j] = u[0] * cx + u[1] * cy + u[2] * cz;
    }
}

}  // namespace

cudaError_t launch_avoidance_rows(const double *world, const double *dist, const int32_t *lin,
                                  const double *centers, int s, const double *radius, const double *buffer,
                                  const int *link, const double *origins, const double *axes, int nj,
                                  double kappa, double offset, double *J, double *act, double *ref,
                                  double *val, int *flag, cudaStream_t st) {
    if (s <= 0) return cudaSuccess;
    k_avoidance_rows<<<(2 * s + 63) / 64, 64, 0, st>>>(world, dist, lin, centers, s, radius, buffer, link,
                                                      origins, axes, nj, kappa, offset, J, act, ref, val,
                                                      flag);
    return cudaGetLastError();
}

}  // namespace vx
