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

__global__ void k_site_world(const int32_t *__restrict__ site, GridGeom g,
                             const double *__restrict__ centers, int s,
                             int32_t *__restrict__ out_lin, double *__restrict__ out_world,
                             double *__restrict__ out_dist) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= s) return;
    const double cx = centers[3 * q], cy = centers[3 * q + 1], cz = centers[3 * q + 2];
    const long long i = clip_index(floor(__ddiv_rn(__dsub_rn(cx, g.ox), g.vs)), g.nx);
    const long long j = clip_index(floor(__ddiv_rn(__dsub_rn(cy, g.oy), g.vs)), g.ny);
    const long long k = clip_index(floor(__ddiv_rn(__dsub_rn(cz, g.oz), g.vs)), g.nz);
    const int32_t lin = site[(i * g.ny + j) * g.nz + k];
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

}  // namespace

cudaError_t launch_site_world(const int32_t *site, GridGeom g, const double *centers, int s,
                              int32_t *out_lin, double *out_world, double *out_dist,
                              cudaStream_t st) {
    if (s <= 0) return cudaSuccess;
    k_site_world<<<(s + 127) / 128, 128, 0, st>>>(site, g, centers, s, out_lin, out_world, out_dist);
    return cudaGetLastError();
}

}  // namespace vx
