// Internal declarations shared by the sm_100a kernels and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#define VX_FULL_MASK 0xffffffffu

// Checked builds (make EXTRA=-DVX_CHECK; tools/checked_suite.sh): device-side
// bounds and invariant assertions on the kernels' shared-memory and global
// index arithmetic; a violation prints its site and traps (the launch fails
// loudly).  Compiled out otherwise.
#ifdef VX_CHECK
#include <cstdio>
#define VX_ASSERT(cond, what)                                                             \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("VX_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                    \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define VX_ASSERT(cond, what) do {} while (0)
#endif

namespace vx {

// Launch configuration / layout decisions for one EDT problem.  Computed on
// the host from the grid shape; documented in DESIGN.md ("EDT kernels").
struct EdtPlan {
    int nx, ny, nz;
    int zb, yb, xb;        // bits(n-1) per axis: packing widths
    int wb;                // bits of the largest pass-3 weight (ny-1)^2 + (nz-1)^2
    bool s2_wide;          // pass-2 output as u64 (y<<32 | z) instead of u32 (y<<zb | z)
    bool e3_wide;          // pass-3 stack entries as u64
    bool fwide;            // int64 weights (F or 2*L^2 beyond int32; and the VX_FORCE_WIDE hooks)
    bool pwide;            // int32 weights, int64 hull-test products (2*F*L beyond int32: ~700-26k)
    int B2, W2;            // pass 2: bands per column, rows per band
    int B3, W3;            // pass 3
    bool gstack2, gstack3; // stack in global scratch (column longer than smem allows)
    bool tma2, tma3;       // input tile staged into shared memory by TMA
    int tw2, tw3;          // columns per TMA-staged tile (32; 16 for columns longer than 512)
    size_t smem2, smem3;   // dynamic smem bytes per CTA
    size_t s1_bytes, s2_bytes, gstack_bytes;  // scratch layout
    int gstack_ctas;       // persistent CTAs when a global stack is used
    bool s1_16;            // pass-1 output (line sites) as int16: pass 2 widens its TMA tiles
};

bool make_plan(int nx, int ny, int nz, EdtPlan *p, int force_global_stack);

// Slab-mode destination table for the fused pass-2 -> pass-3 exchange.
constexpr int kMaxRanks = 64;
struct ScatterTab {
    void *dst[kMaxRanks];           // per owner rank q: its (x_extent, nyl_q, nz) buffer
    int j_start[kMaxRanks + 1];     // rank q owns rows j_start[q] .. j_start[q+1]-1
    long long x_base;               // x index of this launch's first slice in dst
    int nranks;
};

// Occupied-slice list of a single-scene EDT (all device-side): pass 1 and
// pass 2 skip empty slices, pass 3 stages only occupied slices' rows.
struct SparseRows {
    const uint8_t *sflag;   // [nx] 1 if slice i holds an occupied voxel
    const int *xs;          // [nx] ascending occupied slice indices
    const int *hdr;         // hdr[0] = count
    int *m_mirror = nullptr;  // optional host-mapped copy of hdr[0] (the next call's hint)
    int p3_mode = 0;          // pass 3: 0 both kernels, gated on the device by the
                              // count; 1 one warp per tile only; 2 banded only
    int *fails = nullptr;     // windowed search header: fall-back counts, pass-1 k-line counts
    int nscenes = 1;
    int m_hint = -1;          // predicted count (>= 0: skip the windowed search when sparse)
};

// Pass launchers (stream-ordered, no host sync).  Return cudaError_t.
// nslices: number of (ny, nz) slices stacked along i (scenes * local nx).
// s16: int16 output (EdtPlan::s1_16; pass 2 of the same plan reads it)
cudaError_t launch_pass1(const uint8_t *occ, void *s1, long long nslices, int ny, int nz,
                         cudaStream_t st, const SparseRows *sp = nullptr, bool s16 = false);
cudaError_t launch_pass2(const int32_t *s1, void *s2, void *gstack, const EdtPlan &p,
                         long long nslices, cudaStream_t st, const SparseRows *sp = nullptr);
// pass 2 with the fused exchange epilogue (slab mode)
cudaError_t launch_pass2_scatter(const int32_t *s1, const ScatterTab &sc, void *gstack, const EdtPlan &p,
                                 long long nslices, cudaStream_t st, const SparseRows *sp = nullptr);
// pass 3 over nscenes buffers of shape (nx, nyl, nz) holding global rows
// j0 .. j0+nyl-1 (slab mode); site codes are global flat indices.
cudaError_t launch_pass3(const void *s2, int32_t *site, void *gstack, const EdtPlan &p,
                         int nscenes, int j0, int nyl, cudaStream_t st, const SparseRows *sp = nullptr);
// occupied-slice list: flags + compacted list (2 launches)
bool sparse_ok(const EdtPlan &p, int nscenes);
SparseRows sparse_rows_at(void *where, const EdtPlan &p, int nscenes = 1);
cudaError_t launch_slice_list(const uint8_t *occ, const EdtPlan &p, const SparseRows &sp, cudaStream_t st,
                              int nscenes = 1);
cudaError_t launch_slice_list_only(const EdtPlan &p, const SparseRows &sp, cudaStream_t st);
int pass3_mode_hint(const EdtPlan &p, int m);   // SparseRows::p3_mode from a predicted count
bool ring_hint_on(const EdtPlan &p, int m);     // would a call with this predicted count launch the windowed search?
struct DevCounters;
// same from a grid's touched list (valid when it covers every occupied voxel)
cudaError_t launch_slice_list_touched(const int32_t *touched, const DevCounters *ctr, const uint8_t *occ,
                                      const EdtPlan &p, const SparseRows &sp, cudaStream_t st);
size_t scratch_bytes_for(const EdtPlan &p, int nscenes);
// Full EDT: occ (device) -> site (device); scratch >= scratch_bytes_for(p, n).
cudaError_t edt_device(const uint8_t *occ, int32_t *site, void *scratch, const EdtPlan &p,
                       cudaStream_t st);
// Batched EDT over `nscenes` equally-shaped scenes laid out back to back.
cudaError_t edt_device_batched(const uint8_t *occ, int32_t *site, void *scratch,
                               const EdtPlan &p, int nscenes, cudaStream_t st);

// ---- map side -------------------------------------------------------------
struct GridGeom {
    int nx, ny, nz;
    double vs;
    double ox, oy, oz;
};

struct DevCounters {                // device-resident per-grid bookkeeping
    unsigned long long inserted, skipped, oob, stamped_oob;
    int touched;                    // entries in the touched (reset) list
    int pending;                    // new first-touch voxels of the current insert
    int overflow;                   // touched list overflowed -> dense reset
    int dirty;                      // occupancy changed since last EDT (memo)
    unsigned int done;              // blocks finished (last-block commit of reset/stamp/finalize)
};

struct ResetArgs {   // one grid's sparse (touched-list) or dense reset
    float *cells;
    uint8_t *occ;
    const int32_t *touched;
    DevCounters *ctr;
    long long n;
    int dense;
};
struct ZeroSpan {
    void *p;
    size_t bytes;
};
struct CopySpan {   // a small block copied by the reset launch (16-byte units)
    void *dst;
    const void *src;   // may be host-mapped pinned memory
    size_t bytes;
};
cudaError_t launch_reset2(const ResetArgs &a, const ResetArgs &b, ZeroSpan z0, ZeroSpan z1, ZeroSpan z2,
                          cudaStream_t st, CopySpan cp = CopySpan{nullptr, nullptr, 0});
cudaError_t launch_reset(float *cells, uint8_t *occ, int32_t *touched, DevCounters *ctr,
                         int64_t n, int capacity, bool dense, cudaStream_t st);
cudaError_t launch_dense_clip(float *cells, const uint32_t *counts, int64_t n,
                              const DevCounters *ctr, cudaStream_t st);
cudaError_t launch_scatter(const double *pts, int64_t npts, const int64_t *npts_dev,
                           GridGeom g, const float *mask_cells, float thr, uint32_t *counts,
                           int32_t *touched, DevCounters *ctr, int capacity,
                           cudaStream_t st, const uint8_t *keep = nullptr);
cudaError_t launch_finalize(float *cells, uint8_t *occ, uint32_t *counts, int32_t *touched,
                            DevCounters *ctr, int64_t n, int capacity, int64_t max_new,
                            float hit, float occ_thr, cudaStream_t st, bool fresh = false,
                            uint8_t *sflag = nullptr, long long plane = 0, int nx = 0,
                            int *xs = nullptr, int *hdr = nullptr, int *m_mirror = nullptr);
cudaError_t launch_stamp(const int32_t *ijk, const int64_t *offsets, int nsets,
                         const double *set_origin, const double *set_vs, const double *T,
                         GridGeom g, float *cells, uint8_t *occ, float value, float occ_thr,
                         int32_t *touched, DevCounters *ctr, unsigned long long *oob_per_set,
                         int capacity, int64_t total, cudaStream_t st);
cudaError_t launch_occupancy(const float *cells, uint8_t *out, int64_t n, float thr,
                             cudaStream_t st);
// occupancy-set digest {sum mix1, sum mix2, count}: from the touched list when
// use_list (and it did not overflow), else over all n voxels
cudaError_t launch_occ_digest(const uint8_t *occ, int64_t n, const int32_t *touched, const DevCounters *ctr,
                              bool use_list, unsigned long long *out, cudaStream_t st);

// ---- statistical outlier filter (grids.py:224-240) ---------------------------
size_t outlier_scratch_bytes(long long n);
cudaError_t cloud_bounds(const double *pts, long long n, double lo[3], double hi[3], void *scratch,
                         cudaStream_t st);
cudaError_t outlier_filter(const double *pts, long long n, int k, double stdm, const double lo[3],
                           const double hi[3], uint8_t *keep, unsigned long long *removed, void *scratch,
                           size_t scratch_bytes, cudaStream_t st);

// ---- query ----------------------------------------------------------------
// j0 / nyl: site holds rows j0 .. j0+nyl-1 (slab mode; -1 = all rows);
// centres in other rows get lin -2
cudaError_t launch_site_world(const int32_t *site, GridGeom g, const double *centers,
                              int s, int32_t *out_lin, double *out_world, double *out_dist,
                              cudaStream_t st, int j0 = 0, int nyl = -1);

// the tick's gather on both maps + the packed host-mapped result block
cudaError_t launch_gather_pack(const int32_t *site_env, const int32_t *site_self, GridGeom g,
                               const double *centers, int s, int32_t *lin, double *world, double *dist,
                               const DevCounters *ctr, unsigned char *out, cudaStream_t st);
// K7: obstacle / self avoidance rows from the K6 outputs of both maps
cudaError_t launch_avoidance_rows(const double *world, const double *dist, const int32_t *lin,
                                  const double *centers, int s, const double *radius, const double *buffer,
                                  const int *link, const double *origins, const double *axes, int nj,
                                  double kappa, double offset, double *J, double *act, double *ref,
                                  double *val, int *flag, cudaStream_t st);

// export formats (vx_export.cu)
cudaError_t launch_sq_distance(const int32_t *site, int nx, int ny, int nz, long long *out, cudaStream_t st);
size_t dump_scratch_bytes(int ny, int nz);
cudaError_t launch_dump_layout(const int32_t *site, int nx, int ny, int nz, void *scratch, cudaStream_t st);
const long long *dump_total_ptr(void *scratch, int ny, int nz);
cudaError_t launch_dump_write(const int32_t *site, int nx, int ny, int nz, const void *scratch, char *out,
                              cudaStream_t st);
size_t occ_scratch_bytes(long long n);
cudaError_t launch_occ_layout(const uint8_t *occ, long long n, void *scratch, cudaStream_t st);
const long long *occ_total_ptr(void *scratch, long long n);
cudaError_t launch_occ_write(const uint8_t *occ, long long n, int ny, int nz, const void *scratch,
                             long long *out, cudaStream_t st);
// brute_force_edt: sites (K,3) int64 in flat-index order -> site (lexicographic ties)
cudaError_t launch_brute_force(const long long *sites, long long nsites, int nx, int ny, int nz, int32_t *out,
                               cudaStream_t st);

int num_sms();

}  // namespace vx
