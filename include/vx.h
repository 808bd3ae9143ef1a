/*
 * vx.h -- C ABI of libvx.so, the B200 (sm_100a) distance-map pipeline.
 *
 * Drop-in boundary for the reference package voxarm
 * (/root/reference/pkg/src/voxarm).  The reference has no FFI: its boundary is
 * the Python API exported by voxarm/__init__.py:16-37.  Each entry point
 * below replaces the reference function named beside it; the Python shim
 * paper_2407_02363_b200 (edt.py, grids.py, engine.py) binds them with ctypes
 * and re-exposes the reference's names, argument meanings and exceptions.
 * INTEGRATION.md shows the ctypes binding a voxarm maintainer would add.
 *
 * Conventions
 *   - Plain C types only.  Arrays are C-order (i, j, k) with k fastest and
 *     flat index (i*ny + j)*nz + k (edt.py:121, 417).
 *   - Host pointers are borrowed for the duration of the call.  Device memory
 *     belongs to the ctx / grid / field that allocated it.
 *   - Every call is ordered on the ctx's CUDA stream; calls that return host
 *     data synchronise that stream.  One ctx per host thread.
 *   - Return codes: VX_OK (0); VX_EINVAL -> ValueError; VX_ERANGE ->
 *     IndexError; VX_ENOMEM -> MemoryError; VX_ECUDA / VX_ENODEV ->
 *     RuntimeError(vx_last_error()).  There is no CPU fallback: without a
 *     CUDA device vx_ctx_create fails with VX_ENODEV.
 */
#ifndef VX_H
#define VX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_ABI_VERSION 2

enum {
    VX_OK = 0,
    VX_EINVAL = -22,
    VX_ERANGE = -34,
    VX_ENOMEM = -12,
    VX_ENODEV = -19,
    VX_ECUDA = -1000
};

typedef struct vx_ctx vx_ctx;
typedef struct vx_grid vx_grid;
typedef struct vx_field vx_field;
typedef struct vx_cycle vx_cycle;

/* grids.InsertStats (grids.py:91-96) */
typedef struct vx_insert_stats {
    int64_t inserted;
    int64_t outliers_removed;
    int64_t robot_skipped;
    int64_t out_of_bounds;
} vx_insert_stats;

int vx_abi_version(void);
const char *vx_last_error(void);

/* ---- context ----------------------------------------------------------- */
int vx_ctx_create(int device, vx_ctx **out);
int vx_ctx_destroy(vx_ctx *ctx);
int vx_ctx_stream(vx_ctx *ctx, void **stream_out);   /* the cudaStream_t */
int vx_ctx_synchronize(vx_ctx *ctx);
int vx_host_alloc(size_t bytes, void **out);         /* pinned host memory */
int vx_host_free(void *p);
/* kernels this library launched on the ctx since creation (bench evidence) */
int64_t vx_ctx_launches(const vx_ctx *ctx);

/* ---- grids.VoxelGrid (grids.py:99-217) ----------------------------------- */
/* VoxelGrid.__init__ (grids.py:107-118): dims > 0, voxel_size > 0,
 * nx*ny*nz < 2^31, else VX_EINVAL.  cells start at 0. */
int vx_grid_create(vx_ctx *ctx, int nx, int ny, int nz, double voxel_size,
                   const double origin[3], vx_grid **out);
int vx_grid_destroy(vx_grid *g);
/* VoxelGrid.clear (grids.py:146-147); sparse over the voxels written since the
 * last clear when that set is known, dense otherwise. */
int vx_grid_clear(vx_grid *g);
/* VoxelGrid.insert_point_cloud (grids.py:149-188) with k_neighbors = 0, on
 * WORLD points (PointCloud.world_points, grids.py:67-70, applied by the
 * caller).  robot_mask may be NULL; a mask of another geometry is
 * VX_EINVAL (grids.py:159-160).  stats->outliers_removed is left 0. */
int vx_grid_insert_points(vx_grid *g, const double *xyz, int64_t n, float hit_logodds,
                          double occupancy_threshold, const vx_grid *robot_mask,
                          vx_insert_stats *stats);
/* insert_point_cloud with the statistical outlier filter (grids.py:166-169,
 * 224-240) when k_neighbors > 0 (k_neighbors <= 31): exact kNN on the GPU
 * and numpy's summation order, so the survivors equal the reference's.
 * stats->outliers_removed is filled. */
int vx_grid_insert_points_ex(vx_grid *g, const double *xyz, int64_t n, float hit_logodds,
                             double occupancy_threshold, const vx_grid *robot_mask,
                             int k_neighbors, double std_multiplier, vx_insert_stats *stats);
/* statistical_outlier_filter (grids.py:224-240) alone: keep mask (1 = kept) */
int vx_outlier_mask(vx_ctx *ctx, const double *xyz, int64_t n, int k_neighbors,
                    double std_multiplier, uint8_t *keep_out, int64_t *removed);
/* Same, points already in device memory (stream-ordered, stats stay on the
 * device until vx_grid_last_stats). */
int vx_grid_insert_points_device(vx_grid *g, const double *d_xyz, int64_t n, float hit_logodds,
                                 double occupancy_threshold, const vx_grid *robot_mask);
int vx_grid_last_stats(vx_grid *g, vx_insert_stats *stats);
/* VoxelGrid.insert_voxel_set (grids.py:190-203) for nsets voxel sets at once:
 * set s has counts[s] indices ijk[s] (int32 K x 3), origin set_origins[3s..],
 * voxel size set_voxel_sizes[s], optional row-major 4x4 transforms[16s..]
 * (NULL = none).  Cells are set to `value` (L_MAX).  oob_out[s] receives the
 * out-of-grid count each reference call would return. */
int vx_grid_insert_voxel_sets(vx_grid *g, int nsets, const int32_t *const *ijk,
                              const int64_t *counts, const double *set_origins,
                              const double *set_voxel_sizes, const double *transforms,
                              float value, int64_t *oob_out);
int vx_grid_read_cells(vx_grid *g, float *host_out);           /* .cells */
int vx_grid_write_cells(vx_grid *g, const float *host_in);     /* .cells[...] = */
/* VoxelGrid.occupancy_mask (grids.py:207-208) as uint8 0/1 */
int vx_grid_occupancy(vx_grid *g, double threshold, uint8_t *host_out);
/* VoxelGrid.occupied_voxels (grids.py:210-212): np.argwhere of the mask,
 * (count,3) int64 in lexicographic order, compacted on the device.
 * host_out == NULL returns the count only; capacity (rows) < count fails
 * with VX_ERANGE and still sets *count. */
int vx_grid_occupied_voxels(vx_grid *g, double threshold, int64_t *host_out, int64_t capacity,
                            int64_t *count);

/* ---- edt (edt.py) --------------------------------------------------------- */
/* pba_edt (edt.py:466-484) of a host occupancy array (any nonzero byte is
 * occupied).  max extent 2^20 (edt.py:29, 459-460) else VX_EINVAL. */
int vx_edt(vx_ctx *ctx, const uint8_t *occ, int nx, int ny, int nz, double voxel_size,
           vx_field **out);
/* pba_edt(grid.occupancy_mask(threshold)) without leaving the device */
int vx_edt_grid(vx_grid *g, double threshold, vx_field **out);
/* line_nearest_sites (edt.py:444-452): pass 1 only, int32 out */
/* brute_force_edt (edt.py:487-508): exhaustive nearest site per voxel, ties
 * to the lexicographically smallest -- the reference's own test oracle, run on
 * the GPU (O(voxels x sites): grids up to ~48^3 as the reference intends). */
int vx_brute_force_edt(vx_ctx *ctx, const uint8_t *occupancy, int nx, int ny, int nz, vx_field **out);
/* A field to be filled by vx_edt_grid_into (pooled: no allocation per EDT). */
int vx_field_create(vx_ctx *ctx, int nx, int ny, int nz, vx_field **out);
/* pba_edt(grid.occupancy_mask(threshold)) into `field` (same dims), on the
 * device: the occupancy never leaves it.  Replaces the engine's per-tick
 * occupancy_mask -> pba_edt round trip (engine.py:259-268). */
int vx_edt_grid_into(vx_grid *g, double threshold, vx_field *field);
/* The engine's memo key (engine.py:259-268: blake2b of the occupancy mask)
 * as a device digest of the occupied-voxel set: O(touched voxels) when the
 * grid's touched list covers its occupancy, else one pass over it; equal
 * occupancy gives equal digests.  16 bytes cross the bus. */
int vx_grid_occupancy_digest(vx_grid *g, double threshold, uint64_t digest[2]);
/* _site_world (engine.py:212-221) for s centres on field a and (optionally)
 * field b in one round trip: lin/world/dist hold a's s results, then b's. */
int vx_fields_site_world(vx_field *a, vx_field *b, const double origin[3], double voxel_size,
                         const double *centers, int64_t s, int32_t *site_lin, double *site_world,
                         double *dist);
/* Slab mode: _site_world on this rank's j-slab d_site (device, (nx, nyl, nz),
 * rows j0 .. j0+nyl-1, global flat site indices); centres whose clipped row
 * lies outside the slab return site_lin -2 (another rank answers them). */
int vx_site_world_slab(vx_ctx *ctx, const int32_t *d_site, int nx, int ny, int nz, int j0, int nyl,
                       const double origin[3], double voxel_size, const double *centers, int64_t s,
                       int32_t *site_lin, double *site_world, double *dist);
/* Bytes this context's ABI calls have copied host->device [0] and
 * device->host [1] since it was created (evidence: no per-tick grid copy). */
int vx_ctx_transfer_bytes(const vx_ctx *ctx, int64_t out[2]);
int vx_line_nearest_sites(vx_ctx *ctx, const uint8_t *occ, int nx, int ny, int nz,
                          int32_t *s1_out);
int vx_field_destroy(vx_field *f);
int vx_field_dims(const vx_field *f, int dims[3]);
/* DistanceField.site (edt.py:106-111) */
int vx_field_read_site(vx_field *f, int32_t *host_out);
/* DistanceField.site[i,j,k]; VX_ERANGE outside the grid (edt.py:155-156) */
/* DistanceField.sq_distance_grid (edt.py:123-135): int64 squared voxel
 * distance, -1 where there is no site; out is host or (out_on_device) device */
int vx_field_sq_distance(vx_field *f, int64_t *out, int out_on_device);
/* DistanceField.dump_squared (edt.py:137-145): the golden text, formatted on
 * the device.  buf == NULL returns the byte count only; capacity < count
 * fails with VX_ERANGE and still sets *nbytes.  No terminating NUL. */
int vx_field_dump_squared(vx_field *f, char *buf, int64_t capacity, int64_t *nbytes);
int vx_field_site_at(vx_field *f, int64_t i, int64_t j, int64_t k, int32_t *out);
/* SimEngine._site_world (engine.py:212-221) for s centres, plus the
 * distance of tasks.py:102-104.  site_lin[q] = -1 (world NaN, dist +inf)
 * where the reference returns None. */
int vx_field_site_world(vx_field *f, const double origin[3], double voxel_size,
                        const double *centers, int64_t s, int32_t *site_lin,
                        double *site_world, double *dist);

/* ---- device-pointer entry points (stream-ordered, no sync) --------------- */
size_t vx_edt_scratch_bytes(int nx, int ny, int nz, int nscenes);
/* nscenes grids of (nx,ny,nz) back to back; site codes are per-scene flat */
int vx_edt_device(vx_ctx *ctx, const uint8_t *d_occ, int nx, int ny, int nz, int nscenes,
                  int32_t *d_site, void *d_scratch, size_t scratch_bytes);
/* slab mode: passes 1+2 on nxl local i-slices of a grid with
 * global dims (nx,ny,nz); d_s2 receives the pass-2 codes (4 bytes/voxel
 * unless vx_edt_s2_bytes() says 8). */
int vx_edt_s2_bytes(int nx, int ny, int nz);
int vx_edt_pass12_device(vx_ctx *ctx, const uint8_t *d_occ, int nx, int ny, int nz, int nxl,
                         void *d_s2, void *d_scratch, size_t scratch_bytes);
/* slab mode with the exchange fused into pass 2's epilogue: the pass-2 code
 * of row j of local slice i is stored straight into the pass-3 input of the
 * rank q owning j (j_starts[q] <= j < j_starts[q+1], j_starts[0] = 0,
 * j_starts[nranks] = ny): dst[q] + ((x_base + i) * nyl_q + j - j_starts[q])
 * * nz + k.  dst[q] is a device pointer: a peer's buffer mapped over NVLink
 * (x_base = this rank's first global i, buffer (nx, nyl_q, nz)), or this
 * rank's all-to-all send block for q (x_base = 0, block (nxl, nyl_q, nz)).
 * nranks <= 64. */
int vx_edt_pass12_scatter(vx_ctx *ctx, const uint8_t *d_occ, int nx, int ny, int nz, int nxl,
                          int nranks, void *const *dst, const int *j_starts, long long x_base,
                          void *d_scratch, size_t scratch_bytes);
/* pass 3 over a j-slab: d_s2 holds (nx, nyl, nz) codes for global rows
 * j0..j0+nyl-1; d_site receives global flat indices, shape (nx, nyl, nz). */
int vx_edt_pass3_device(vx_ctx *ctx, const void *d_s2, int nx, int ny, int nz, int j0, int nyl,
                        int32_t *d_site, void *d_scratch, size_t scratch_bytes);

/* ---- one camera tick of SimEngine.step (engine.py:233-280) ---------------
 * clear env/self/mask, stamp self-obstacle links into self and all links
 * into mask (engine.py:243-248), scatter the cloud into env with the robot
 * mask (249-254), EDT of env and (when its voxel set changed, engine.py:259-
 * 268) of self, and the per-sphere gather for both maps (272-280). */
typedef struct vx_cycle_result {
    vx_insert_stats stats;
    int32_t self_recomputed;   /* 1 when the self field was rebuilt */
} vx_cycle_result;

int vx_cycle_create(vx_ctx *ctx, int nx, int ny, int nz, double voxel_size,
                    const double origin[3], int nlinks, const int32_t *const *link_ijk,
                    const int64_t *link_counts, const double *link_origins,
                    double link_voxel_size, const int32_t *self_links, int n_self_links,
                    int64_t max_points, int max_spheres, vx_cycle **out);
int vx_cycle_destroy(vx_cycle *c);
/* pts: host world points (pinned for async H2D), link_T: nlinks row-major
 * 4x4 FK frames, centers: s sphere centres.  Outputs (host, may be NULL):
 * per sphere and map (env then self) the site flat index, world point and
 * distance.  sync=0 leaves results in flight (read with vx_cycle_wait). */
int vx_cycle_step(vx_cycle *c, const double *pts, int64_t npts, const double *link_T,
                  float hit_logodds, double occupancy_threshold, const double *centers,
                  int s, int sync);
/* same tick with the cloud already in device memory (d_pts, npts points;
 * it must stay valid until the tick has run); frames and centres are host
 * arrays (a few hundred bytes), copied into a pinned staging block at the call */
int vx_cycle_step_device(vx_cycle *c, const double *d_pts, int64_t npts, const double *link_T,
                         float hit_logodds, double occupancy_threshold, const double *centers,
                         int s, int sync);
/* Stage a later tick's cloud (pinned host memory, npts points) on a copy
 * stream while the current tick computes, and return a ticket (> 0) naming
 * the staged copy.  vx_cycle_step_staged(ticket) runs a tick on exactly that
 * copy; the host buffer may be rewritten once that tick has completed
 * (vx_cycle_wait), since the upload itself is asynchronous.  Two
 * slots: a third prefetch overwrites the oldest unconsumed slot, and a
 * consumed or overwritten ticket fails with VX_EINVAL (never a stale cloud).
 * vx_cycle_step never reads a staged copy. */
int vx_cycle_prefetch(vx_cycle *c, const double *pts, int64_t npts, uint64_t *ticket);
int vx_cycle_step_staged(vx_cycle *c, uint64_t ticket, const double *link_T, float hit_logodds,
                         double occupancy_threshold, const double *centers, int s, int sync);
/* wait for the last step and copy its results (the tick already packed them
 * into host-mapped memory); any output may be NULL */
int vx_cycle_wait(vx_cycle *c, vx_cycle_result *res, int32_t *site_lin /* 2*s */,
                  double *site_world /* 2*s*3 */, double *dist /* 2*s */);
/* How the last tick ran (tests and bench evidence), after waiting for it:
 * info[0] pass-3 kernel choice (0 both launched, the device picks; 1 the
 * one-warp streaming kernel; 2 the banded kernel), info[1] 1 if it replayed
 * the CUDA graph, info[2] graph captures so far, info[3] the env map's
 * occupied i-slice count written by that tick (-1 before the first). */
int vx_cycle_info(vx_cycle *c, int32_t info[4]);
/* Per-phase CUDA-event timing of vx_cycle_step (bench evidence).  Phases:
 * 0 H2D, 1 self map (stamp + EDT, only when it changed), 2 mask stamp +
 * env/mask reset, 3 scatter + finalize, 4 EDT pass 1, 5 pass 2, 6 pass 3,
 * 7 sphere gather.  vx_cycle_profile(c, 1) resets and enables; phase_ms
 * returns the mean over the profiled steps (up to 64). */
#define VX_CYCLE_PHASES 8
/* Replay the per-tick kernel sequence as one CUDA graph (default on; the
 * profiled steps always launch directly so the phase events can be recorded). */
int vx_cycle_use_graph(vx_cycle *c, int enable);
int vx_cycle_profile(vx_cycle *c, int enable);
int vx_cycle_phase_ms(vx_cycle *c, double *ms, int *nsteps);
/* Avoidance rows on the device (tasks.py:88-123 _distance_rows, fused after
 * the gather of every step with s == the configured sphere count).  Per
 * sphere: radius, buffer (> 0), link index (< n_joints); kappa > 0;
 * x_star_offset <= 0 means 2*buffer (tasks.py:63-73).  Re-configuring drops
 * the captured graph; s = 0 disables. */
int vx_cycle_set_avoidance(vx_cycle *c, int s, const double *radius, const double *buffer,
                           const int32_t *link_index, int n_joints, double kappa,
                           double x_star_offset);
/* joint frames at this step's q (robot.py:545-558): n_joints world origins
 * and axes, each n_joints*3 row-major; set before vx_cycle_step */
int vx_cycle_set_joint_frames(vx_cycle *c, const double *origins, const double *axes);
/* rows of the last step, env then self (2*s rows): J (2*s x n_joints),
 * activation, xdot_ref, value (|O - C|, inf when no site), flag (0 no site /
 * inert row, 1 built, 2 x <= 1e-12: activation 1, J zero -- the caller
 * applies its held direction, tasks.py:111-119).  Any output may be NULL. */
int vx_cycle_rows(vx_cycle *c, double *J, double *activation, double *xdot_ref, double *value,
                  int32_t *flag);
/* fields of the last step (owned by the cycle; do not destroy) */
int vx_cycle_fields(vx_cycle *c, vx_field **env, vx_field **self_field);
int vx_cycle_grids(vx_cycle *c, vx_grid **env, vx_grid **self_grid, vx_grid **mask);

#ifdef __cplusplus
}
#endif
#endif /* VX_H */
