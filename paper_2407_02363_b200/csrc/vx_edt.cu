// Exact 3D EDT with nearest-site index on sm_100a: three separable passes.
//
// Reference algorithm: voxarm edt.py (pkg/src/voxarm/edt.py)
//   pass 1  _sweep_lines       edt.py:168-224  -> k_pass1_*      (K3)
//   pass 2  _slice_transform   edt.py:227-317  -> k_column<2>    (K4)
//   pass 3  _column_transform  edt.py:320-420  -> k_column<3>    (K5)
//
// The output is bit-identical to the reference `site` array.  The
// reference's passes select, for every voxel, the lexicographically smallest
// nearest occupied voxel (ties: lower k in pass 1 edt.py:221; pop-on->= in the
// stacks edt.py:267-268; strict < in the query walk edt.py:311).  These
// kernels keep the same pass order and the same integer comparisons:
//   * pass 1: per line nearest occupied k, ties to the lower k;
//   * passes 2/3: the stack of edt.py is the strict lower convex hull of the
//     points (row, w + row^2).  That hull is unique, so building it as 32-row
//     band hulls merged pairwise by bridge walks (all with the >= dominance
//     test of edt.py:267) yields the same stack; each query then takes the
//     FIRST hull vertex minimising (y - y_p)^2 + w_p, which is what the
//     strict-< walk of edt.py:300-317 returns.
//
// Layout (C order, k fastest, flat index (i*ny + j)*nz + k as edt.py:417):
//   occ  u8  N   -> s1  i32 N (nearest k or -1)
//   s1   i32 N   -> s2  u32 N (y << zb | z, all-ones = none)   [u64 if wide]
//   s2   u32 N   -> site i32 N (flat index, -1 = none)
// Pass 1 is one warp per k-line with 16-byte vector I/O and warp scans.
// Passes 2/3: a CTA owns 32 consecutive k columns (one warp = 32 columns, so
// every global load/store is a 128-byte coalesced row segment) and B bands
// along the column (one warp per band).  Band stacks live in shared memory,
// laid out [row][32 columns] so each lane owns one bank.
#include "vx_internal.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>
#include <mutex>
#include <set>
#include <utility>
#include <cstdlib>

namespace vx {
namespace {

constexpr int BIG = 0x7fffffff;

#ifdef VX_PHASE_TIMING   // tools/phase_timing.cu: per-CTA phase timestamps
__device__ unsigned long long *g_phase_buf = nullptr;
#define VX_PT(i)                                                                       \
    do {                                                                               \
        if (threadIdx.x == 0 && threadIdx.y == 0 && g_phase_buf)                       \
            g_phase_buf[(size_t)blockIdx.x * 8 + (i)] = clock64();                     \
    } while (0)
#define VX_PTW(slot, i)                                                                \
    do {                                                                               \
        if ((threadIdx.x & 31) == 0 && g_phase_buf)                                   \
            g_phase_buf[(size_t)(slot) * 8 + (i)] = clock64();                         \
    } while (0)
#else
#define VX_PT(i) do {} while (0)
#define VX_PTW(slot, i) do {} while (0)
#endif
// column passes: at most 16 bands (512 threads) per CTA, 3 CTAs per SM
#ifndef VX_MAX_BANDS
#define VX_MAX_BANDS 16
#endif
constexpr int kMaxBands = VX_MAX_BANDS;
constexpr int kColThreads = 32 * kMaxBands;
// pass-3 narrow stack entries: 1 = (x, w) (F is one IMAD; the winner's site
// code is re-read from L2), 0 = (x, sy, sz) (F decodes; no re-read)
#ifndef VX_P3_XW
#define VX_P3_XW 1
#endif
constexpr bool kP3XW = VX_P3_XW != 0;
#ifndef VX_CMP_GROUP_ROWS
#define VX_CMP_GROUP_ROWS 24   // target candidates per group in compact pass 3
#endif
#ifndef VX_P2_REVERSE
#define VX_P2_REVERSE 1
#endif
#ifndef VX_P2_EVICT_FIRST
#define VX_P2_EVICT_FIRST 0
#endif
#ifndef VX_STREAM_CAP
#define VX_STREAM_CAP 63   // shared-memory stack entries per column (k_pass3_stream; 28 warps x 63 x 128 B)
#endif
#ifndef VX_STREAM_U
#define VX_STREAM_U 16
#endif
#ifndef VX_P3S_WPF
#define VX_P3S_WPF 1    // k_pass3_stream walk: the vertex after the successor loaded a switch ahead
#endif
#ifndef VX_P3S_DYN
#define VX_P3S_DYN 1    // k_pass3_stream: tiles after the first from an atomic counter
#endif
#ifndef VX_P3S_ENDS
#define VX_P3S_ENDS 1   // k_pass3_stream: store-only rows before the warp's first and after its last switch
#endif
#ifndef VX_STREAM_MAX_ROWS
#define VX_STREAM_MAX_ROWS 256   // occupied slices up to which pass 3 runs one warp per tile
#endif
constexpr int kStreamMaxRows = VX_STREAM_MAX_ROWS;
#ifndef VX_BAND_ROWS
#define VX_BAND_ROWS 32   // target rows per band
#endif
#ifndef VX_P1_WAVES
#define VX_P1_WAVES 1   // pass 1 over occupied slices: persistent CTAs per SM / 8
#endif
#ifndef VX_P1_X16
#define VX_P1_X16 1     // pass 1 with 16 voxels per lane for 256 < nz <= 1024 (nz % 16 == 0)
#endif
#ifndef VX_P1_LPW512
#define VX_P1_LPW512 1  // lines per warp iteration for nz <= 512 (occupied-slice path)
#endif
#ifndef VX_COL_MIN_BLOCKS
#define VX_COL_MIN_BLOCKS 2
#endif
#ifndef VX_COL_WALK_UNROLL
#define VX_COL_WALK_UNROLL 4   // phase-D rows per loop trip in the banded column kernels
#endif
constexpr int kColWalkUnroll = VX_COL_WALK_UNROLL;

constexpr int kColMinBlocks = VX_COL_MIN_BLOCKS;

// bit e (e = 0..3) set iff byte e of w is non-zero
__device__ __forceinline__ uint32_t nibble4(uint32_t w) {
    const uint32_t t = __vcmpne4(w, 0u);
    return (((t & 0x01010101u) * 0x01020408u) >> 24) & 0xfu;
}

__device__ __forceinline__ int pick(int k, int l, int r) {
    // edt.py:217-224: l if k-l <= r-k (ties -> lower k)
    if (l < 0) return r == BIG ? -1 : r;
    if (r == BIG) return l;
    return (k - l <= r - k) ? l : r;
}

__device__ __forceinline__ uint32_t pack16(int a, int b) {
    return (uint32_t)(uint16_t)a | ((uint32_t)(uint16_t)b << 16);
}

// s1 element type: int32, or int16 when pass 2 stages its tiles by TMA
// (EdtPlan::s1_16; pass 2 widens them in registers).  Four consecutive values
// stored at 4-element unit q: one 16-byte (int32) or 8-byte (int16) store.
template <typename T>
__device__ __forceinline__ void store4(T *line, int q, int a, int b, int c, int d) {
    if constexpr (sizeof(T) == 4) {
        reinterpret_cast<int4 *>(line)[q] = make_int4(a, b, c, d);
    } else {
        reinterpret_cast<uint2 *>(line)[q] = make_uint2(pack16(a, b), pack16(c, d));
    }
}

// ---------------------------------------------------------------------------
// Pass 1, vector path: nz % 4 == 0, nz <= 128 * CMAX.  One warp per line;
// lane owns 4 consecutive voxels of each 128-voxel chunk.
// ---------------------------------------------------------------------------
template <int CMAX, typename T>
__device__ __forceinline__ void pass1_line(const uint32_t (&nib)[CMAX], T *__restrict__ dst, int nq,
                                           int lane) {
    // The nearest occupied k before / after this lane's 4 voxels comes from
    // the nearest lane holding any site: a ballot names the lanes with sites,
    // __fls / __ffs of its masked bits picks the neighbour lane, and one
    // shuffle reads that lane's nibble (instead of 5-step prefix scans).
    const unsigned lt = (1u << lane) - 1u;
    const unsigned gt = lane == 31 ? 0u : ~((2u << lane) - 1u);
    unsigned m[CMAX];
#pragma unroll
    for (int c = 0; c < CMAX; ++c) m[c] = __ballot_sync(VX_FULL_MASK, nib[c] != 0u);
    // warp-uniform carries: last site before chunk c, first site after it
    int lastc[CMAX], firstc[CMAX];
    int run = -1;
#pragma unroll
    for (int c = 0; c < CMAX; ++c) {
        lastc[c] = run;
        const int hl = m[c] ? 31 - __clz(m[c]) : 0;
        const uint32_t nb = __shfl_sync(VX_FULL_MASK, nib[c], hl);
        if (m[c]) run = (c * 32 + hl) * 4 + 31 - __clz(nb);
    }
    run = BIG;
#pragma unroll
    for (int c = CMAX - 1; c >= 0; --c) {
        firstc[c] = run;
        const int ll = m[c] ? __ffs(m[c]) - 1 : 0;
        const uint32_t nb = __shfl_sync(VX_FULL_MASK, nib[c], ll);
        if (m[c]) run = (c * 32 + ll) * 4 + __ffs(nb) - 1;
    }
#pragma unroll
    for (int c = 0; c < CMAX; ++c) {
        const int q = c * 32 + lane;
        const int base = q * 4;
        const uint32_t nb = nib[c];
        const unsigned pm = m[c] & lt, nm = m[c] & gt;
        const int lp = pm ? 31 - __clz(pm) : 0, ln = nm ? __ffs(nm) - 1 : 0;
        const uint32_t nbp = __shfl_sync(VX_FULL_MASK, nb, lp);
        const uint32_t nbn = __shfl_sync(VX_FULL_MASK, nb, ln);
        const int exl = pm ? (c * 32 + lp) * 4 + 31 - __clz(nbp) : lastc[c];   // last site < base
        const int exr = nm ? (c * 32 + ln) * 4 + __ffs(nbn) - 1 : firstc[c];   // first site > base + 3
        int lv[4];
        int r = exl;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if ((nb >> e) & 1u) r = base + e;
            lv[e] = r;
        }
        int o[4];
        r = exr;
#pragma unroll
        for (int e = 3; e >= 0; --e) {
            if ((nb >> e) & 1u) r = base + e;
            o[e] = pick(base + e, lv[e], r);
        }
        if (q < nq) store4(dst, q, o[0], o[1], o[2], o[3]);
    }
}

// LPW lines per warp: all their loads are issued before any line is scanned
// (memory-level parallelism for the streaming read).
template <int CMAX, int LPW, typename T>
__global__ void __launch_bounds__(256) k_pass1_v4(const uint8_t *__restrict__ occ,
                                                  T *__restrict__ s1,
                                                  long long nlines, int nz,
                                                  const uint8_t *__restrict__ sflag, int ny,
                                                  const int *__restrict__ xs, const int *__restrict__ hdr,
                                                  int *__restrict__ linestat) {
    const int lane = threadIdx.x & 31;
    const int nq = nz >> 2;
    int nempty = 0, nseen = 0;   // k-lines without a site / processed (the windowed search's gate)
    uint32_t nib[LPW][CMAX];
    bool act[LPW];
    long long lines[LPW];
    const int m = xs ? __ldg(hdr) : 0;
    // the occupied-slice path runs a persistent grid over the m * ny lines
    // (m is read here); the dense path's grid covers every line once
    const long long total = xs ? (long long)m * ny : nlines;
    const long long wstep = (long long)gridDim.x * (blockDim.x >> 5) * LPW;
    for (long long line0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * LPW; line0 < total;
         line0 += wstep) {
#pragma unroll
    for (int l = 0; l < LPW; ++l) {
        long long line = line0 + l;
        // warp-uniform; empty slices are skipped (nothing downstream reads them)
        if (xs) {   // lines of occupied slices, slot-major
            const uint32_t slot = (uint32_t)line / (uint32_t)ny;
            act[l] = line < total;
            if (act[l]) line = (long long)__ldg(xs + slot) * ny + (line - (long long)slot * ny);
        } else {
            act[l] = line < nlines && (!sflag || sflag[(uint32_t)line / (uint32_t)ny]);
        }
        lines[l] = line;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(occ + line * nz);
#pragma unroll
        for (int c = 0; c < CMAX; ++c) {
            const int q = c * 32 + lane;
            nib[l][c] = nibble4(act[l] && q < nq ? __ldg(src + q) : 0u);
        }
    }
#pragma unroll
    for (int l = 0; l < LPW; ++l) {
        if (!act[l]) continue;
        T *dst = s1 + lines[l] * nz;
        uint32_t any = 0;
#pragma unroll
        for (int c = 0; c < CMAX; ++c) any |= nib[l][c];
        ++nseen;
        if (!__any_sync(VX_FULL_MASK, any != 0u)) {   // empty line: no site anywhere (edt.py:212)
            ++nempty;
#pragma unroll
            for (int c = 0; c < CMAX; ++c) {
                const int q = c * 32 + lane;
                if (q < nq) store4(dst, q, -1, -1, -1, -1);
            }
            continue;
        }
        pass1_line<CMAX>(nib[l], dst, nq, lane);
    }
    }
    if (linestat) {   // per CTA: two atomics
        __shared__ int s_cnt[2];
        if (threadIdx.x == 0) s_cnt[0] = s_cnt[1] = 0;
        __syncthreads();
        if (lane == 0 && nseen) {
            atomicAdd(&s_cnt[0], nempty);
            atomicAdd(&s_cnt[1], nseen);
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_cnt[1]) {
            atomicAdd(linestat + 2, s_cnt[0]);
            atomicAdd(linestat + 3, s_cnt[1]);
        }
    }
}

// Pass 1, 16 voxels per lane (nz % 16 == 0, 256 < nz <= 512 * CH): one
// 16-byte load per lane and 512-voxel chunk, so a warp reads a 512-voxel line
// in one instruction.  Per voxel the nearest site before (l) and after (r)
// comes from a running scan over the lane's 16 voxels, seeded by the nearest
// site in the lanes before / after (ballot + one shuffle); the answer is l if
// k - l <= r - k (edt.py:217-224; l + r >= 2k), with missing sides at -/+2^30.
template <int CH, bool FULL, typename T>
__global__ void __launch_bounds__(256, 6) k_pass1_x16(const uint8_t *__restrict__ occ, T *__restrict__ s1,
                                                   long long nlines, int nz, const uint8_t *__restrict__ sflag,
                                                   int ny, const int *__restrict__ xs, const int *__restrict__ hdr,
                                                   int *__restrict__ linestat) {
    constexpr int NONE_L = -(1 << 30), NONE_R = 1 << 30;
    __shared__ int4 s_stage[8][128];   // per warp: one 512-voxel chunk of s1 (2 KB)
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned gt = lane == 31 ? 0u : ~((2u << lane) - 1u);
    int nempty = 0, nseen = 0;
    const int m = xs ? __ldg(hdr) : 0;
    const long long total = xs ? (long long)m * ny : nlines;
    const long long wstep = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long line = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); line < total;
         line += wstep) {
        long long L = line;
        if (xs) {   // lines of occupied slices, slot-major
            const uint32_t slot = (uint32_t)line / (uint32_t)ny;
            L = (long long)__ldg(xs + slot) * ny + (line - (long long)slot * ny);
        } else if (sflag && !sflag[(uint32_t)line / (uint32_t)ny]) {
            continue;   // empty slice: nothing downstream reads it (warp-uniform)
        }
        const uint4 *src = reinterpret_cast<const uint4 *>(occ + L * nz);
        uint32_t msk[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int q = c * 32 + lane;   // 16-byte unit
            uint32_t mm = 0;
            if (q * 16 < nz) {
                const uint4 v = __ldcs(src + q);
                mm = nibble4(v.x) | (nibble4(v.y) << 4) | (nibble4(v.z) << 8) | (nibble4(v.w) << 12);
            }
            msk[c] = mm;
        }
        ++nseen;
        unsigned any = 0;
#pragma unroll
        for (int c = 0; c < CH; ++c) any |= msk[c];
        // 16-byte units: 4 (int32) or 8 (int16) values; UPC units per 512-voxel chunk
        constexpr int VPU = 16 / (int)sizeof(T), UPC = 512 / VPU;
        int4 *dst = reinterpret_cast<int4 *>(s1 + L * nz);
        if (!__any_sync(VX_FULL_MASK, any != 0u)) {   // empty line: no site anywhere (edt.py:212)
            ++nempty;
            const int nu = nz / VPU;   // 16-byte units of the line (coalesced rows)
            for (int j = lane; j < nu; j += 32) dst[j] = make_int4(-1, -1, -1, -1);
            continue;
        }
        // this warp's staging block; per lane, the XOR-swizzled 16-byte slots it
        // writes (units lane*4 + g) and reads (units g*32 + lane), as shared addresses
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_stage[threadIdx.x >> 5]);
        // int32: the lane writes units lane*4 + g (g < 4); int16: units lane*2 + h
        // (h < 2); units j live at slot j ^ ((j >> 3) & 7); reads take units g*32 + lane
        const uint32_t st_idx = VPU == 4 ? (uint32_t)((lane * 4) ^ ((lane >> 1) & 7))
                                         : (uint32_t)((lane * 2) ^ ((lane >> 2) & 7));
        const uint32_t ld_idx = (uint32_t)(lane ^ (lane >> 3));
        // warp-uniform carries: last site before chunk c, first site after it
        unsigned bal[CH];
        int lastc[CH], firstc[CH];
        int run = NONE_L;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            bal[c] = __ballot_sync(VX_FULL_MASK, msk[c] != 0u);
            lastc[c] = run;
            const int hl = bal[c] ? 31 - __clz(bal[c]) : 0;
            const uint32_t mb = __shfl_sync(VX_FULL_MASK, msk[c], hl);
            if (bal[c]) run = (c * 32 + hl) * 16 + 31 - __clz(mb);
        }
        run = NONE_R;
#pragma unroll
        for (int c = CH - 1; c >= 0; --c) {
            firstc[c] = run;
            const int ll = bal[c] ? __ffs(bal[c]) - 1 : 0;
            const uint32_t mb = __shfl_sync(VX_FULL_MASK, msk[c], ll);
            if (bal[c]) run = (c * 32 + ll) * 16 + __ffs(mb) - 1;
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int q = c * 32 + lane;
            const int base = q * 16;
            const uint32_t mm = msk[c];
            const unsigned pm = bal[c] & lt, nm = bal[c] & gt;
            const int lp = pm ? 31 - __clz(pm) : 0, ln = nm ? __ffs(nm) - 1 : 0;
            const uint32_t mbp = __shfl_sync(VX_FULL_MASK, mm, lp);
            const uint32_t mbn = __shfl_sync(VX_FULL_MASK, mm, ln);
            // sites relative to the lane's first voxel: l is the last site before it
            // (< 0), r the first after its 16 voxels (>= 16); far sentinels when none
            const int lrel = (pm ? (c * 32 + lp) * 16 + 31 - __clz(mbp) : lastc[c]) - base;
            int rrel = (nm ? (c * 32 + ln) * 16 + __ffs(mbn) - 1 : firstc[c]) - base;
            // backward over the lane's 16 voxels: rrel runs, the last site <= e is
            // one FLO of the masked bits (or lrel); ties -> lower k.  The four
            // 16-byte groups go through this warp's shared staging (XOR-swizzled
            // 16-byte units: conflict-free both ways) so that the global stores
            // are 512-byte coalesced rows (plain stores: pass 2 reads s1 from L2)
            if (FULL || base < nz) {
                int o8[8];   // int16: two groups per 16-byte unit
#pragma unroll
                for (int g = 3; g >= 0; --g) {
                    int o[4];
#pragma unroll
                    for (int u = 3; u >= 0; --u) {
                        const int e = 4 * g + u;
                        if (mm & (1u << e)) rrel = e;
                        const uint32_t le = mm & ((2u << e) - 1u);
                        const int lv = le ? 31 - __clz(le) : lrel;
                        o[u] = base + ((lv + rrel >= 2 * e) ? lv : rrel);
                    }
                    if constexpr (VPU == 4) {
                        VX_ASSERT((((lane * 4 + g) ^ ((lane >> 1) & 7))) < UPC, "pass-1 staging slot");
                        asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + ((st_idx ^ (uint32_t)g) << 4)),
                                     "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]) : "memory");
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u) o8[4 * (g & 1) + u] = o[u];
                        if ((g & 1) == 0) {   // groups g, g+1 complete unit lane*2 + g/2
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};"
                                         ::"r"(sbase + ((st_idx ^ (uint32_t)(g >> 1)) << 4)),
                                         "r"(pack16(o8[0], o8[1])), "r"(pack16(o8[2], o8[3])),
                                         "r"(pack16(o8[4], o8[5])), "r"(pack16(o8[6], o8[7])) : "memory");
                        }
                    }
                }
            }
            __syncwarp();
            const int nu = FULL ? UPC : min(UPC, (nz - c * 512) / VPU);   // 16-byte units of this chunk
#pragma unroll
            for (int g = 0; g < UPC / 32; ++g) {
                const int j = g * 32 + lane;
                VX_ASSERT(c * 512 + VPU * j < nz || j >= nu, "pass-1 store inside the line");
                if (FULL || j < nu) {
                    int4 v;
                    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(sbase + (((uint32_t)(g * 32) + (ld_idx ^ (uint32_t)((g & 1) * 4))) << 4)) : "memory");
                    dst[c * UPC + j] = v;
                }
            }
            __syncwarp();
        }
    }
    if (linestat) {   // per CTA: two atomics
        __shared__ int s_cnt[2];
        if (threadIdx.x == 0) s_cnt[0] = s_cnt[1] = 0;
        __syncthreads();
        if (lane == 0 && nseen) {
            atomicAdd(&s_cnt[0], nempty);
            atomicAdd(&s_cnt[1], nseen);
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_cnt[1]) {
            atomicAdd(linestat + 2, s_cnt[0]);
            atomicAdd(linestat + 3, s_cnt[1]);
        }
    }
}

// Pass 1, generic path (any nz): 32-voxel chunks with ballots; the forward
// sweep parks `l` in the output, the backward sweep combines.
template <typename T>
__global__ void __launch_bounds__(256) k_pass1_generic(const uint8_t *__restrict__ occ,
                                                       T *__restrict__ s1,
                                                       long long nlines, int nz,
                                                       const uint8_t *__restrict__ sflag, int ny) {
    const int lane = threadIdx.x & 31;
    const long long line = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (line >= nlines) return;
    if (sflag && !sflag[(uint32_t)line / (uint32_t)ny]) return;
    const uint8_t *src = occ + line * nz;
    T *dst = s1 + line * nz;
    int carry = -1;
    for (int base = 0; base < nz; base += 32) {
        const int k = base + lane;
        const bool o = k < nz && src[k] != 0;
        const uint32_t m = __ballot_sync(VX_FULL_MASK, o);
        const uint32_t below = m & ((2u << lane) - 1u);
        const int l = below ? base + 31 - __clz(below) : carry;
        if (k < nz) dst[k] = l;
        if (m) carry = base + 31 - __clz(m);
    }
    int carr = BIG;
    for (int base = ((nz - 1) / 32) * 32; base >= 0; base -= 32) {
        const int k = base + lane;
        const bool o = k < nz && src[k] != 0;
        const uint32_t m = __ballot_sync(VX_FULL_MASK, o);
        const uint32_t above = m & (0xffffffffu << lane);
        const int r = above ? base + __ffs(above) - 1 : carr;
        if (k < nz) dst[k] = pick(k, dst[k], r);
        if (m) carr = base + __ffs(m) - 1;
    }
}

// ---------------------------------------------------------------------------
// Passes 2 and 3: lower-envelope (strict lower hull) per column.
// ---------------------------------------------------------------------------
// row bits of the windowed search's keys (w << kRingRb | row): columns of up to
// 1024 rows; fixed so that the key constants compile to immediates
constexpr int kRingRb = 10;

struct ColParams {
    int nx, ny, nz;
    int L;             // column length (ny for pass 2, nx for pass 3)
    int B, W;          // bands per column, rows per band
    int nkt;           // k tiles of 32
    long long ntiles;  // total CTA tiles
    int zb, yzb;       // packing shifts (narrow)
    uint32_t zmask, ymask;
    long long plane;   // ny * nz            (global; output flat index)
    int nyl, j0;       // pass 3: rows of j held in this buffer and their offset
    long long splane;  // nyl * nz           (pass-3 addressing stride along x)
    long long nvox;    // nx * nyl * nz      (pass-3 scene stride)
    int boxh, rows_alloc;  // TMA staging: rows per box, rows of smem (>= L)
    int wb;                // pass 3 narrow entry: (x << wb) | w, w = dy^2 + dz^2
    uint32_t wmask;
    // occupied-slice list (single-scene EDT): pass 2 skips empty slices,
    // pass 3 stages and scans only the rows of occupied slices
    const uint8_t *sflag;  // per slice: any occupied voxel (nullptr = dense)
    const int *xs;         // occupied slice indices, ascending
    const int *hdr;        // hdr[0] = number of occupied slices (device-side)
    int stream_max;        // pass 3: k_pass3_stream takes m <= stream_max (-1: never)
    // windowed search (ring_tile) for dense scenes, tried first by k_column_tma<RING>
    const int *mcount;     // per-scene occupied-slice counts (nullptr: treat every scene as dense)
    const uint8_t *sflag3; // pass 3: per (scene, slice) flags (rows of empty slices hold no codes)
    int ring_min;          // scenes with >= ring_min occupied slices take the windowed search
    int *rhdr;             // search header: [0] pass-2 / [1] pass-3 fall-back counts, [2] empty
                           // k-lines and [3] k-lines seen by pass 1 (nullptr: no search)
    int fslot;             // 0 pass 2, 1 pass 3
    int nkt2, ny2;         // pass-2 tiling (pass 3's gate on pass 2's hand-backs)
    int rb;                // row bits of the search keys (w << rb | row)
    int ring_cap;          // largest search radius before a tile is handed back
    int ring_budget;       // mean window steps per 4-row block above which a tile is handed back
    uint32_t kinv;         // key of a row without a candidate (stays above every reachable key)
    int s16;               // pass 2: s1 holds int16 line sites (EdtPlan::s1_16)
};

template <int PASS, bool S2W, bool EW, int FW>
struct Col {
    using S2T = typename std::conditional<S2W, unsigned long long, uint32_t>::type;
    // pass 2: the stack entry is the s2 code itself; pass 3: (x, sy, sz)
    using EntT = typename std::conditional<PASS == 2 ? S2W : EW, unsigned long long, uint32_t>::type;
    // FW: 0 = int32 weights and products; 1 = int32 weights, int64 products
    // in the hull test; 2 = int64 weights
    using FT = typename std::conditional<FW == 2, long long, int>::type;
    using PT = typename std::conditional<FW >= 1, long long, int>::type;
    using InT = typename std::conditional<PASS == 2, int32_t, S2T>::type;
    using OutT = typename std::conditional<PASS == 2, S2T, int32_t>::type;

    static __device__ __forceinline__ bool valid(InT v) {
        if constexpr (PASS == 2) return v >= 0;
        else return v != (S2T)~(S2T)0;
    }
    static __device__ __forceinline__ InT invalid() {
        if constexpr (PASS == 2) return -1;
        else return (S2T)~(S2T)0;
    }
    // pass-2 entry == the s2 code of the site (row y, line site z).
    // pass-3 narrow entry == (x << wb) | w with w = (j-sy)^2 + (k-sz)^2, so
    // F = x^2 + w costs one multiply; the site code of a winning row is
    // re-read from the (L2-resident) pass-3 input when it is emitted.
    static __device__ __forceinline__ EntT make(const ColParams &P, InT v, int row, int j, int k) {
        if constexpr (PASS == 2) {
            if constexpr (S2W) return ((EntT)row << 32) | (EntT)(uint32_t)v;
            else return ((EntT)row << P.zb) | (EntT)v;
        } else {
            uint32_t sy, sz;
            if constexpr (S2W) { sy = (uint32_t)(v >> 32); sz = (uint32_t)v; }
            else { sy = (uint32_t)v >> P.zb; sz = (uint32_t)v & P.zmask; }
            if constexpr (EW) {
                return ((EntT)row << 42) | ((EntT)sy << 21) | (EntT)sz;
            } else if constexpr (kP3XW) {
                const int dy = j - (int)sy, dz = k - (int)sz;
                return ((EntT)row << P.wb) | (EntT)(uint32_t)(dy * dy + dz * dz);
            } else {
                return ((EntT)row << P.yzb) | (EntT)v;
            }
        }
    }
    static __device__ __forceinline__ int row(const ColParams &P, EntT e) {
        if constexpr (PASS == 2) {
            if constexpr (S2W) return (int)(e >> 32);
            else return (int)(e >> P.zb);
        } else {
            if constexpr (EW) return (int)(e >> 42);
            else if constexpr (kP3XW) return (int)(e >> P.wb);
            else return (int)(e >> P.yzb);
        }
    }
    // F = w + row^2 (edt.py:261-262, 362-364 fold the row term in at test time)
    static __device__ __forceinline__ FT F(const ColParams &P, EntT e, int j, int k) {
        if constexpr (PASS == 2) {
            int y, z;
            if constexpr (S2W) { y = (int)(e >> 32); z = (int)(uint32_t)e; }
            else { y = (int)(e >> P.zb); z = (int)((uint32_t)e & P.zmask); }
            const FT dz = (FT)(k - z);
            return dz * dz + (FT)y * (FT)y;
        } else {
            if constexpr (EW) {
                const int x = (int)(e >> 42), sy = (int)((e >> 21) & 0x1fffffull), sz = (int)(e & 0x1fffffull);
                const FT dy = (FT)(j - sy), dz = (FT)(k - sz);
                return dy * dy + dz * dz + (FT)x * (FT)x;
            } else if constexpr (kP3XW) {
                const int x = (int)(e >> P.wb);
                return (FT)x * (FT)x + (FT)((uint32_t)e & P.wmask);
            } else {
                const int x = (int)(e >> P.yzb), sy = (int)(((uint32_t)e >> P.zb) & P.ymask);
                const int sz = (int)((uint32_t)e & P.zmask);
                const FT dy = (FT)(j - sy), dz = (FT)(k - sz);
                return dy * dy + dz * dz + (FT)x * (FT)x;
            }
        }
    }
    // pass 3 narrow: does output() need the site code re-read from the input?
    static constexpr bool kRereadCode = PASS == 3 && !EW && kP3XW;
    static __device__ __forceinline__ OutT output(const ColParams &P, EntT e, InT code) {
        if constexpr (PASS == 2) {
            return (OutT)e;  // the entry is the s2 code
        } else {
            long long x, sy, sz;
            if constexpr (EW) {
                x = (long long)(e >> 42); sy = (long long)((e >> 21) & 0x1fffffull);
                sz = (long long)(e & 0x1fffffull);
            } else if constexpr (kP3XW) {
                x = (long long)(e >> P.wb);
                if constexpr (S2W) { sy = (long long)(code >> 32); sz = (long long)(uint32_t)code; }
                else { sy = (long long)((uint32_t)code >> P.zb); sz = (long long)((uint32_t)code & P.zmask); }
            } else {
                x = (long long)(e >> P.yzb); sy = (long long)(((uint32_t)e >> P.zb) & P.ymask);
                sz = (long long)((uint32_t)e & P.zmask);
            }
            return (int32_t)(x * P.plane + sy * P.nz + sz);  // edt.py:417
        }
    }
    static __device__ __forceinline__ OutT none() {
        if constexpr (PASS == 2) return (OutT)~(OutT)0;
        else return -1;
    }
};

// b on or above segment a-c  ==> pop b   (edt.py:267-268, written with F=w+y^2)
// (PT: the product type; int32 weights with int64 products are one IMAD.WIDE each)
template <typename FT, typename PT = FT>
__device__ __forceinline__ bool dominated(int ya, FT Fa, int yb, FT Fb, int yc, FT Fc) {
    return (PT)(Fb - Fa) * (PT)(yc - yb) >= (PT)(Fc - Fb) * (PT)(yb - ya);
}

// succ strictly closer than cur at query row y (edt.py:311 strict <)
template <typename FT>
__device__ __forceinline__ bool better(int ys, FT Fs, int yp, FT Fp, int y) {
    return Fs - Fp < (FT)2 * (FT)y * (FT)(ys - yp);
}

// ---- TMA helpers (tile staging) ---------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lds_u32(int addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_ef(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                               int c2) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

// One CTA tile: 32 consecutive k columns x the whole column length L, B bands
// of W rows.  STAGED: the input tile was brought into the stack region of
// shared memory by TMA and the band hulls are built in place (a band's stack
// never grows past the rows it has consumed); otherwise rows are read with
// coalesced 128-byte LDGs.
// Where pass-2 rows go.  Default: the s2 array.  SCAT (slab mode): row j of
// slice i goes straight into the pass-3 input of the rank that owns j --
// dst[q] + ((x_base + i) * nyl_q + j - j_start[q]) * nz + k -- a peer buffer
// mapped over NVLink, or this rank's all-to-all send block.
template <typename OutT, bool SCAT>
struct RowOut {
    OutT *p;
    long long step;
    int q, qend;
    __device__ __forceinline__ void begin(OutT *out, long long base, long long stride, int lo,
                                          const ScatterTab *sc, long long slice, int k, int nz) {
        if constexpr (!SCAT) {
            p = out + base + (long long)lo * stride;
            step = stride;
        } else {
            step = nz;
            q = 0;
            while (sc->j_start[q + 1] <= lo) ++q;
            seek(lo, sc, slice, k, nz);
        }
    }
    __device__ __forceinline__ void seek(int y, const ScatterTab *sc, long long slice, int k, int nz) {
        const int j0 = sc->j_start[q], nyl = sc->j_start[q + 1] - j0;
        qend = sc->j_start[q + 1];
        p = reinterpret_cast<OutT *>(sc->dst[q]) + ((sc->x_base + slice) * nyl + (y - j0)) * (long long)nz + k;
    }
    __device__ __forceinline__ void put(int y, OutT v, const ScatterTab *sc, long long slice, int k, int nz) {
        if constexpr (SCAT) {
            if (y == qend) {
                ++q;
                seek(y, sc, slice, k, nz);
            }
        }
        VX_ASSERT(p != nullptr, "column output pointer");
        *p = v;
        p += step;
    }
};

template <int PASS, bool S2W, bool EW, int FW, bool STAGED, bool SCAT = false, bool CMP = false, int TW = 32>
__device__ __forceinline__ void column_tile(const typename Col<PASS, S2W, EW, FW>::InT *__restrict__ in,
                                            typename Col<PASS, S2W, EW, FW>::OutT *__restrict__ out,
                                            typename Col<PASS, S2W, EW, FW>::EntT *stk, int *meta,
                                            const ColParams &P, long long tile,
                                            const ScatterTab *sc = nullptr) {
    using C = Col<PASS, S2W, EW, FW>;
    using EntT = typename C::EntT;
    using FT = typename C::FT;
    using PT = typename C::PT;
    using InT = typename C::InT;
    using OutT = typename C::OutT;

    const int kk = threadIdx.x;
    const int b = threadIdx.y;
    const int kt = (int)(tile % P.nkt);
    const long long outer = tile / P.nkt;
    const int k = kt * TW + kk;
    const bool colok = k < P.nz;
    long long base, stride;
    int jq = 0;
    if constexpr (PASS == 2) {  // outer = i (slices of every scene stack along i)
        base = outer * P.plane + k;
        stride = P.nz;
    } else {                    // outer = scene * nyl + local j
        const long long scene = outer / P.nyl;
        const int jl = (int)(outer - scene * P.nyl);
        jq = P.j0 + jl;          // global j: weights use global coordinates
        base = scene * P.nvox + (long long)jl * P.nz + k;
        stride = P.splane;
    }
    int *bs = meta;
    int *be = bs + P.B * TW;
    int *nbl = be + P.B * TW;
    int *ncnt = nbl + P.B * TW;
    const int lo = min(P.L, b * P.W);
    const int hi = min(P.L, lo + P.W);

    VX_PT(1);
    // ---- phase A: band-local hull (edt.py:253-276 for one band) ----------
    // slots [alo, ahi) of the staged tile; CMP: the tile holds only the rows
    // of occupied slices (slot t = row xs[t]), split evenly over the bands
    int alo = lo, ahi = hi;
    int G = P.B;   // groups that build band hulls (and then merge: log2 G rounds)
    // CMP: this scene's occupied-slice list (one list per scene of a batch)
    const long long cscene = PASS == 3 ? outer / P.nyl : 0;
    const int *cxs = CMP ? P.xs + cscene * P.nx : nullptr;
    if constexpr (CMP) {
        const int m = __ldg(P.hdr + cscene);
        if (m < P.L) {
            // few occupied slices: longer groups, fewer merge rounds
            G = 1;
            while (2 * G <= P.B && 2 * G * VX_CMP_GROUP_ROWS <= m) G *= 2;
        }
        const int wc = (m + G - 1) / G;
        alo = b < G ? min(m, b * wc) : m;
        ahi = b < G ? min(m, alo + wc) : m;
    }
    int n = 0;
    if (colok) {
        int ya = 0, yb = 0;
        FT Fa = 0, Fb = 0;
        auto consume = [&](InT v, int yc) {
            if (!C::valid(v)) return;
            const EntT ec = C::make(P, v, yc, jq, k);
            const FT Fc = C::F(P, ec, jq, k);
            while (n >= 2 && dominated<FT, PT>(ya, Fa, yb, Fb, yc, Fc)) {
                --n;
                yb = ya;
                Fb = Fa;
                if (n >= 2) {
                    const EntT t = stk[(size_t)(alo + n - 2) * TW + kk];
                    ya = C::row(P, t);
                    Fa = C::F(P, t, jq, k);
                }
            }
            VX_ASSERT(alo + n < (STAGED ? P.rows_alloc : P.L), "column stack slot");
            stk[(size_t)(alo + n) * TW + kk] = ec;
            ya = yb; Fa = Fb;
            yb = yc; Fb = Fc;
            ++n;
        };
        if constexpr (STAGED) {
            const InT *tin = reinterpret_cast<const InT *>(stk);
            if constexpr (CMP) {
                for (int t = alo; t < ahi; ++t) consume(tin[(size_t)t * TW + kk], __ldg(cxs + t));
            } else {
#pragma unroll 4
                for (int y = lo; y < hi; ++y) consume(tin[(size_t)y * TW + kk], y);
            }
        } else {
            const InT *src = in + base + (long long)lo * stride;
            for (int y0 = lo; y0 < hi; y0 += 8) {
                InT v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    v[u] = (y0 + u < hi) ? __ldg(src) : C::invalid();
                    src += stride;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) consume(v[u], y0 + u);
            }
        }
    }
    bs[b * TW + kk] = alo;
    be[b * TW + kk] = alo + n;
    __syncthreads();
    VX_PT(2);

    // ---- phase B: pairwise bridge merges (same hull as edt.py:277-294) ---
    for (int r = 1; r < G; r <<= 1) {
        if (colok && (b & (2 * r - 1)) == r) {
            const int gl = b - r, gm = b, ge = min(P.B, b + r);
            int bl = gm - 1;
            while (bl >= gl && bs[bl * TW + kk] == be[bl * TW + kk]) --bl;
            int br = gm;
            while (br < ge && bs[br * TW + kk] == be[br * TW + kk]) ++br;
            if (bl >= gl && br < ge) {
                int pl1 = be[bl * TW + kk] - 1;
                EntT e = stk[(size_t)pl1 * TW + kk];
                int yl1 = C::row(P, e);
                FT Fl1 = C::F(P, e, jq, k);
                int pr0 = bs[br * TW + kk];
                e = stk[(size_t)pr0 * TW + kk];
                int yr0 = C::row(P, e);
                FT Fr0 = C::F(P, e, jq, k);
                while (true) {
                    while (true) {  // pop the left tail while dominated
                        int bl2 = bl, pl2 = pl1 - 1;
                        if (pl2 < bs[bl * TW + kk]) {
                            bl2 = bl - 1;
                            while (bl2 >= gl && bs[bl2 * TW + kk] == be[bl2 * TW + kk]) --bl2;
                            if (bl2 < gl) break;
                            pl2 = be[bl2 * TW + kk] - 1;
                        }
                        e = stk[(size_t)pl2 * TW + kk];
                        const int yl2 = C::row(P, e);
                        const FT Fl2 = C::F(P, e, jq, k);
                        if (!dominated<FT, PT>(yl2, Fl2, yl1, Fl1, yr0, Fr0)) break;
                        be[bl * TW + kk] = pl1;
                        bl = bl2; pl1 = pl2; yl1 = yl2; Fl1 = Fl2;
                    }
                    bool popped = false;
                    while (true) {  // pop the right head while dominated
                        int br2 = br, pr1 = pr0 + 1;
                        if (pr1 >= be[br * TW + kk]) {
                            br2 = br + 1;
                            while (br2 < ge && bs[br2 * TW + kk] == be[br2 * TW + kk]) ++br2;
                            if (br2 >= ge) break;
                            pr1 = bs[br2 * TW + kk];
                        }
                        e = stk[(size_t)pr1 * TW + kk];
                        const int yr1 = C::row(P, e);
                        const FT Fr1 = C::F(P, e, jq, k);
                        if (!dominated<FT, PT>(yl1, Fl1, yr0, Fr0, yr1, Fr1)) break;
                        bs[br * TW + kk] = pr0 + 1;
                        br = br2; pr0 = pr1; yr0 = yr1; Fr0 = Fr1;
                        popped = true;
                    }
                    if (!popped) break;
                }
            }
        }
        __syncthreads();
    }

    VX_PT(3);
    // ---- phase C: list of non-empty bands per column ---------------------
    if (b == 0) {
        int c = 0;
        for (int q = 0; q < P.B; ++q)
            if (bs[q * TW + kk] < be[q * TW + kk]) nbl[(c++) * TW + kk] = q;
        ncnt[kk] = c;
    }
    __syncthreads();

    VX_PT(4);
    // ---- phase D: queries for this band's rows (edt.py:300-317) ----------
    if (colok && lo < hi) {
        const int cnt = ncnt[kk];
        RowOut<OutT, SCAT> dst;
        dst.begin(out, base, stride, lo, sc, outer, k, P.nz);
        if (cnt == 0) {  // no candidate in the whole column (edt.py:295-299)
            for (int y = lo; y < hi; ++y) dst.put(y, C::none(), sc, outer, k, P.nz);
        } else {
            const int y0 = lo;
            // first hull vertex minimising at y0: binary search over bands ...
            int mlo = 0, mhi = cnt - 1;
            while (mlo < mhi) {
                const int mid = (mlo + mhi) >> 1;
                const int bm = nbl[mid * TW + kk], bn = nbl[(mid + 1) * TW + kk];
                const EntT a = stk[(size_t)(be[bm * TW + kk] - 1) * TW + kk];
                const EntT s = stk[(size_t)bs[bn * TW + kk] * TW + kk];
                if (better<FT>(C::row(P, s), C::F(P, s, jq, k), C::row(P, a), C::F(P, a, jq, k), y0))
                    mlo = mid + 1;
                else
                    mhi = mid;
            }
            int m = mlo;
            int bm = nbl[m * TW + kk];
            // ... then inside the band
            int ilo = bs[bm * TW + kk], ihi = be[bm * TW + kk] - 1;
            while (ilo < ihi) {
                const int mid = (ilo + ihi) >> 1;
                const EntT a = stk[(size_t)mid * TW + kk];
                const EntT s = stk[(size_t)(mid + 1) * TW + kk];
                if (better<FT>(C::row(P, s), C::F(P, s, jq, k), C::row(P, a), C::F(P, a, jq, k), y0))
                    ilo = mid + 1;
                else
                    ihi = mid;
            }
            int pos = ilo;
            int epos = be[bm * TW + kk];
            EntT cur = stk[(size_t)pos * TW + kk];
            int yc = C::row(P, cur);
            FT Fc = C::F(P, cur, jq, k);
            const InT *src = in + base;
            auto code_of = [&](int row) -> InT {
                if constexpr (C::kRereadCode) return __ldg(src + (long long)row * stride);
                else return InT(0);
            };
            OutT ocur = C::output(P, cur, code_of(yc));
            // successor
            int spos = -1, sm = m;
            if (pos + 1 < epos) spos = pos + 1;
            else if (m + 1 < cnt) { sm = m + 1; spos = bs[nbl[sm * TW + kk] * TW + kk]; }
            EntT sent = 0;
            int ys = 0;
            FT Fs = 0;
            InT scode = InT(0);   // the successor's site code, prefetched
            if (spos >= 0) {
                sent = stk[(size_t)spos * TW + kk];
                ys = C::row(P, sent);
                Fs = C::F(P, sent, jq, k);
                scode = code_of(ys);
            }
            // successor strictly closer at row y  <=>  Fs - Fc < y * 2 (ys - yc)
            // (edt.py:311); the right side is stepped by t per row
            constexpr FT kNever = sizeof(FT) == 4 ? (FT)0x7fffffff : (FT)0x7fffffffffffffffLL;
            FT dN = spos >= 0 ? Fs - Fc : kNever;
            FT t = spos >= 0 ? (FT)2 * (FT)(ys - yc) : (FT)0;
            FT rhs = (FT)lo * t;
#pragma unroll kColWalkUnroll
            for (int y = lo; y < hi; ++y, rhs += t) {
                if (dN < rhs) {
                    InT ccode = scode;
                    do {
                        cur = sent; yc = ys; Fc = Fs; pos = spos; ccode = scode;
                        if (sm != m) { m = sm; epos = be[nbl[m * TW + kk] * TW + kk]; }
                        if (pos + 1 < epos) spos = pos + 1;
                        else if (m + 1 < cnt) { sm = m + 1; spos = bs[nbl[sm * TW + kk] * TW + kk]; }
                        else spos = -1;
                        if (spos >= 0) {
                            sent = stk[(size_t)spos * TW + kk];
                            ys = C::row(P, sent);
                            Fs = C::F(P, sent, jq, k);
                            scode = code_of(ys);
                        }
                    } while (spos >= 0 && better<FT>(ys, Fs, yc, Fc, y));
                    ocur = C::output(P, cur, ccode);
                    dN = spos >= 0 ? Fs - Fc : kNever;
                    t = spos >= 0 ? (FT)2 * (FT)(ys - yc) : (FT)0;
                    rhs = (FT)y * t;
                }
                dst.put(y, ocur, sc, outer, k, P.nz);
            }
        }
    }
}

template <int PASS, bool S2W, bool EW, int FW, bool SCAT>
__global__ void __launch_bounds__(kColThreads, kColMinBlocks) k_column_smem(const typename Col<PASS, S2W, EW, FW>::InT *__restrict__ in,
                                                      typename Col<PASS, S2W, EW, FW>::OutT *__restrict__ out,
                                                      const ColParams P, const __grid_constant__ ScatterTab sc) {
    extern __shared__ __align__(128) unsigned char smem[];
    using EntT = typename Col<PASS, S2W, EW, FW>::EntT;
    EntT *stk = reinterpret_cast<EntT *>(smem);
    int *meta = reinterpret_cast<int *>(smem + (size_t)P.L * 32 * sizeof(EntT));
    column_tile<PASS, S2W, EW, FW, false, SCAT>(in, out, stk, meta, P, blockIdx.x, &sc);
}

// int16 s1 (EdtPlan::s1_16): the tile arrived packed (2 bytes per value) at the
// start of shared memory and is widened in place to 32-bit words cv(value, row).
// Widened row y covers packed rows 2y and 2y+1, so (L = 32 B rows): (1) rows
// >= L/2 widen directly -- their words land past the packed tile; (2) rows
// < L/2 are read into registers (two per word) before a barrier and written
// after it.  Each thread (column kk, band b) takes 16 rows in each step.
// Ends with a barrier.
template <int TW, typename CV>
__device__ __forceinline__ void widen16(unsigned char *smem, CV cv) {
    const uint16_t *src = reinterpret_cast<const uint16_t *>(smem) + threadIdx.x;
    uint32_t *dst = reinterpret_cast<uint32_t *>(smem) + threadIdx.x;
    const int hi0 = (int)blockDim.y * 16 + (int)threadIdx.y * 16;   // upper half: rows L/2 + 16 b ...
#pragma unroll 8
    for (int y = hi0; y < hi0 + 16; ++y) dst[y * TW] = cv((int)(int16_t)src[y * TW], y);
    const int lo = (int)threadIdx.y * 16;                            // lower half: rows 16 b ...
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        v[i] = (uint32_t)src[(lo + 2 * i) * TW] | ((uint32_t)src[(lo + 2 * i + 1) * TW] << 16);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        dst[(lo + 2 * i) * TW] = cv((int)(int16_t)(v[i] & 0xffffu), lo + 2 * i);
        dst[(lo + 2 * i + 1) * TW] = cv((int)(int16_t)(v[i] >> 16), lo + 2 * i + 1);
    }
    __syncthreads();
}

// TMA-staged variant (narrow 32-bit codes, nz % 4 == 0): one elected thread
// issues the bulk tensor loads of the whole 32-column tile into the stack
// region; every row of the column is in flight at once.
template <int PASS, int FW, bool SCAT, bool CMP, int TW>
__device__ __forceinline__ void col_tma_run(const CUtensorMap *tmap, const CUtensorMap *tmap1,
                                            const typename Col<PASS, false, false, FW>::InT *__restrict__ in,
                                            typename Col<PASS, false, false, FW>::OutT *__restrict__ out,
                                            const ColParams &P, const ScatterTab *sc, unsigned char *smem,
                                            long long tile, long long outer, int kt) {
    using EntT = typename Col<PASS, false, false, FW>::EntT;
    EntT *stk = reinterpret_cast<EntT *>(smem);
    int *meta = reinterpret_cast<int *>(smem + (size_t)P.rows_alloc * TW * sizeof(EntT));
    uint64_t *bar = reinterpret_cast<uint64_t *>(meta + 3 * P.B * TW + TW);
    VX_PT(0);
    bool all_rows = true;
    if constexpr (CMP) {
        // rows of occupied slices only (slot t <- row xs[t]); when every slice
        // is occupied the plain box loads below are used instead
        const int scene = (int)(outer / P.nyl);
        const int m = __ldg(P.hdr + scene);
        if (m <= P.stream_max) return;   // k_pass3_stream did this pass
        all_rows = m == P.L;
        if (!all_rows) {
            const int jl = (int)(outer - (long long)scene * P.nyl);
            const int *xsl = P.xs + (long long)scene * P.nx;
            // 16-column rows are 64 B, below the 128-B smem alignment of tensor
            // boxes: plain bulk copies of the row's in-range columns instead
            const uint32_t rbytes = TW == 32 ? 0u : (uint32_t)min(TW, P.nz - kt * TW) * (uint32_t)sizeof(EntT);
            if (threadIdx.x == 0 && threadIdx.y == 0) {
                mbar_init(bar, 1);
                mbar_expect_tx(bar, TW == 32 ? (uint32_t)m * (uint32_t)TW * (uint32_t)sizeof(EntT)
                                             : (uint32_t)m * rbytes);
            }
            __syncthreads();
            // one TW-column x 1-row load per occupied row, issued by all threads
            const int tid = threadIdx.y * TW + threadIdx.x, nth = blockDim.x * blockDim.y;
            if constexpr (TW == 32) {
                for (int t = tid; t < m; t += nth)
                    tma_load_4d(stk + (size_t)t * TW, tmap1, bar, kt * TW, jl, __ldg(xsl + t), scene);
            } else {
                const EntT *row0 = reinterpret_cast<const EntT *>(in) + (long long)scene * P.nvox +
                                   (long long)jl * P.nz + kt * TW;
                for (int t = tid; t < m; t += nth)
                    bulk_load(stk + (size_t)t * TW, row0 + (long long)__ldg(xsl + t) * P.splane, rbytes, bar);
            }
        }
    }
    if (all_rows) {
        if (threadIdx.x == 0 && threadIdx.y == 0) {
            mbar_init(bar, 1);
            const int nbox = P.rows_alloc / P.boxh;
            const int esz = PASS == 2 && P.s16 ? 2 : (int)sizeof(EntT);   // int16 s1: packed tile
            mbar_expect_tx(bar, (uint32_t)(P.rows_alloc * TW * esz));
            for (int q = 0; q < nbox; ++q) {
                void *dst = smem + (size_t)q * P.boxh * TW * esz;
                if constexpr (PASS == 2) {
                    if constexpr (VX_P2_EVICT_FIRST)   // s1 is read once: keep s2 in L2 for pass 3
                        tma_load_3d_ef(dst, tmap, bar, kt * TW, q * P.boxh, (int)outer);
                    else
                        tma_load_3d(dst, tmap, bar, kt * TW, q * P.boxh, (int)outer);
                } else {
                    const int scene = (int)(outer / P.nyl);
                    const int jl = (int)(outer - (long long)scene * P.nyl);
                    tma_load_4d(dst, tmap, bar, kt * TW, jl, q * P.boxh, scene);
                }
            }
        }
    }
    __syncthreads();
    mbar_wait(bar, 0);
    if constexpr (PASS == 2) {
        if (P.s16) widen16<TW>(smem, [](int v, int) { return (uint32_t)v; });
    }
    column_tile<PASS, false, false, FW, true, SCAT, CMP, TW>(in, out, stk, meta, P, tile, sc);
#ifdef VX_PHASE_TIMING
    VX_PT(5);
    __syncthreads();
    VX_PT(6);
#endif
}

// is the windowed search on for this call?  Pass 1 counted the k-lines without
// any site: when more than 1 in 10 is empty the rows are too sparse for it.
// Pass 3 also stays off when pass 2 fell back on more than 1 tile in 8.
__device__ __forceinline__ bool ring_active(const ColParams &P) {
    if (!P.rhdr) return false;
    const int empty = __ldcg(P.rhdr + 2), lines = __ldcg(P.rhdr + 3);
    if (empty * 10LL > (long long)lines) return false;
    if (P.fslot == 1 && __ldcg(P.rhdr) * 8LL > (long long)lines / max(P.ny2, 1) * P.nkt2) return false;
    return true;
}
// does this tile's scene take the windowed search?
__device__ __forceinline__ bool ring_scene(const ColParams &P, int pass, long long outer) {
    const long long scene = pass == 2 ? outer / P.nx : outer / P.nyl;
    return (P.mcount ? __ldg(P.mcount + scene) : P.L) >= P.ring_min;
}

// ---- dense tiles: windowed exact search ------------------------------------------
// When every slice is occupied and sites are dense, each query row's answer
// lies within a few rows: the reference's lower envelope (edt.py:253-317) gives,
// for query row q, the FIRST row y minimising (q - y)^2 + w_y (ties: lowest row,
// SURVEY 0.3).  With keys K_y = (w_y << rb) | y that is min_y (K_y + ((q-y)^2 << rb)),
// and no row with (q - y)^2 > d_min can win, so the window around q grows one
// row per side until the next distance squared exceeds the running minimum.
// One warp = 32 columns (lanes) x one band of rows, all lanes on the same rows
// (coalesced stores); four query rows share one window; the tile (TMA-staged,
// then turned into keys in place) is read-only.  Returns false when a window
// would exceed P.ring_cap rows or the windows cost more than P.ring_budget steps
// per block on average: the caller then runs the banded kernel on the tile.
template <int PASS, bool SCAT, int TW>
__device__ __forceinline__ bool ring_tile(const typename Col<PASS, false, false, 0>::InT *__restrict__ in,
                                          typename Col<PASS, false, false, 0>::OutT *__restrict__ out,
                                          const ColParams &P, const ScatterTab *scp, unsigned char *smem,
                                          const CUtensorMap *tmapp, long long tile, long long outer, int kt) {
    using C = Col<PASS, false, false, 0>;
    using InT = typename C::InT;
    using OutT = typename C::OutT;
    const ScatterTab &sc = *scp;
    const CUtensorMap &tmap = *tmapp;
    uint32_t *key = reinterpret_cast<uint32_t *>(smem);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + (size_t)P.rows_alloc * TW * 4);
    int *s_fail = reinterpret_cast<int *>(bar + 1);
    const int scene = PASS == 2 ? 0 : (int)(outer / P.nyl);
    const int jl = PASS == 2 ? 0 : (int)(outer - (long long)scene * P.nyl);
    const bool s16 = PASS == 2 && P.s16;   // int16 s1: packed tile, widened into keys below
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        *s_fail = 0;
        mbar_init(bar, 1);
        const int nbox = P.rows_alloc / P.boxh;
        mbar_expect_tx(bar, (uint32_t)(P.rows_alloc * TW * (s16 ? 2 : 4)));
        for (int q = 0; q < nbox; ++q) {
            void *dst = smem + (size_t)q * P.boxh * TW * (s16 ? 2 : 4);
            if constexpr (PASS == 2) tma_load_3d(dst, &tmap, bar, kt * TW, q * P.boxh, (int)outer);
            else tma_load_4d(dst, &tmap, bar, kt * TW, jl, q * P.boxh, scene);
        }
    }
    const int kk = threadIdx.x, b = threadIdx.y;
    const int k = kt * TW + kk;
    const bool colok = k < P.nz;
    const int lo = min(P.L, b * P.W), hi = min(P.L, lo + P.W);
    const int jq = PASS == 2 ? 0 : P.j0 + jl;
    long long base, stride;
    if constexpr (PASS == 2) {
        base = outer * P.plane + k;
        stride = P.nz;
    } else {
        base = (long long)scene * P.nvox + (long long)jl * P.nz + k;
        stride = P.splane;
    }
    // rows of empty slices hold no pass-2 codes (pass 2 skipped them)
    const uint8_t *sfl = PASS == 3 && P.sflag3 && (P.mcount ? __ldg(P.mcount + scene) : 0) < P.nx
                             ? P.sflag3 + (long long)scene * P.nx : nullptr;
    constexpr int rb = kRingRb;   // fixed: the key constants are immediates
    __syncthreads();
    mbar_wait(bar, 0);
    // the tile's values -> search keys, in place (each thread its band's rows)
    uint32_t *col = key + kk;
    if (s16) {   // pass 2 from int16 s1: the band's values through registers, then keys
        const uint32_t kinv = P.kinv;
        widen16<TW>(smem, [=](int v, int y) -> uint32_t {
            if (v < 0) return kinv;
            const int dz = k - v;
            return ((uint32_t)(dz * dz) << rb) | (uint32_t)y;
        });
    } else if (colok) {
#pragma unroll 4
        for (int y = lo; y < hi; ++y) {
            VX_ASSERT(y >= 0 && y < P.rows_alloc, "ring key row");
            const uint32_t v = col[y * TW];
            uint32_t kv = P.kinv;
            if constexpr (PASS == 2) {
                if ((int)v >= 0) {
                    const int dz = k - (int)v;
                    kv = ((uint32_t)(dz * dz) << rb) | (uint32_t)y;
                }
            } else {
                if (v != 0xffffffffu && (!sfl || sfl[y])) {
                    const int dy = jq - (int)(v >> P.zb), dz = k - (int)(v & P.zmask);
                    kv = ((uint32_t)(dy * dy + dz * dz) << rb) | (uint32_t)y;
                }
            }
            col[y * TW] = kv;
        }
    }
    __syncthreads();
    if (colok && lo < hi) {
        const uint32_t rmask = (1u << rb) - 1u;
        const uint32_t one = 1u << rb;
        // shared byte addresses: this lane's column at row 0 and at row L-1;
        // windows are clamped to them (a clamped read re-reads an edge row at a
        // larger distance: a larger key, never a new minimum)
        constexpr int rowb = TW * 4;
        const int cb = (int)smem_u32(col), ce = cb + (P.L - 1) * rowb;
        const int cap = P.ring_cap;
        // cost guard: a tile whose windows average more than ring_budget steps
        // per block is cheaper in the banded kernel -- hand it back early
        const int budget = P.ring_budget;
        int spent = -2 * budget;
        // the winners' codes are re-read from the input (int16 or int32 s1 in pass 2)
        const int esz = s16 ? 2 : (int)sizeof(InT);
        const char *srcb = reinterpret_cast<const char *>(in) + base * esz;
        const uint32_t ustride4 = (uint32_t)stride * (uint32_t)esz;   // row byte offsets fit 32 bits
        RowOut<OutT, SCAT> dst;
        dst.begin(out, base, stride, lo, &sc, outer, k, P.nz);
        // four query rows per block share one window: step s reads rows
        // q0 - s and q0 + 3 + s, at distances s..s+3 from the block's rows
        constexpr int R = 4;
        int wrow[R];
        InT wcode[R];
        int pend = 0;   // rows of the previous block waiting for their store
        const uint32_t plane = (uint32_t)P.plane, nzu = (uint32_t)P.nz, zb = (uint32_t)P.zb, zmask = P.zmask;
        auto out_of = [&](int row, InT c) -> OutT {
            if constexpr (PASS == 2) return ((OutT)row << zb) | (OutT)(uint32_t)c;
            else return (int32_t)((uint32_t)row * plane + (c >> zb) * nzu + (c & zmask));
        };
        auto emit_pending = [&](int q0) {
            if (pend == R) {   // full block: four straight stores
#pragma unroll
                for (int i = 0; i < R; ++i) dst.put(q0 + i, out_of(wrow[i], wcode[i]), &sc, outer, k, P.nz);
            } else {
#pragma unroll
                for (int i = 0; i < R; ++i)
                    if (i < pend) dst.put(q0 + i, out_of(wrow[i], wcode[i]), &sc, outer, k, P.nz);
            }
        };
        int qa = cb + lo * rowb;
        int q0 = lo;
        for (; q0 < hi; q0 += R, qa += R * rowb) {
            if (*(volatile int *)s_fail) break;
            emit_pending(q0 - R);   // the previous block's codes were fetched a block ago
            VX_ASSERT(qa >= cb && qa <= ce, "ring block row");
            const uint32_t k0 = lds_u32(qa), k1 = lds_u32(min(qa + rowb, ce));
            const uint32_t k2 = lds_u32(min(qa + 2 * rowb, ce)), k3 = lds_u32(min(qa + 3 * rowb, ce));
            uint32_t b0 = min(min(k0, k1 + one), min(k2 + 4u * one, k3 + 9u * one));
            uint32_t b1 = min(min(k0 + one, k1), min(k2 + one, k3 + 4u * one));
            uint32_t b2 = min(min(k0 + 4u * one, k1 + one), min(k2, k3 + one));
            uint32_t b3 = min(min(k0 + 9u * one, k1 + 4u * one), min(k2 + one, k3));
            // o_i = (s + i)^2 << rb; rows 0 and 3 next see distance s, rows 1 and 2
            // distance s + 1.  Two steps per trip (one exit test; an extra step
            // only adds larger keys)
            uint32_t o0 = one, o1 = 4u * one, o2 = 9u * one, o3 = 16u * one, d3 = 9u * one;
            const int qb = qa + 3 * rowb;
            bool more = (max(b0, b3) >= o0) | (max(b1, b2) >= o1);
            // interior trips first: while both windows stay inside the column
            // (left rows q0-1-2t, q0-2-2t >= 0; right rows q0+4+2t, q0+5+2t <= L-1)
            // the loads need no clamps -- two running pointers, immediate offsets
            const int tfree = min(min(q0, P.L - R - q0), cap) >> 1;   // warp-uniform
            const uint32_t *pl = col + (q0 - 1) * TW, *pr = col + (q0 + R) * TW;
            int t = 0;
#pragma unroll 3
            for (; more && t < tfree; ++t) {
                const uint32_t o4 = o3 + d3;   // (s + 4)^2
                d3 += 2u * one;
                const uint32_t kl = pl[0], kl2 = pl[-TW], kr = pr[0], kr2 = pr[TW];
                b0 = min(b0, kl + o0); b1 = min(b1, kl + o1); b2 = min(b2, kl + o2); b3 = min(b3, kl + o3);
                b0 = min(b0, kr + o3); b1 = min(b1, kr + o2); b2 = min(b2, kr + o1); b3 = min(b3, kr + o0);
                b0 = min(b0, kl2 + o1); b1 = min(b1, kl2 + o2); b2 = min(b2, kl2 + o3); b3 = min(b3, kl2 + o4);
                b0 = min(b0, kr2 + o4); b1 = min(b1, kr2 + o3); b2 = min(b2, kr2 + o2); b3 = min(b3, kr2 + o1);
                o0 = o2; o1 = o3; o2 = o4;
                o3 = o4 + d3;                  // (s + 5)^2
                d3 += 2u * one;
                pl -= 2 * TW;
                pr += 2 * TW;
                more = (max(b0, b3) >= o0) | (max(b1, b2) >= o1);
            }
            // then the clamped steps near the column ends
            int ro = (1 + 2 * t) * rowb, sdone = 2 * t;
            while (more & (sdone < cap)) {
                const uint32_t o4 = o3 + d3;   // (s + 4)^2
                d3 += 2u * one;
                uint32_t kl = lds_u32(max(qa - ro, cb)), kr = lds_u32(min(qb + ro, ce));
                const uint32_t kl2 = lds_u32(max(qa - ro - rowb, cb)), kr2 = lds_u32(min(qb + ro + rowb, ce));
                b0 = min(b0, kl + o0); b1 = min(b1, kl + o1); b2 = min(b2, kl + o2); b3 = min(b3, kl + o3);
                b0 = min(b0, kr + o3); b1 = min(b1, kr + o2); b2 = min(b2, kr + o1); b3 = min(b3, kr + o0);
                b0 = min(b0, kl2 + o1); b1 = min(b1, kl2 + o2); b2 = min(b2, kl2 + o3); b3 = min(b3, kl2 + o4);
                b0 = min(b0, kr2 + o4); b1 = min(b1, kr2 + o3); b2 = min(b2, kr2 + o2); b3 = min(b3, kr2 + o1);
                o0 = o2; o1 = o3; o2 = o4;
                o3 = o4 + d3;                  // (s + 5)^2
                d3 += 2u * one;
                ro += 2 * rowb;
                sdone += 2;
                more = (max(b0, b3) >= o0) | (max(b1, b2) >= o1);
            }
            spent += sdone - budget;
            if (more | (spent > 0)) {   // beyond the cap, or too costly
                *(volatile int *)s_fail = 1;
                break;
            }
            const uint32_t bb[R] = {b0, b1, b2, b3};
            pend = min(R, hi - q0);
#pragma unroll
            for (int i = 0; i < R; ++i) {
                // every block row holds a real winner (a clamped read only repeats
                // an edge row); its code is loaded now and stored a block later
                const int row = (int)(bb[i] & rmask);
                VX_ASSERT(row >= 0 && row < P.L && bb[i] < P.kinv, "ring winner row");
                wrow[i] = row;
                const char *pc = srcb + (unsigned long long)(uint32_t)row * ustride4;
                wcode[i] = s16 ? (InT)(int)__ldg(reinterpret_cast<const short *>(pc)) : __ldg(reinterpret_cast<const InT *>(pc));
            }
        }
        if (q0 >= hi) emit_pending(q0 - R);
    }
    __syncthreads();
    const bool failed = *(volatile int *)s_fail != 0;
    if (failed && threadIdx.x == 0 && threadIdx.y == 0) atomicAdd(P.rhdr + P.fslot, 1);   // pass 3's gate
    return !failed;
}


// Passes 2/3 with TMA-staged tiles, one tile per CTA.  RING: dense scenes first
// try the windowed search on the tile; on a fall-back the tile is re-staged
// and takes the banded path (column_tile).
template <int PASS, int FW, bool SCAT, bool CMP, int MAXT, int TW = 32, bool RING = false>
__global__ void __launch_bounds__(MAXT, MAXT >= 1024 ? 1 : (RING ? 3 : kColMinBlocks)) k_column_tma(const __grid_constant__ CUtensorMap tmap,
                                                     const __grid_constant__ CUtensorMap tmap1,
                                                     const typename Col<PASS, false, false, FW>::InT *__restrict__ in,
                                                     typename Col<PASS, false, false, FW>::OutT *__restrict__ out,
                                                     const ColParams P, const __grid_constant__ ScatterTab sc) {
    extern __shared__ __align__(128) unsigned char smem[];
    long long tile = blockIdx.x;
    if constexpr (PASS == 2) {   // surplus CTAs leave before any index math
        if (P.xs && (long long)blockIdx.x >= (long long)__ldg(P.hdr) * P.nkt) return;
    }
    const int kt = (int)(tile % P.nkt);
    long long outer = tile / P.nkt;
    if constexpr (PASS == 2) {
        if (P.xs) {   // occupied-slice list: CTA rows map to occupied slices, the
                      // surplus CTAs (empty slices) all sit at the end of the grid
            const int m = __ldg(P.hdr);
            // VX_P2_REVERSE: last occupied slice first -- pass 1 wrote the
            // slices in ascending order, so the newest s1 lines, still in L2,
            // are read first
            outer = __ldg(P.xs + (VX_P2_REVERSE ? m - 1 - outer : outer));
            tile = outer * P.nkt + kt;
        } else if (P.sflag && !P.sflag[outer]) {
            return;   // empty slice: pass 3 never reads it
        }
    }
    if constexpr (RING && FW <= 1) {
        // the scene's slice count first (one cached load): sparse scenes never
        // touch the search header
        if (ring_scene(P, PASS, outer) && ring_active(P)) {
            if (ring_tile<PASS, SCAT, TW>(reinterpret_cast<const typename Col<PASS, false, false, 0>::InT *>(in),
                                          reinterpret_cast<typename Col<PASS, false, false, 0>::OutT *>(out), P,
                                          &sc, smem, &tmap, tile, outer, kt))
                return;
            __syncthreads();   // the search's shared memory and barrier are free again
        }
    }
    col_tma_run<PASS, FW, SCAT, CMP, TW>(&tmap, &tmap1, in, out, P, &sc, smem, tile, outer, kt);
}

// Columns too long for shared memory: per-CTA stack slab in global scratch,
// persistent over tiles.
template <int PASS, bool S2W, bool EW, int FW, bool SCAT>
__global__ void __launch_bounds__(kColThreads, kColMinBlocks) k_column_gstack(const typename Col<PASS, S2W, EW, FW>::InT *__restrict__ in,
                                                        typename Col<PASS, S2W, EW, FW>::OutT *__restrict__ out,
                                                        typename Col<PASS, S2W, EW, FW>::EntT *gstack,
                                                        const ColParams P, const __grid_constant__ ScatterTab sc) {
    extern __shared__ __align__(128) unsigned char smem[];
    using EntT = typename Col<PASS, S2W, EW, FW>::EntT;
    EntT *stk = gstack + (size_t)blockIdx.x * P.L * 32;
    int *meta = reinterpret_cast<int *>(smem);
    for (long long t = blockIdx.x; t < P.ntiles; t += gridDim.x) {
        column_tile<PASS, S2W, EW, FW, false, SCAT>(in, out, stk, meta, P, t, &sc);
        __syncthreads();
    }
}

#ifndef VX_STREAM_WARPS
#define VX_STREAM_WARPS 28
#endif
constexpr int kWarpCtaThreads = 32 * VX_STREAM_WARPS;   // k_pass3_stream CTA: one per SM

// ---- pass 3 with one warp per tile (few occupied slices) ----------------------
// A warp owns a whole 32-column tile: the m candidate rows (occupied slices,
// read on the device) stream through registers as 128-byte LDG rows, 8 in
// flight; the 32 column hulls are built in one sequential sweep (edt.py:253-276
// with no bands and no merges) and all L query rows are walked (edt.py:300-
// 317).  Only the hulls live in shared memory: the first kStreamCap entries of
// every column stack, the rest spill to a per-warp slab of global scratch
// (rare: hulls are short when few slices are occupied).  No CTA barrier: 32
// independent warps per SM.  Stack entry (x << yzb) | (y << zb | z): the output
// site needs no re-read; F = x^2 + (j - y)^2 + (k - z)^2.
// Runs when m <= P.stream_max; otherwise it exits and the banded
// k_column_tma (launched right after it) does the pass.
constexpr int kStreamCap = VX_STREAM_CAP;
#ifndef VX_WALK_UNROLL
#define VX_WALK_UNROLL 4
#endif
#ifndef VX_STREAM_STCS
#define VX_STREAM_STCS 1
#endif
constexpr int kWalkUnroll = VX_WALK_UNROLL;   // query-walk rows per loop trip

// the one-warp pass 3 needs enough tiles to keep its warps busy: each walks its
// tile alone (VX_STREAM_MIN_TILES overrides; default 16 per SM)
inline long long stream_min_tiles() {
    static const long long v = [] {
        const char *e = getenv("VX_STREAM_MIN_TILES");
        return e ? atoll(e) : 16LL * num_sms();
    }();
    return v;
}

#ifndef VX_STREAM_LDCS
#define VX_STREAM_LDCS 1
#endif
// candidate rows are read once per pass
__device__ __forceinline__ uint32_t cand_load(const uint32_t *p) {
#if VX_STREAM_LDCS
    return __ldcs(p);
#else
    return __ldg(p);
#endif
}

template <typename FT, typename PT, int C512>
__global__ void __launch_bounds__(kWarpCtaThreads, 1) k_pass3_stream(const uint32_t *__restrict__ in,
                                                                     int32_t *__restrict__ out,
                                                                     uint32_t *__restrict__ ovf, const ColParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int U = VX_STREAM_U;   // candidate rows in flight per lane
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int m = __ldg(P.hdr);
    if (m > P.stream_max) return;
    const bool all_rows = m == P.L;
    const int mp = (m + U - 1) / U * U;   // the list padded to whole batches (-1 = no row)
    uint32_t *sst = reinterpret_cast<uint32_t *>(smem) + (size_t)w * kStreamCap * 32 + lane;
    // candidate rows, staged once per CTA (every tile of the pass scans the same list)
    int *rows_s = reinterpret_cast<int *>(smem + (size_t)nw * kStreamCap * 32 * 4);
    for (int t = threadIdx.x; t < mp; t += blockDim.x) rows_s[t] = t < m ? (all_rows ? t : __ldg(P.xs + t)) : -1;
    __syncthreads();
    const long long gw = (long long)blockIdx.x * nw + w;
    uint32_t *gst = ovf + gw * (long long)max(P.L - kStreamCap, 0) * 32 + lane - (long long)kStreamCap * 32;
    auto ent = [&](int i) -> uint32_t { return i < kStreamCap ? sst[i * 32] : gst[(long long)i * 32]; };
    auto put = [&](int i, uint32_t e) {
        VX_ASSERT(i >= 0 && i < P.L, "stream hull slot");
        if (i < kStreamCap) sst[i * 32] = e;
        else gst[(long long)i * 32] = e;
    };
    // Stack entry (x << eb) | code: F = x^2 + (j - y)^2 + (k - z)^2 decodes and
    // the walk's sites need no re-read.
    // C512: the 512^3 single-scene grid, whose strides and shifts are constants
    const uint32_t eb = C512 ? 18u : (uint32_t)P.yzb;
    const uint32_t zb = C512 ? 9u : (uint32_t)P.zb, zmask = C512 ? 511u : P.zmask, ymask = C512 ? 511u : P.ymask;
    const long long plane = C512 ? 262144LL : P.plane, splane = C512 ? 262144LL : P.splane;
    const int nz = C512 ? 512 : P.nz, L = C512 ? 512 : P.L;
    constexpr FT kNever = sizeof(FT) == 4 ? (FT)0x7fffffff : (FT)0x7fffffffffffffffLL;
    const long long step = (long long)gridDim.x * nw;
    const int nkt = C512 ? 16 : P.nkt;
    const uint32_t ssp = (uint32_t)splane;   // row offsets fit 32 bits (int32 sites)
#if VX_P3S_DYN
    // tiles after each warp's first come from a counter (hdr[32], zeroed with
    // the occupied-slice list): deep-hull tiles do not hold up a static share
    int *tctr = const_cast<int *>(P.hdr) + 32;
    auto next_tile = [&]() -> long long {
        int t = 0;
        if (lane == 0) t = atomicAdd(tctr, 1);
        return step + __shfl_sync(0xffffffffu, t, 0);
    };
    for (long long tile = gw; tile < P.ntiles; tile = next_tile()) {
#else
    for (long long tile = gw; tile < P.ntiles; tile += step) {
#endif
        const int kt = (int)(tile % nkt);
        const long long outer = tile / nkt;
        const int scene = C512 ? 0 : (int)(outer / P.nyl);
        const int jl = (int)(outer - (long long)scene * P.nyl);
        const int jq = C512 ? jl : P.j0 + jl;
        const int k = kt * 32 + lane;
        const unsigned am = C512 ? 0xffffffffu : __ballot_sync(0xffffffffu, k < nz);
        if (k >= nz) continue;   // lanes only; the votes below use am
        const long long base = (long long)scene * P.nvox + (long long)jl * nz + k;
        const uint32_t *src = in + base;
        VX_PTW(tile, 0);
        VX_PTW(tile, 1);
        auto wof = [&](uint32_t v) -> uint32_t {   // (j - y)^2 + (k - z)^2 of an s2 code
            const uint32_t dy = (uint32_t)(jq - (int)((v >> zb) & ymask)), dz = (uint32_t)(k - (int)(v & zmask));
            return dy * dy + dz * dz;   // < 2^wb (mod-2^32 arithmetic is exact)
        };
        int n = 0, ya = 0, yb = 0;
        FT Fa = 0, Fb = 0;
        // SPILL: some lane's stack may pass kStreamCap in this batch (checked
        // once per batch of U rows: a batch grows a stack by at most U); the
        // other batches touch shared memory only, with no per-access branch
        auto consume = [&](uint32_t v, int yc, auto spill) {
            constexpr bool SPILL = decltype(spill)::value;
            if (v == 0xffffffffu) return;
            const uint32_t wc = wof(v);
            const uint32_t ec = ((uint32_t)yc << eb) | v;
            const FT Fc = (FT)yc * (FT)yc + (FT)wc;
            while (n >= 2 && dominated<FT, PT>(ya, Fa, yb, Fb, yc, Fc)) {
                --n;
                yb = ya;
                Fb = Fa;
                if (n >= 2) {
                    const uint32_t e = SPILL ? ent(n - 2) : sst[(n - 2) * 32];
                    ya = (int)(e >> eb);
                    Fa = (FT)ya * (FT)ya + (FT)wof(e);
                }
            }
            if (SPILL) put(n, ec);
            else sst[n * 32] = ec;
            ya = yb;
            Fa = Fb;
            yb = yc;
            Fb = Fc;
            ++n;
        };
        // whole batches of U rows (the padded tail loads nothing)
        for (int t0 = 0; t0 < mp; t0 += U) {
            uint32_t v[U];
            int yr[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                yr[u] = rows_s[t0 + u];
                v[u] = yr[u] >= 0 ? cand_load(src + (uint32_t)yr[u] * ssp) : 0xffffffffu;
            }
            if (__any_sync(am, n + U > kStreamCap)) {
#pragma unroll
                for (int u = 0; u < U; ++u) consume(v[u], yr[u], std::true_type());
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) consume(v[u], yr[u], std::false_type());
            }
        }
#ifdef VX_PHASE_TIMING
        {   // hull size (max over the warp's columns) for tools/phase_timing
            int hmax = n;
            for (int d = 16; d; d >>= 1) hmax = max(hmax, __shfl_xor_sync(am, hmax, d));
            if (lane == __ffs(am) - 1 && g_phase_buf) g_phase_buf[(size_t)tile * 8 + 7] = (unsigned long long)hmax;
        }
#endif
        VX_PTW(tile, 2);
        // ---- queries: first minimiser at every row, stepped walk (edt.py:300-317)
        int32_t *dst = out + base;
        auto xof = [&](uint32_t e) -> int { return (int)(e >> eb); };
        auto Fof = [&](uint32_t e) -> FT {
            const FT x = (FT)(int)(e >> eb);
            return x * x + (FT)wof(e);
        };
        auto site_of = [&](uint32_t e) -> int32_t {   // edt.py:417
            return (int32_t)((long long)(e >> eb) * plane + (long long)((e >> zb) & ymask) * nz + (long long)(e & zmask));
        };
        int pos = 0, yc = 0, ys = 0;
        FT Fc = 0, Fs = 0;
        int32_t ocur = -1;   // no candidate in the column (edt.py:295-299)
        uint32_t sent = 0;
        bool has = false;
        if (n > 0) {
            const uint32_t c0 = ent(0);
            yc = xof(c0);
            Fc = Fof(c0);
            ocur = site_of(c0);
            has = n > 1;
            if (has) {
                sent = ent(1);
                ys = xof(sent);
                Fs = Fof(sent);
            }
        }
#if VX_P3S_WPF
        uint32_t snext = n > 2 ? ent(2) : 0u;   // the successor's successor, loaded a switch ahead
#endif
        FT dN = has ? Fs - Fc : kNever;
        FT tt = has ? (FT)2 * (FT)(ys - yc) : (FT)0;
        // rows before the warp's first switch are stores only: the successor is
        // strictly closer from row dN / tt + 1 on (dN < y * tt, tt > 0)
        int y0 = L;
        if (has) y0 = dN < 0 ? 0 : (int)min((FT)L, dN / tt + 1);
        y0 = VX_P3S_ENDS ? __reduce_min_sync(am, y0) : 0;
        int y = 0;
#if VX_STREAM_STCS
#define VX_P3ST(p, v) __stcs((p), (v))   // evict-first: the sites are not re-read by this pass
#else
#define VX_P3ST(p, v) (*(p) = (v))
#endif
        for (; y + 4 <= y0; y += 4, dst += 4 * splane) {
            VX_P3ST(dst, ocur);
            VX_P3ST(dst + splane, ocur);
            VX_P3ST(dst + 2 * splane, ocur);
            VX_P3ST(dst + 3 * splane, ocur);
        }
        for (; y < y0; ++y, dst += splane) VX_P3ST(dst, ocur);
        FT rhs = (FT)y * tt;
        auto row = [&](int yy) {
            if (dN < rhs) {   // successor strictly closer at row yy (edt.py:311)
                uint32_t cur;
                do {
                    cur = sent;
                    yc = ys;
                    Fc = Fs;
                    ++pos;
                    has = pos + 1 < n;
                    if (has) {
#if VX_P3S_WPF
                        sent = snext;
                        if (pos + 2 < n) snext = ent(pos + 2);
#else
                        sent = ent(pos + 1);
#endif
                        ys = xof(sent);
                        Fs = Fof(sent);
                    }
                } while (has && better<FT>(ys, Fs, yc, Fc, yy));
                ocur = site_of(cur);
                dN = has ? Fs - Fc : kNever;
                tt = has ? (FT)2 * (FT)(ys - yc) : (FT)0;
                rhs = (FT)yy * tt;
            }
            VX_P3ST(dst, ocur);
            dst += splane;
            rhs += tt;
        };
        // rows where some lane may still switch; once every lane sits on its
        // last vertex the rest are stores only
        for (; y + kWalkUnroll <= L; y += kWalkUnroll) {
            if (VX_P3S_ENDS && !__any_sync(am, has)) break;
#pragma unroll
            for (int u = 0; u < kWalkUnroll; ++u) row(y + u);
        }
        if (__any_sync(am, has)) {
            for (; y < L; ++y) row(y);
        } else {
            for (; y + 4 <= L; y += 4, dst += 4 * splane) {
                VX_P3ST(dst, ocur);
                VX_P3ST(dst + splane, ocur);
                VX_P3ST(dst + 2 * splane, ocur);
                VX_P3ST(dst + 3 * splane, ocur);
            }
            for (; y < L; ++y, dst += splane) VX_P3ST(dst, ocur);
        }
#undef VX_P3ST
        VX_PTW(tile, 3);
        VX_PTW(tile, 4);
        VX_PTW(tile, 5);
        VX_PTW(tile, 6);
    }
#if VX_P3S_DYN
    // the last warp out re-arms the counter (hdr[33] counts finished warps), so
    // a later launch on the same list starts from zero as well
    if (lane == 0 && atomicAdd(tctr + 1, 1) == (int)(gridDim.x * nw) - 1) {
        tctr[0] = 0;
        tctr[1] = 0;
    }
#endif
}

int bits_of(long long v) {  // bits to hold values 0..v
    int b = 0;
    while (v > 0) { ++b; v >>= 1; }
    return b;
}

int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

constexpr size_t kSmemLimit = 227 * 1024;

// k_pass3_stream: its stack entries fit 32 bits, and its dynamic shared
// memory (the warps' stacks plus the row list padded to whole batches)
inline bool stream_bits_ok(const EdtPlan &p) {
    return p.xb + p.yb + p.zb <= 32;
}
inline size_t stream_smem(int L) {
    return (size_t)VX_STREAM_WARPS * kStreamCap * 32 * 4 + (size_t)(L + VX_STREAM_U) * 4;
}

// windowed search (ring_tile): VX_RING=0 disables it, VX_RING_CAP sets the
// largest search radius (rows) before a tile goes back to the banded kernel,
// VX_RING_MIN the fraction (percent) of occupied slices from which a scene counts as dense
inline int ring_cap() {
    const char *e = getenv("VX_RING_CAP");
    return e ? std::max(1, std::min(atoi(e), 1024)) : 64;
}
inline int ring_budget(int pass) {
    const char *e = getenv(pass == 2 ? "VX_RING_BUDGET2" : "VX_RING_BUDGET3");
    return e ? std::max(1, atoi(e)) : 24;
}
inline bool ring_enabled() {
    const char *e = getenv("VX_RING");
    return !(e && atoi(e) == 0);
}
inline int ring_min_for(int nx) {
    const char *e = getenv("VX_RING_MIN");
    const int pct = e ? atoi(e) : 90;
    return std::max(1, (int)(((long long)nx * pct + 99) / 100));
}
// keys (w << rb | row) plus the largest window offset ((cap + 4)^2 << rb)
// stay below the invalid key, which plus that offset stays below 2^32
constexpr int kRingBlock = 4;
inline uint32_t ring_kinv(int rb) {
    const long long c = ring_cap() + kRingBlock + 1;
    return (uint32_t)(0xFFFFFFFFLL - ((c * c) << rb));
}
// may this call use the windowed search at all (host side; the device gates it per call)?
bool ring_possible(const EdtPlan &p, const SparseRows *sp) {
    return sp && sp->fails && ring_enabled() && p.tma2 && p.tma3 &&
           (sp->m_hint < 0 || sp->m_hint >= ring_min_for(p.nx));
}
bool ring_fits(const EdtPlan &p, int pass, int L) {
    const int rb = kRingRb;
    const long long wmax = pass == 2 ? (long long)(p.nz - 1) * (p.nz - 1)
                                     : (long long)(p.ny - 1) * (p.ny - 1) + (long long)(p.nz - 1) * (p.nz - 1);
    const long long c = ring_cap() + kRingBlock + 1;
    return L <= (1 << rb) && ((wmax + c * c + 1) << rb) < (long long)ring_kinv(rb);
}

// pass 2: `outer` counts slices (nscenes * local nx); pass 3: `outer` counts
// (scene, local j) with nyl rows of j starting at global row j0.
ColParams col_params(const EdtPlan &p, int pass, long long nouter, int nyl, int j0) {
    ColParams P;
    P.nx = p.nx; P.ny = p.ny; P.nz = p.nz;
    P.L = pass == 2 ? p.ny : p.nx;
    P.B = pass == 2 ? p.B2 : p.B3;
    P.W = pass == 2 ? p.W2 : p.W3;
    P.nkt = (p.nz + 31) / 32;
    P.ntiles = (long long)P.nkt * nouter;
    P.nyl = nyl;
    P.j0 = j0;
    P.splane = (long long)nyl * p.nz;
    P.zb = p.zb;
    P.yzb = p.yb + p.zb;
    P.zmask = p.zb >= 32 ? 0xffffffffu : ((1u << p.zb) - 1u);
    P.ymask = p.yb >= 32 ? 0xffffffffu : ((1u << p.yb) - 1u);
    P.plane = (long long)p.ny * p.nz;
    P.nvox = P.splane * p.nx;
    P.wb = p.wb;
    P.wmask = p.wb >= 32 ? 0xffffffffu : ((1u << p.wb) - 1u);
    P.sflag = nullptr;
    P.xs = nullptr;
    P.hdr = nullptr;
    P.stream_max = -1;
    P.mcount = nullptr;
    P.sflag3 = nullptr;
    P.ring_min = 0x7fffffff;
    P.s16 = pass == 2 && p.s1_16;
    P.rhdr = nullptr;
    P.fslot = pass == 2 ? 0 : 1;
    P.nkt2 = (p.nz + p.tw2 - 1) / p.tw2;
    P.ny2 = p.ny;
    P.rb = kRingRb;
    P.ring_cap = ring_cap();
    P.ring_budget = ring_budget(pass);
    P.kinv = ring_kinv(P.rb);
    P.boxh = std::min(P.L, 256);
    P.rows_alloc = (P.L + P.boxh - 1) / P.boxh * P.boxh;
    return P;
}

// raise the dynamic shared-memory ceiling once per kernel and device (the
// per-launch size is the launch parameter); keeps the launch path cheap
template <typename K>
cudaError_t allow_smem(K kern) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(reinterpret_cast<const void *>(kern), dev);
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return cudaSuccess;
    // static shared memory counts against the same 227 KB
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSmemLimit - fa.sharedSizeBytes));
    if (e == cudaSuccess) done.insert(key);
    return e;
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// TMA view of a column pass input: 3D (k, y, slice) for pass 2, 4D
// (k, j, x, scene) for pass 3; box = 32 columns x boxh rows.
bool make_tmap(CUtensorMap *m, const void *in, const EdtPlan &p, int pass, long long nouter, int nyl,
               int boxh, int boxw = 32) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    const int es = pass == 2 && p.s1_16 ? 2 : 4;   // int16 line sites (EdtPlan::s1_16)
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
    cuuint32_t rank;
    if (pass == 2) {
        rank = 3;
        dims[0] = p.nz; dims[1] = p.ny; dims[2] = (cuuint64_t)nouter;
        strides[0] = (cuuint64_t)p.nz * es; strides[1] = (cuuint64_t)p.ny * p.nz * es;
        box[0] = (cuuint32_t)boxw; box[1] = boxh; box[2] = 1;
    } else {
        rank = 4;
        const long long nscenes = nouter / nyl;
        dims[0] = p.nz; dims[1] = nyl; dims[2] = p.nx; dims[3] = (cuuint64_t)nscenes;
        strides[0] = (cuuint64_t)p.nz * 4; strides[1] = (cuuint64_t)nyl * p.nz * 4;
        strides[2] = (cuuint64_t)p.nx * nyl * p.nz * 4;
        box[0] = (cuuint32_t)boxw; box[1] = 1; box[2] = boxh; box[3] = 1;
    }
    CUresult r = enc(m, es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32, rank, const_cast<void *>(in), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int PASS, bool S2W, bool EW, int FW, bool SCAT>
cudaError_t launch_col(const void *in, void *out, void *gstack, const EdtPlan &p, long long nouter,
                       int nyl, int j0, const ScatterTab &sc, cudaStream_t st, const SparseRows *sp) {
    using C = Col<PASS, S2W, EW, FW>;
    ColParams P = col_params(p, PASS, nouter, nyl, j0);
    if (sp) {   // the caller only passes one when both column passes are TMA-staged
        if (PASS == 2) P.sflag = sp->sflag;
        // pass 2 maps CTAs through the list only for a single scene (a batch
        // skips its empty slices by flag); pass 3 reads each scene's own list
        if (PASS == 3 || nouter == p.nx) {
            P.xs = sp->xs;
            P.hdr = sp->hdr;
        }
    }
    if (P.ntiles == 0) return cudaSuccess;
    const dim3 block(32, P.B);
    const bool gs = PASS == 2 ? p.gstack2 : p.gstack3;
    const bool staged = PASS == 2 ? p.tma2 : p.tma3;
    if constexpr (!S2W && !EW) {
        if (staged && !gs) {
            CUtensorMap m, m1;
            const bool cmp = PASS == 3 && P.xs != nullptr;
            // long columns (L > 512): 16-column tiles, so a 1024-row tile is
            // 64 KB and three CTAs share an SM (make_plan: tw2 / tw3)
            const int tw = PASS == 2 ? p.tw2 : p.tw3;
            if (make_tmap(&m, in, p, PASS, nouter, nyl, P.boxh, tw) &&
                (!cmp || make_tmap(&m1, in, p, PASS, nouter, nyl, 1, tw))) {
                if (!cmp) m1 = m;
                if constexpr (PASS == 3 && !SCAT) {
                    // few occupied slices: one warp per tile (k_pass3_stream) when
                    // m <= stream_max, decided on the device; s1 (gstack here) is
                    // its spill slab
                    const long long spill = std::min<long long>(P.ntiles, (long long)num_sms() * VX_STREAM_WARPS) *
                                            std::max(P.L - kStreamCap, 0) * 32 * 4;
                    // only with tiles enough for >= 16 warps per SM: each warp walks
                    // its tile alone, so small grids keep the banded kernel
                    const int mode = sp ? sp->p3_mode : 0;
                    const size_t ssm = stream_smem(P.L);   // stacks + row list
                    if (mode != 2 && cmp && gstack && nouter == nyl && stream_bits_ok(p) &&
                        spill <= (long long)p.s1_bytes && P.ntiles >= (long long)stream_min_tiles() && ssm <= kSmemLimit) {
                        const char *sm = getenv("VX_STREAM_MAX");
                        P.stream_max = mode == 1 ? 0x7fffffff : sm ? atoi(sm) : std::min(kStreamMaxRows, P.L / 2);
                        const bool c512 = !p.fwide && !p.pwide && p.nx == 512 && p.ny == 512 && p.nz == 512 && nyl == 512 &&
                                          j0 == 0 && nouter == 512;
                        auto kern = c512 ? k_pass3_stream<typename C::FT, typename C::PT, 1>
                                         : k_pass3_stream<typename C::FT, typename C::PT, 0>;
                        cudaError_t e = allow_smem(kern);
                        if (e != cudaSuccess) return e;
                        const unsigned grid = (unsigned)std::min<long long>((P.ntiles + VX_STREAM_WARPS - 1) / VX_STREAM_WARPS, num_sms());
                        kern<<<grid, kWarpCtaThreads, ssm, st>>>(reinterpret_cast<const uint32_t *>(in),
                                                                 reinterpret_cast<int32_t *>(out),
                                                                 reinterpret_cast<uint32_t *>(gstack), P);
                        e = cudaGetLastError();
                        if (e != cudaSuccess || mode == 1) return e;   // mode 1: no banded launch
                    } else {
                        P.stream_max = -1;
                    }
                }
                const size_t smem = PASS == 2 ? p.smem2 : p.smem3;
                if (tw == 16) {   // 32 bands x 16 columns = 512 threads (two bands per warp)
                    P.nkt = (p.nz + 15) / 16;
                    P.ntiles = (long long)P.nkt * nouter;
                }
                // dense scenes first try the windowed search inside the same
                // kernel (decided per scene on the device)
                bool ring = false;
                if constexpr (FW <= 1) {
                    const int mode3 = PASS == 3 && sp ? sp->p3_mode : 0;
                    if (ring_possible(p, sp) && mode3 != 1 && ring_fits(p, PASS, P.L) && tw * P.B <= kColThreads) {
                        P.mcount = sp->hdr;
                        P.sflag3 = PASS == 3 ? sp->sflag : nullptr;
                        P.ring_min = ring_min_for(p.nx);
                        P.rhdr = sp->fails;   // zeroed by launch_pass1 of this call
                        ring = true;
                    }
                }
                // long columns (L > 512) with 32-column tiles take 32 bands =
                // 1024 threads: one CTA per SM (VX_NARROW_TILES=0)
                auto kern = tw == 16
                                ? (ring ? (cmp ? k_column_tma<PASS, FW, SCAT, true, kColThreads, 16, true>
                                               : k_column_tma<PASS, FW, SCAT, false, kColThreads, 16, true>)
                                        : (cmp ? k_column_tma<PASS, FW, SCAT, true, kColThreads, 16>
                                               : k_column_tma<PASS, FW, SCAT, false, kColThreads, 16>))
                                : P.B > kMaxBands
                                      ? (cmp ? k_column_tma<PASS, FW, SCAT, true, 1024> : k_column_tma<PASS, FW, SCAT, false, 1024>)
                                      : (ring ? (cmp ? k_column_tma<PASS, FW, SCAT, true, kColThreads, 32, true>
                                                     : k_column_tma<PASS, FW, SCAT, false, kColThreads, 32, true>)
                                              : (cmp ? k_column_tma<PASS, FW, SCAT, true, kColThreads>
                                                     : k_column_tma<PASS, FW, SCAT, false, kColThreads>));
                cudaError_t e = allow_smem(kern);
                if (e != cudaSuccess) return e;
                kern<<<(unsigned)P.ntiles, dim3(tw, P.B), smem, st>>>(m, m1, reinterpret_cast<const typename C::InT *>(in),
                                                                   reinterpret_cast<typename C::OutT *>(out), P, sc);
                return cudaGetLastError();
            }
        }
    }
    // TMA-staged kernel only: occupied-slice lists, 32 bands, int16 s1
    if (P.xs || P.B > kMaxBands || P.s16) return cudaErrorNotSupported;
    P.rows_alloc = P.L;
    if (!gs) {
        const size_t smem = (size_t)P.L * 32 * sizeof(typename C::EntT) + (size_t)(3 * P.B * 32 + 32) * 4;
        auto kern = k_column_smem<PASS, S2W, EW, FW, SCAT>;
        cudaError_t e = allow_smem(kern);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)P.ntiles, block, smem, st>>>(
            reinterpret_cast<const typename C::InT *>(in), reinterpret_cast<typename C::OutT *>(out), P, sc);
    } else {
        const size_t smem = (size_t)(3 * P.B * 32 + 32) * 4;
        auto kern = k_column_gstack<PASS, S2W, EW, FW, SCAT>;
        cudaError_t e = allow_smem(kern);
        if (e != cudaSuccess) return e;
        const long long g = std::min<long long>(P.ntiles, p.gstack_ctas);
        kern<<<(unsigned)g, block, smem, st>>>(reinterpret_cast<const typename C::InT *>(in),
                                              reinterpret_cast<typename C::OutT *>(out),
                                              reinterpret_cast<typename C::EntT *>(gstack), P, sc);
    }
    return cudaGetLastError();
}

template <int PASS, bool SCAT>
cudaError_t dispatch_col(const void *in, void *out, void *gstack, const EdtPlan &p, long long nouter,
                         int nyl, int j0, const ScatterTab &sc, cudaStream_t st,
                         const SparseRows *sp = nullptr) {
    // narrow: u32 s2, u32 entries, int weights (the 512^3 path)
    if (!p.s2_wide && !p.e3_wide && !p.fwide && !p.pwide)
        return launch_col<PASS, false, false, 0, SCAT>(in, out, gstack, p, nouter, nyl, j0, sc, st, sp);
    // int32 weights, int64 hull-test products (the 1024^3 path)
    if (!p.s2_wide && !p.e3_wide && !p.fwide)
        return launch_col<PASS, false, false, 1, SCAT>(in, out, gstack, p, nouter, nyl, j0, sc, st, sp);
    if (!p.s2_wide && !p.e3_wide)
        return launch_col<PASS, false, false, 2, SCAT>(in, out, gstack, p, nouter, nyl, j0, sc, st, sp);
    if (!p.s2_wide)
        return launch_col<PASS, false, true, 2, SCAT>(in, out, gstack, p, nouter, nyl, j0, sc, st, sp);
    return launch_col<PASS, true, true, 2, SCAT>(in, out, gstack, p, nouter, nyl, j0, sc, st, sp);
}

}  // namespace

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

bool make_plan(int nx, int ny, int nz, EdtPlan *p, int force_global_stack) {
    if (nx <= 0 || ny <= 0 || nz <= 0) return false;
    EdtPlan q{};
    q.nx = nx; q.ny = ny; q.nz = nz;
    q.xb = bits_of(nx - 1);
    q.yb = bits_of(ny - 1);
    q.zb = bits_of(nz - 1);
    // test hooks: VX_FORCE_WIDE=1|2|3 selects the wider code paths on small
    // grids (1: int64 weights, 2: +u64 pass-3 entries, 3: +u64 s2 codes,
    // 4: int32 weights with int64 hull-test products);
    // VX_FORCE_GSTACK=1 puts the column stacks in global memory
    const char *fw = getenv("VX_FORCE_WIDE");
    const int force_wide = fw ? atoi(fw) : 0;
    const char *fg = getenv("VX_FORCE_GSTACK");
    if (fg && atoi(fg)) force_global_stack = 1;
    q.s2_wide = q.yb + q.zb > 31 || force_wide >= 3;   // keep all-ones free as the sentinel
    q.wb = bits_of((long long)(ny - 1) * (ny - 1) + (long long)(nz - 1) * (nz - 1));
    q.e3_wide = q.s2_wide || (kP3XW ? q.xb + q.wb > 32 : q.xb + q.yb + q.zb > 32) || force_wide >= 2;
    // weights: F = w + row^2 <= (nx-1)^2+(ny-1)^2+(nz-1)^2; products F * L
    const double fmax = (double)(nx - 1) * (nx - 1) + (double)(ny - 1) * (ny - 1) +
                        (double)(nz - 1) * (nz - 1);
    const double lmax = (double)std::max(nx, ny);
    // int64 weights when F, or the walk's 2*L*L right-hand side, leaves int32
    // (or a test hook asks); otherwise int32 weights, and int64 products in the
    // hull test only when F*L can leave int32 (the 1024^3 grids)
    q.fwide = q.e3_wide || (force_wide >= 1 && force_wide <= 3) || fmax >= 2147483647.0 ||
              (2.0 * lmax * lmax >= 2147483647.0);
    q.pwide = !q.fwide && (2.0 * fmax * lmax >= 2147483647.0 || force_wide == 4);
    auto bands = [](int L, int &B, int &W) {
        B = std::min(kMaxBands, pow2ceil((L + VX_BAND_ROWS - 1) / VX_BAND_ROWS));
        W = (L + B - 1) / B;
    };
    bands(ny, q.B2, q.W2);
    bands(nx, q.B3, q.W3);
    const size_t e2 = (q.s2_wide ? 8 : 4);  // pass-2 entry == s2 code width
    const size_t e3 = (q.e3_wide ? 8 : 4);
    const size_t meta2 = (size_t)(3 * q.B2 * 32 + 32) * 4;
    const size_t meta3 = (size_t)(3 * q.B3 * 32 + 32) * 4;
    const size_t st2 = (size_t)ny * 32 * e2, st3 = (size_t)nx * 32 * e3;
    q.gstack2 = force_global_stack || st2 + meta2 > kSmemLimit;
    q.gstack3 = force_global_stack || st3 + meta3 > kSmemLimit;
    q.smem2 = q.gstack2 ? meta2 : st2 + meta2;
    q.smem3 = q.gstack3 ? meta3 : st3 + meta3;
    // TMA tile staging: 32-bit codes, 16-byte row strides (nz % 4 == 0), and
    // the box-rounded tile (+ mbarrier) must fit; VX_NO_TMA=1 disables it
    const char *nt = getenv("VX_NO_TMA");
    const bool tma_ok = !(nt && atoi(nt)) && nz % 4 == 0;
    auto staged_bytes = [](int L, int B, int tw = 32) {
        const int boxh = std::min(L, 256);
        const size_t rows = (size_t)(L + boxh - 1) / boxh * boxh;
        return rows * tw * 4 + (size_t)(3 * B * tw + tw) * 4 + 16;
    };
    const size_t sb2 = staged_bytes(ny, q.B2), sb3 = staged_bytes(nx, q.B3);
    q.tma2 = tma_ok && !q.s2_wide && !q.gstack2 && sb2 <= kSmemLimit;
    q.tma3 = tma_ok && !q.s2_wide && !q.e3_wide && !q.gstack3 && sb3 <= kSmemLimit;
    // TMA-staged long columns: up to 32 bands, as 16-column tiles (32 x 16 =
    // 512 threads; a 1024-row tile is 64 KB, three CTAs per SM) or, with
    // VX_NARROW_TILES=0, 32-column tiles (1024 threads, one CTA per SM)
    const char *ntl = getenv("VX_NARROW_TILES");
    const bool narrow_ok = !(ntl && atoi(ntl) == 0);
    q.tw2 = q.tw3 = 32;
    // (16-column tiles for L <= 512 measured: +1-3 %, 6 CTAs/SM buy nothing there)
    auto widen = [&](int L, bool tma, int &B, int &W, size_t &smem, int &tw) {
        if (!tma || L <= 512) return;
        const int B32 = std::min(32, pow2ceil((L + VX_BAND_ROWS - 1) / VX_BAND_ROWS));
        if (B32 <= B) return;
        if (narrow_ok && B32 * 16 <= kColThreads && 3 * staged_bytes(L, B32, 16) <= kSmemLimit) {
            tw = 16;
        } else if (staged_bytes(L, B32) > kSmemLimit) {
            return;
        }
        B = B32;
        W = (L + B - 1) / B;
        smem = staged_bytes(L, B, tw);
    };
    if (q.tma2) q.smem2 = sb2;
    if (q.tma3) q.smem3 = sb3;
    widen(ny, q.tma2, q.B2, q.W2, q.smem2, q.tw2);
    widen(nx, q.tma3, q.B3, q.W3, q.smem3, q.tw3);
    q.gstack_ctas = 2 * num_sms();
    size_t gs = 0;
    if (q.gstack2) gs = std::max(gs, (size_t)q.gstack_ctas * st2);
    if (q.gstack3) gs = std::max(gs, (size_t)q.gstack_ctas * st3);
    const size_t n = (size_t)nx * ny * nz;
    q.s1_bytes = (n * 4 + 255) & ~(size_t)255;
    q.s2_bytes = (n * (q.s2_wide ? 8 : 4) + 255) & ~(size_t)255;
    q.gstack_bytes = gs;
    // pass 1 writes int16 line sites when pass 2 stages its tiles by TMA and
    // widens them in shared memory: half the bytes of
    // pass 1's writes and of pass 2's tile loads.  Needs 16-byte rows (nz % 8)
    // and sites below 2^15; VX_S1_16=0 keeps int32
    const char *s16 = getenv("VX_S1_16");
    // (pass-2 columns: L = ny a power of two in [64, 1024] in bands of 32 rows --
    // the in-place widening, widen16, relies on that shape)
    q.s1_16 = q.tma2 && !q.e3_wide && q.W2 == 32 && ny >= 64 && ny <= 1024 && (ny & (ny - 1)) == 0 &&
              nz % 8 == 0 && nz <= 32767 && !(s16 && atoi(s16) == 0);
    *p = q;
    return true;
}


template <typename T>
cudaError_t launch_pass1_t(const uint8_t *occ, T *s1, long long nslices, int ny, int nz,
                           cudaStream_t st, const SparseRows *sp) {
    const long long nlines = nslices * ny;
    if (nlines == 0) return cudaSuccess;
    const uint8_t *sflag = sp ? sp->sflag : nullptr;
    const int *xs = sp ? sp->xs : nullptr, *hdr = sp ? sp->hdr : nullptr;
    unsigned grid = (unsigned)((nlines + 7) / 8);
    unsigned grid2 = (unsigned)((nlines + 15) / 16);
    if (xs) {   // persistent: VX_P1_WAVES x 8 CTAs of 256 threads per SM
        grid = (unsigned)std::min<long long>(grid, (long long)num_sms() * 8 * VX_P1_WAVES);
        grid2 = (unsigned)std::min<long long>(grid2, (long long)num_sms() * 8 * VX_P1_WAVES);
    }
    const bool vec = (nz % 4 == 0) && ((uintptr_t)occ % 16 == 0) && ((uintptr_t)s1 % 16 == 0);
    // the windowed search's header (hand-back counts, k-line statistics) starts
    // at zero for this call; pass 1 counts the empty k-lines into it
    int *ls = nullptr;
    if (sp && sp->fails && ring_enabled() &&
        (sp->m_hint < 0 || sp->m_hint >= ring_min_for((int)(nslices / std::max(sp->nscenes, 1))))) {
        ls = sp->fails;
        cudaError_t e = cudaMemsetAsync(ls, 0, 16, st);
        if (e != cudaSuccess) return e;
    }
    if (vec && nz <= 128) k_pass1_v4<1, 2, T><<<grid2, 256, 0, st>>>(occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else if (vec && nz <= 256) k_pass1_v4<2, 2, T><<<grid2, 256, 0, st>>>(occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else if (vec && nz <= 512 && xs && VX_P1_LPW512 == 2) k_pass1_v4<4, 2, T><<<grid2, 256, 0, st>>>(occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else if (vec && nz % 16 == 0 && nz <= 512 && VX_P1_X16)   // persistent: 6 CTAs of 8 warps per SM
        (nz % 512 == 0 ? k_pass1_x16<1, true, T> : k_pass1_x16<1, false, T>)
            <<<(unsigned)std::min<long long>(grid, (long long)num_sms() * 6), 256, 0, st>>>(
            occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else if (vec && nz <= 512) k_pass1_v4<4, 1, T><<<grid, 256, 0, st>>>(occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else if (vec && nz % 16 == 0 && nz <= 1024 && VX_P1_X16)
        (nz % 512 == 0 ? k_pass1_x16<2, true, T> : k_pass1_x16<2, false, T>)
            <<<(unsigned)std::min<long long>(grid, (long long)num_sms() * 6), 256, 0, st>>>(
            occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else if (vec && nz <= 1024) k_pass1_v4<8, 1, T><<<grid, 256, 0, st>>>(occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else if (vec && nz <= 2048) k_pass1_v4<16, 1, T><<<grid, 256, 0, st>>>(occ, s1, nlines, nz, sflag, ny, xs, hdr, ls);
    else k_pass1_generic<T><<<grid, 256, 0, st>>>(occ, s1, nlines, nz, sflag, ny);
    return cudaGetLastError();
}

cudaError_t launch_pass1(const uint8_t *occ, void *s1, long long nslices, int ny, int nz,
                         cudaStream_t st, const SparseRows *sp, bool s16) {
    if (s16) {   // int16 line sites (EdtPlan::s1_16)
        if (nz % 8 != 0 || nz > 32767) return cudaErrorInvalidValue;
        return launch_pass1_t(occ, static_cast<int16_t *>(s1), nslices, ny, nz, st, sp);
    }
    return launch_pass1_t(occ, static_cast<int32_t *>(s1), nslices, ny, nz, st, sp);
}

cudaError_t launch_pass2(const int32_t *s1, void *s2, void *gstack, const EdtPlan &p,
                         long long nslices, cudaStream_t st, const SparseRows *sp) {
    return dispatch_col<2, false>(s1, s2, gstack, p, nslices, p.ny, 0, ScatterTab{}, st, sp);
}

cudaError_t launch_pass2_scatter(const int32_t *s1, const ScatterTab &sc, void *gstack, const EdtPlan &p,
                                 long long nslices, cudaStream_t st, const SparseRows *sp) {
    return dispatch_col<2, true>(s1, nullptr, gstack, p, nslices, p.ny, 0, sc, st, sp);
}

cudaError_t launch_pass3(const void *s2, int32_t *site, void *gstack, const EdtPlan &p,
                         int nscenes, int j0, int nyl, cudaStream_t st, const SparseRows *sp) {
    return dispatch_col<3, false>(s2, site, gstack, p, (long long)nscenes * nyl, nyl, j0, ScatterTab{}, st, sp);
}

// ---- occupied-slice list ------------------------------------------------------
// per slice: does it hold any occupied voxel?
__global__ void __launch_bounds__(256) k_slice_flags(const uint8_t *__restrict__ occ, long long plane,
                                                     uint8_t *__restrict__ sflag) {
    const uint8_t *src = occ + (long long)blockIdx.x * plane;
    bool any = false;
    if ((plane & 15) == 0 && ((uintptr_t)occ & 15) == 0) {
        const uint4 *v = reinterpret_cast<const uint4 *>(src);
        const long long nv = plane >> 4;
        for (long long q0 = threadIdx.x; q0 < nv && !any; q0 += 8 * blockDim.x) {
            uint32_t acc = 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {   // 8 independent 16-byte loads in flight
                const long long q = q0 + (long long)u * blockDim.x;
                if (q < nv) {
                    const uint4 w = __ldg(v + q);
                    acc |= w.x | w.y | w.z | w.w;
                }
            }
            any = acc != 0u;
        }
    } else {
        for (long long q = threadIdx.x; q < plane && !any; q += blockDim.x) any = src[q] != 0;
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) sflag[blockIdx.x] = any ? 1 : 0;
}

// ascending list of occupied slices (one CTA, block-wide prefix sums)
__global__ void __launch_bounds__(1024) k_slice_list(const uint8_t *__restrict__ sflag, int nslices,
                                                     int *__restrict__ xs, int *__restrict__ hdr,
                                                     int *__restrict__ m_mirror) {
    // one CTA per scene of a batch: its flags, list and count
    sflag += (size_t)blockIdx.x * nslices;
    xs += (size_t)blockIdx.x * nslices;
    hdr += blockIdx.x;
    if (blockIdx.x) m_mirror = nullptr;
    __shared__ int wsum[32];
    __shared__ int base_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    for (int c0 = 0; c0 < nslices; c0 += blockDim.x) {
        const int x = c0 + threadIdx.x;
        const int f = (x < nslices && sflag[x]) ? 1 : 0;
        const unsigned m = __ballot_sync(VX_FULL_MASK, f);
        const int wpre = __popc(m & ((1u << lane) - 1u));
        if (lane == 0) wsum[warp] = __popc(m);
        __syncthreads();
        int wbase = 0, tot = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
            if (q < warp) wbase += wsum[q];
            tot += wsum[q];
        }
        const int base = base_s;
        if (f) xs[base + wbase + wpre] = x;
        __syncthreads();
        if (threadIdx.x == 0) base_s = base + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        hdr[0] = base_s;
        if (gridDim.x == 1) hdr[32] = hdr[33] = 0;   // single scene: k_pass3_stream's tile counters
        if (m_mirror) *(volatile int *)m_mirror = base_s;   // host-mapped hint
    }
}

// slice flags from a grid's touched list (every voxel written since its last
// reset, so every occupied voxel): a few hundred thousand entries instead of
// a pass over the whole occupancy array
__global__ void __launch_bounds__(1024) k_slice_flags_touched(const int32_t *__restrict__ touched,
                                                             const DevCounters *__restrict__ ctr,
                                                             const uint8_t *__restrict__ occ, long long plane,
                                                             long long n, int nx, uint8_t *__restrict__ sflag) {
    // per-CTA bitmap of slices (nx <= 32768): one global store per slice
    // and CTA instead of one per occupied voxel on a handful of hot bytes
    __shared__ unsigned bits[1024];
    const bool local = nx <= 32768;
    if (local)
        for (int w = threadIdx.x; w < (nx + 31) / 32; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    const long long nth = (long long)gridDim.x * blockDim.x;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    auto mark = [&](long long v) {
        const int i = (int)(v / plane);
        if (local) atomicOr(&bits[i >> 5], 1u << (i & 31));
        else sflag[i] = 1;
    };
    if (ctr->overflow) {   // the list is incomplete: scan every voxel
        for (long long v = tid; v < n; v += nth)
            if (occ[v]) mark(v);
    } else {
        const int cnt = ctr->touched;
        for (long long t = tid; t < cnt; t += nth) {
            const int v = touched[t];
            if (occ[v]) mark(v);
        }
    }
    if (!local) return;
    __syncthreads();
    for (int w = threadIdx.x; w < (nx + 31) / 32; w += blockDim.x)
        for (unsigned b = bits[w]; b; b &= b - 1) sflag[w * 32 + __ffs(b) - 1] = 1;
}

cudaError_t launch_slice_list_touched(const int32_t *touched, const DevCounters *ctr, const uint8_t *occ,
                                      const EdtPlan &p, const SparseRows &sp, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(const_cast<uint8_t *>(sp.sflag), 0, (size_t)p.nx, st);
    if (e != cudaSuccess) return e;
    k_slice_flags_touched<<<std::max(1, num_sms() / 4), 1024, 0, st>>>(
        touched, ctr, occ, (long long)p.ny * p.nz, (long long)p.nx * p.ny * p.nz, p.nx,
        const_cast<uint8_t *>(sp.sflag));
    k_slice_list<<<1, 1024, 0, st>>>(sp.sflag, p.nx, const_cast<int *>(sp.xs), const_cast<int *>(sp.hdr),
                                     sp.m_mirror);
    return cudaGetLastError();
}

// the list alone, when the flags were already set (by a fresh-grid finalize)
cudaError_t launch_slice_list_only(const EdtPlan &p, const SparseRows &sp, cudaStream_t st) {
    k_slice_list<<<1, 1024, 0, st>>>(sp.sflag, p.nx, const_cast<int *>(sp.xs), const_cast<int *>(sp.hdr),
                                     sp.m_mirror);
    return cudaGetLastError();
}

cudaError_t launch_slice_list(const uint8_t *occ, const EdtPlan &p, const SparseRows &sp, cudaStream_t st,
                              int nscenes) {
    k_slice_flags<<<(unsigned)(p.nx * nscenes), 256, 0, st>>>(occ, (long long)p.ny * p.nz,
                                                             const_cast<uint8_t *>(sp.sflag));
    k_slice_list<<<(unsigned)nscenes, 1024, 0, st>>>(sp.sflag, p.nx, const_cast<int *>(sp.xs), const_cast<int *>(sp.hdr),
                                     sp.m_mirror);
    return cudaGetLastError();
}

// which pass-3 kernels to launch given a predicted occupied-slice count m
// (the previous call's, read from SparseRows::m_mirror): mirrors the gates of
// launch_col.  Any mode is correct for any m; a wrong guess only costs time.
bool ring_hint_on(const EdtPlan &p, int m) {
    return ring_enabled() && (m < 0 || m >= ring_min_for(p.nx));
}

int pass3_mode_hint(const EdtPlan &p, int m) {
    if (m < 0) return 0;
    const long long ntiles = (long long)((p.nz + 31) / 32) * p.ny;
    const long long spill = std::min<long long>(ntiles, (long long)num_sms() * VX_STREAM_WARPS) *
                            std::max(p.nx - kStreamCap, 0) * 32 * 4;
    const bool ok = p.tma2 && p.tma3 && !p.gstack3 && !p.s2_wide && !p.e3_wide &&
                    stream_bits_ok(p) && spill <= (long long)p.s1_bytes &&
                    ntiles >= (long long)stream_min_tiles() && stream_smem(p.nx) <= kSmemLimit;
    if (!ok) return 2;
    const char *sm = getenv("VX_STREAM_MAX");
    const int smax = sm ? atoi(sm) : std::min(kStreamMaxRows, p.nx / 2);
    return m <= smax ? 1 : 2;
}

// the windowed search's header (fall-back counts, pass-1 k-line counts)
static size_t fail_list_bytes(const EdtPlan &, int) { return 256; }

size_t sparse_bytes(const EdtPlan &p, int nscenes) {
    const size_t sx = (size_t)p.nx * nscenes;
    return (sx + 255) / 256 * 256 + (sx * 4 + 255) / 256 * 256 + ((size_t)nscenes * 4 + 255) / 256 * 256 +
           fail_list_bytes(p, nscenes);
}

size_t scratch_bytes_for(const EdtPlan &p, int nscenes) {
    const size_t n = (size_t)p.nx * p.ny * p.nz * nscenes;
    const size_t s1b = (n * 4 + 255) & ~(size_t)255;
    const size_t s2b = (n * (p.s2_wide ? 8 : 4) + 255) & ~(size_t)255;
    return s1b + s2b + p.gstack_bytes + sparse_bytes(p, nscenes);
}

bool sparse_ok(const EdtPlan &p, int nscenes) {
    const char *ns = getenv("VX_NO_SPARSE");
    return nscenes >= 1 && p.tma2 && p.tma3 && !(ns && atoi(ns));
}

SparseRows sparse_rows_at(void *where, const EdtPlan &p, int nscenes) {
    unsigned char *b = static_cast<unsigned char *>(where);
    const size_t sx = (size_t)p.nx * nscenes;
    SparseRows sp;
    sp.sflag = b;
    sp.xs = reinterpret_cast<int *>(b + (sx + 255) / 256 * 256);
    sp.hdr = reinterpret_cast<int *>(b + (sx + 255) / 256 * 256 + (sx * 4 + 255) / 256 * 256);
    sp.fails = reinterpret_cast<int *>(b + (sx + 255) / 256 * 256 + (sx * 4 + 255) / 256 * 256 +
                                       ((size_t)nscenes * 4 + 255) / 256 * 256);
    sp.nscenes = nscenes;
    return sp;
}

cudaError_t edt_device_batched(const uint8_t *occ, int32_t *site, void *scratch,
                               const EdtPlan &p, int nscenes, cudaStream_t st) {
    // scratch = [s1 i32 N*nscenes][s2 N*nscenes][global stacks][slice list]
    unsigned char *base = static_cast<unsigned char *>(scratch);
    const size_t n = (size_t)p.nx * p.ny * p.nz * nscenes;
    int32_t *s1 = reinterpret_cast<int32_t *>(base);
    const size_t s1b = (n * 4 + 255) & ~(size_t)255;
    void *s2 = base + s1b;
    const size_t s2b = (n * (p.s2_wide ? 8 : 4) + 255) & ~(size_t)255;
    void *gs = base + s1b + s2b;
    cudaError_t e;
    if (sparse_ok(p, nscenes)) {
        const SparseRows sp = sparse_rows_at(base + s1b + s2b + p.gstack_bytes, p, nscenes);
        e = launch_slice_list(occ, p, sp, st, nscenes);
        // a batch skips its empty slices by flag in passes 1-2 (the list remap
        // is per scene); pass 3 stages each scene's occupied rows
        SparseRows spf = sp;
        if (nscenes > 1) spf.xs = nullptr, spf.hdr = nullptr;
        const long long nsl = (long long)p.nx * nscenes;
        if (e == cudaSuccess) e = launch_pass1(occ, s1, nsl, p.ny, p.nz, st, &spf, p.s1_16);
        if (e == cudaSuccess) e = launch_pass2(s1, s2, gs, p, nsl, st, &sp);
        // pass 3 of the sparse path: s1 is dead by now and serves as the
        // spill slab of the per-warp column stacks (single scene)
        if (e == cudaSuccess) e = launch_pass3(s2, site, s1, p, nscenes, 0, p.ny, st, &sp);
        return e;
    }
    e = launch_pass1(occ, s1, (long long)p.nx * nscenes, p.ny, p.nz, st, nullptr, p.s1_16);
    if (e != cudaSuccess) return e;
    e = launch_pass2(s1, s2, gs, p, (long long)p.nx * nscenes, st);
    if (e != cudaSuccess) return e;
    return launch_pass3(s2, site, gs, p, nscenes, 0, p.ny, st);
}

cudaError_t edt_device(const uint8_t *occ, int32_t *site, void *scratch, const EdtPlan &p,
                       cudaStream_t st) {
    return edt_device_batched(occ, site, scratch, p, 1, st);
}

}  // namespace vx
