// Fused deskew + XY/XZ/YZ projections -- TMA-pipelined persistent kernel (sm_100a).
//
// Same contract and bit-exact arithmetic as the tiled path in ssb_deskew.cu
// (ss/pipeline.py:229-236 canvas lerp, ss/phantom.py:396-402 np.interp lerp,
// ss/geometry.py:236-255 spans), organised for B200:
//
//  * one persistent CTA per SM: 15 consumer warps + 1 producer warp;
//  * the producer pulls work items (u-tile x 256-column x-tile x slice chunk) from a
//    global atomic counter -- big chunks first, a tail of short chunks last, u-tiles
//    centre-out (heaviest first) -- and for every slice that touches the tile issues
//    one 3-D TMA box load (256 columns x TU+2*slack frame rows, OOB zero-filled) into a
//    5-stage (3 for 8-row tiles) shared-memory ring guarded by full/empty mbarriers (the box
//    load goes out as soon as a stage frees; the row table is built while it is in flight);
//    its lanes also derive the per-row sampling table (fp64, once per row per slice);
//  * consumer warp w owns 4 (or 8) canvas rows, lane l 8 columns: it reads the two
//    taps of each canvas row from shared memory (conflict-free 512 B rows; chained
//    rows reuse the converted tap row), evaluates 8 voxels with the exact fp64
//    expression, streams them to the volume with st.global.cs, and folds them into the
//    XY (registers), YZ (REDUX) and XZ (shared memory, named barrier) reductions, which
//    land in u32 scratch through L2 reductions (red.global.max/add);
//  * int->double conversion is folded into the products: fma(w, 2^52 + a,
//    -w*2^52) == fl(w*a) exactly (one rounding), so a voxel costs 2 DFMA + 2 DADD;
//  * rows that are not 16-byte aligned (W % 8 != 0, odd-offset crops) run the same pipeline
//    in row-class TMA mode (template AC = 32 + alignment, canvas formula): one tensor map per residue
//    class of rows (P = 16 / gcd(2 * row_stride, 16) classes), P boxes per stage, 248-column tiles;
//    batched or otherwise ineligible calls take the row-copy modes (AC < 16: cp.async or
//    per-row 1-D bulk copies instead of the TMA box).  Both use narrower shared loads / volume stores.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cudaTypedefs.h>
#include <mutex>
#include <numeric>

#include "ssb_plan.h"

#include "ssb_common.cuh"
#include "ssb_host.h"
#include "ssb_tma.cuh"

namespace ssb {
namespace tma_path {

constexpr int kConsumerWarps = 15;  // + 1 producer = 16 warps: 128 registers per thread
constexpr int kTX = 256;            // columns per tile (32 lanes x 8)
constexpr int kQueue = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr uint32_t kRowBytes = kTX * 2;

// Frame rows a tile needs (box height) and the slack above its first row:
//   nearest   rows u - lo exactly                              -> TU rows, slack 0
//   canvas    j0 in {u-b-1, u-b}, j1 <= u-b+1, b = floor(off)  -> TU+2 rows, slack 1
//   npinterp  j = max{k: fl(off+k) <= u} may move +-1 more     -> TU+4 rows, slack 2
template <int INTERP, int FORMULA>
__host__ __device__ constexpr int box_slack() {
    return INTERP == SSB_INTERP_NEAREST ? 0 : (FORMULA == SSB_FORMULA_CANVAS ? 1 : 2);
}

// Tile shape: 4 canvas rows per consumer warp (TU = 60, 5 stages) by default; projection-
// only max mode with XZ/YZ uses 8 rows (TU = 120, 3 stages), amortising the per-slice XZ
// barrier and bookkeeping over twice the voxels.  Sum mode needs 8 u32 accumulators per row
// and always keeps 4 rows.
#ifndef SSB_LOAD_EVICT_NORMAL
#define SSB_LOAD_EVICT_NORMAL 1  // A/B knob (profiles/README.md)
#endif
#ifndef SSB_L2_PROMO  // A/B knob: L2 promotion of the TMA box loads
#define SSB_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
#ifndef SSB_ALIGNED_ROW_STORES
#define SSB_ALIGNED_ROW_STORES 0  // A/B knob: 8-byte-aligned volume rows use 16-byte stores where aligned
#endif
#ifndef SSB_LOOKAHEAD_GAP
#define SSB_LOOKAHEAD_GAP 3  // consumer-copy mode: lookahead = stages - gap (A/B knob)
#endif
#ifndef SSB_REGULAR_STAGES
#define SSB_REGULAR_STAGES 1  // A/B knob: 0 = per-row tables for every stage
#endif
#ifndef SSB_YZ_LIVE_ONLY
#define SSB_YZ_LIVE_ONLY 1  // A/B knob (profiles/README.md)
#endif
#ifndef SSB_XY_STAGES
#define SSB_XY_STAGES 6  // ring depth of 4-row kernels without XZ staging (A/B knob)
#endif
template <int ROWS, bool SIDE = true>
struct Cfg {
    static constexpr int kRows = ROWS;
    static constexpr int kTU = kConsumerWarps * ROWS;
    static constexpr int kBoxRows = kTU + 4;
    // without side projections the XZ staging buffer is not needed and a deeper ring fits
    static constexpr int kStages = ROWS >= 8 ? 3 : (SIDE ? 5 : SSB_XY_STAGES);
#ifndef SSB_XZ_BATCH
#define SSB_XZ_BATCH 3  // 3: 3 MIPs 1.175 -> 1.154 ms, XY+XZ 1.112 -> 1.092 (profiles/r02_notes.md)
#endif
    static constexpr int kXzBatch = ROWS >= 8 ? 1 : SSB_XZ_BATCH;  // max-mode slices per XZ barrier
    static constexpr int kRowWords = (kTU + 31) / 32;   // 32-row groups the producer lanes cover
    // XZ staging: max mode packs u16x2 (kTX/2 words per warp and slice); sum mode (ROWS 4) u32
    static constexpr int kXzWords = !SIDE ? 4
                                    : ROWS >= 8 ? 2 * kXzBatch * kConsumerWarps * (kTX / 2)
                                                : (kXzBatch > 2 ? kXzBatch : 2) * kConsumerWarps * kTX;
    template <int INTERP, int FORMULA>
    static constexpr int box_rows() {
        return kTU + 2 * box_slack<INTERP, FORMULA>();
    }
};


// Sampling parameters of one canvas row for one slice (written by the producer).
// Rows outside the slice's span point both taps at a shared zero row with weights
// (1, 0), which yields exactly 0 -- the consumer loop has no per-row branches.
//
// Every linear voxel is rint(E) with E the reference's fp64 expression, and E lies within
// 2^-34.5 of a + w*(b - a) for the row weight w (canvas: w = f; npinterp: w = t/dx).  The
// consumers evaluate rint(a + w*(b - a)) in fp32 twice, with w rounded down (w_lo <= w - 2^-33)
// and up (w_hi >= w + 2^-33): one FFMA on 2^23 + a rounds to the integer grid exactly once, ties
// to even.  E lies between the two (monotone in w), so where both round to the same integer
// that integer is rint(E); the rare lanes where they differ (a half-integer inside the bracket:
// about 2^-23 |b - a| of the voxels) recompute their 8 voxels with the exact fp64 expression.
struct alignas(16) RowP {
    uint32_t off_a;  // shared-memory byte address of tap a (row j0)
    uint32_t off_b;  // tap b (row j1)
    int32_t kind;    // npinterp only: 3 = dx == 1 (incl. copies, t = 0), 2 = general dx
    int32_t pad;
    union {
        struct {
            float w_lo, w_lo2, w_hi, w_hi2;  // fp32 bracket of the row weight, duplicated for f32x2 ops
        };
        struct {
            double n0, n1;  // fp64 kernels (kF64): -c0 * 2^52, -c1 * 2^52
        };
    };
    double c0;       // canvas: w0 = 1-f       npinterp: t
    double c1;       // canvas: f              npinterp: dx
};

// A regular stage: every row of the tile lies inside the slice's span and the output window,
// its taps are unclamped (tap a of tile row r is frame row j0 + r, tap b the next one) and one
// fp32 bracket holds every row's weight (canvas formula; nearest copies row j0 + r).  About 94 % of
// the stages of a 2048-row frame; the producer then writes these 24 bytes instead of a row table.
struct alignas(16) StageP {
    double off;    // i*s of the slice (the fallback re-derives each row's exact weight from it)
    float w_lo, w_hi;
    int32_t a0;    // box row of tap a of tile row 0
    int32_t j0;    // frame row of tap a of tile row 0
};

// consumer-copy mode: the frame rows box rows [r_lo, r_hi) of a stage come from row0 + r * row_stride
struct CopyRec {
    const uint16_t *row0;  // box row 0, column xt * 256 (may lie outside the frame; only rows in range are read)
    int32_t r_lo, r_hi;
    int32_t x0;            // first column of the tile
    int32_t state;         // 0: no copy (slice misses the tile), 1: copy, 2: past the last stage
};

struct Params {
    uint16_t *vol;
    uint32_t *xy;  // u32 reduction targets (zeroed, or the caller's sum outputs)
    uint32_t *xz;
    uint32_t *yz;
    unsigned int *counters;  // [0] next item (zeroed by the host before the launch)
    int64_t n, h, w, first, u_begin, u_count, chunk;
    double shear;
    int64_t n1, chunk2;  // phase split: slices [0, n1) in chunks of `chunk`, [n1, n) of `chunk2`
    int32_t UT, XT, S, S2, n_items, xy_accumulate;
    int32_t clip;        // projection-only: each u-tile visits only the slices that can touch it
    int32_t big_pct;     // (clip) phase-1 share of a tile's slice range, percent
    const uint16_t *raw;  // row-copy mode (AC < 16): frames and their element strides
    int64_t row_stride, frame_stride;
    // batched launch (ssb_deskew_batch, TMA mode): stack b's frames are tensor-map frames
    // [b*n, (b+1)*n); its outputs sit b strides (elements) past the first stack's
    int32_t batch;
    int64_t vol_bstride, xy_bstride, xz_bstride, yz_bstride;
    int32_t rt_P, rt_B;  // row-class TMA: classes and box rows per class
    int32_t rt_B31;      // row-class TMA: rows per class in the lane-31 blocks
    uint32_t rt_d0;      // row-class TMA: byte offset (mod 16) of frame row 0 (delta_c = (d0 + c*rs2) & 15)
};

// AC: 16 = rows reach shared memory through one 3-D TMA box (16-byte aligned rows);
// 8 = rows 8-byte aligned (e.g. W % 8 == 4): the producer lanes copy each row's 256 pixels with
// 8-byte cp.async into the same 16-byte aligned layout as the TMA box;
// 4 / 2 = rows 4- / 2-byte aligned: one 1-D bulk copy per frame row of its 16-byte-aligned
// superset into a 528-byte slot, the row table points each tap at its first pixel inside the slot
// and consumers read with 4- / 2-byte granularity.  Volume stores use AC-byte accesses.
// Measured at 512 x 2048 x W (B200, volume + 3 MIPs): row-copy W = 2044 (AC 8) 2.59 ms, 2046 (AC 4)
// 2.81 ms, 2047 (AC 2) 3.66 ms; row-class TMA 2.04 / 2.15 / 2.98 ms; TMA boxes at W = 2048 1.60 ms.
// AC 8 / 4 (rows 8- / 4-byte aligned): consumer-copy mode -- the consumer warps copy the frame rows of
// the stage kLookahead stages ahead with 8- / 4-byte cp.async into 16-byte aligned shared-memory rows
// (the producer only publishes each stage's copy geometry), so the copies get 15 warps' issue slots
// and memory-level parallelism instead of one producer warp's.  AC 2 (odd widths): one 1-D bulk copy
// per frame row (its 16-byte-aligned superset) into 528-byte slots.
//
// Row-class TMA mode (AC = 32 + row alignment: 40 / 36 / 34), the default for rows that are not 16-byte
// aligned: with P = 16 / gcd(2 * row_stride, 16), the frame rows j = c (mod P) of class c all sit at the
// same byte offset delta_c (mod 16), so class c gets its own tensor map over every P-th row, based at its
// first row rounded down to 16 bytes (pixel x of a class-c row is map column x + delta_c / 2).  A stage
// loads one 256-column box per class at the tile's map column (16-byte aligned), class after class
// (B rows each); tiles are 248 columns wide so that every class's box covers them (lane 31 idles: in
// max mode it duplicates lane 30's columns, in sum mode its voxels are masked to zero).  Consumers read
// taps at the rows' alignment (delta_c); stores keep the volume's.  No per-row copy instructions at all.
template <int AC>
__host__ __device__ constexpr bool consumer_copy() {
    return AC == 8 || AC == 4;
}
template <int AC>
__host__ __device__ constexpr bool rt_mode() {
    return AC > 16;
}
// alignment (bytes) of the frame-row taps in shared memory and of the volume rows
template <int AC>
__host__ __device__ constexpr int acl() {
    return AC > 16 ? AC & 31 : AC;
}
// Row-class TMA tiles are 248 columns wide (lane 31 idles: in max mode it duplicates lane 30, in sum mode its
// voxels are masked) -- except projection-only launches with 8-byte rows (two classes, AC = 104 = 64 + 40):
// there lane 31 reads its pixels from a small per-class box, so tiles keep 256 columns (W = 2044 XY only
// 1.005 -> 0.955 ms, 3 MIPs 1.356 -> 1.300; with a volume, or 4 / 8 classes, it measured slower)
template <int AC>
__host__ __device__ constexpr bool lane31_boxes() {
    return AC > 64;
}
// columns per tile
template <int AC>
__host__ __device__ constexpr int tile_w() {
    return AC > 16 && !lane31_boxes<AC>() ? kTX - 8 : kTX;
}
template <int AC>
__host__ __device__ constexpr int row_pitch() {
    return AC == 2 ? kTX + 8 : kTX;
}
// shared-memory rows are 16-byte aligned except in bulk-copy mode (AC 2) and row-class TMA mode
template <int AC>
__host__ __device__ constexpr int smem_ac() {
    return AC == 2 ? 2 : rt_mode<AC>() ? acl<AC>() : 16;
}
// row-class TMA: box rows per class for P classes (a stage needs box_rows consecutive frame rows from
// any start; the class boxes start at the multiple of P at or below it)
__host__ __device__ constexpr int rt_class_rows(int box_rows, int P) {
    return (box_rows + 2 * P - 2) / P;
}
// shared-memory box rows per stage
template <int ROWS, bool SIDE, int AC>
__host__ __device__ constexpr int box_rows_alloc() {
    return rt_mode<AC>() ? (16 / acl<AC>()) * rt_class_rows(Cfg<ROWS, SIDE>::kTU + 2, 16 / acl<AC>())
                         : Cfg<ROWS, SIDE>::kBoxRows;
}
// ring depth: the 4- / 8-class boxes take more rows per stage than one box, and the lane-31 blocks and
// tables of the row-class mode leave no room for a fifth stage next to the XZ staging
template <int ROWS, bool SIDE, int AC>
__host__ __device__ constexpr int stage_count() {
    return rt_mode<AC>() && acl<AC>() < 8 ? Cfg<ROWS, SIDE>::kStages - 1 : Cfg<ROWS, SIDE>::kStages;
}

// row-class TMA: lane-31 block rows per stage (classes of B rows rounded up to 4: 128-byte aligned boxes)
template <int ROWS, bool SIDE, int AC>
__host__ __device__ constexpr int l31_rows_alloc() {
    return lane31_boxes<AC>() ? (16 / acl<AC>()) * ((rt_class_rows(Cfg<ROWS, SIDE>::kTU + 2, 16 / acl<AC>()) + 3) / 4 * 4)
                              : 1;
}
// Staged YZ (TMA mode, 4-row tiles with side projections, max mode): each lane's per-row u16x2 candidate
// words go to shared memory with the XZ partials, and threads of the XZ hand-off fold each row pair's 32
// words after the batch barrier -- no per-row split + `redux` on the consumers (3 MIPs 1.158 -> 1.126 ms,
// XY+XZ 1.094 -> 1.088; a YZ-only view now takes the batch barrier too: XY+YZ 1.060 -> 1.113).
template <int ROWS, bool SIDE, int AC>
__host__ __device__ constexpr bool staged_yz() {
    return AC == 16 && SIDE && ROWS == 4;
}
// max-mode slices per XZ hand-off: the lane-31 blocks of the 8-byte row-class mode, and the YZ staging,
// take the room of a third slice of XZ staging
template <int ROWS, bool SIDE, int AC>
__host__ __device__ constexpr int xz_batch() {
    return (lane31_boxes<AC>() || staged_yz<ROWS, SIDE, AC>()) && Cfg<ROWS, SIDE>::kXzBatch > 2
               ? 2
               : Cfg<ROWS, SIDE>::kXzBatch;
}

// tensor maps of one launch: [0] the frame box (TMA mode) or the row classes (row-class TMA mode)
struct alignas(64) TmapSet {
    CUtensorMap m[16];  // row-class TMA: [c] class c's 256-column boxes, [8 + c] its lane-31 boxes
};

template <int ROWS, int AC = 16, bool SIDE = true>
struct Smem {
    using C = Cfg<ROWS, SIDE>;
    static constexpr int kStages = stage_count<ROWS, SIDE, AC>();
    uint16_t box[kStages][box_rows_alloc<ROWS, SIDE, AC>()][row_pitch<AC>()];
    uint16_t zero_row[kTX + 8];
    // row-class TMA, regular stages: shared address of tap rows j0 + i of the stage (no lane offset)
    alignas(16) uint32_t taddr[rt_mode<AC>() ? kStages : 1][rt_mode<AC>() ? C::kTU + 4 : 4];
    // row-class TMA: lane 31's pixels come from a 16-pixel box per class at map column x0 + 248 (lane 31's
    // 8 pixels sit delta_c bytes into each 32-byte row), and its regular-stage tap addresses from taddr31
    alignas(128) uint16_t l31[rt_mode<AC>() ? kStages : 1][rt_mode<AC>() ? l31_rows_alloc<ROWS, SIDE, AC>() : 1][16];
    alignas(16) uint32_t taddr31[lane31_boxes<AC>() ? kStages : 1][lane31_boxes<AC>() ? C::kTU + 4 : 4];
    RowP rows[kStages][C::kTU];
    uint32_t hdr[kStages];  // bit 16: slice touches the tile; bits 0..14: warps with live rows;
                               // bits 17..31: warps whose rows chain their taps; bit 15: regular
                               // stage (taps and weights from sp[], the row table is not written)
    StageP sp[kStages];
    CopyRec cp[kStages];     // consumer-copy mode: what to copy into each stage
    uint64_t geo[kStages];   // consumer-copy mode: cp[] of the stage's current use is published
    alignas(16) uint32_t xz[(lane31_boxes<AC>() || staged_yz<ROWS, SIDE, AC>()) && C::kXzWords > 2 * kConsumerWarps * kTX
                                ? 2 * kConsumerWarps * kTX
                                : C::kXzWords];
    // staged YZ: [buffer][slice of the batch][row pair][32 lane words, swizzled by (row pair & 7) << 2]
    alignas(16) uint32_t yzs[staged_yz<ROWS, SIDE, AC>() ? 2 : 1][staged_yz<ROWS, SIDE, AC>() ? 2 : 1]
                            [staged_yz<ROWS, SIDE, AC>() ? C::kTU / 2 : 1][32];
    uint64_t full[kStages];
    uint64_t empty[kStages];
    uint64_t qfull[kQueue];
    uint64_t qempty[kQueue];
    int32_t queue[kQueue];
};

// Slices whose span can touch canvas rows [tu0, tu0 + TU): slice g covers about
// [g*s - 1, g*s + H] under both interpolations, so the bounds below (2 rows of margin) are
// conservative; the producer still tests every slice exactly.
template <int TU>
__device__ __forceinline__ void tile_slices(const Params &p, int ut, int64_t &lo, int64_t &hi) {
    lo = 0;
    hi = p.n;
    if (!(p.shear > 0.0)) return;
    const double tu0 = (double)(p.u_begin + (int64_t)ut * TU);
    const double first = (double)p.first, n = (double)p.n;
    // clamp in fp64 before converting (tiny shears give huge quotients)
    const double glo = fmin(fmax(floor((tu0 - (double)p.h - 2.0) / p.shear) - first, 0.0), n);
    const double ghi = fmin(fmax(floor((tu0 + (double)(TU + 1)) / p.shear) + 1.0 - first, glo), n);
    lo = (int64_t)glo;
    hi = (int64_t)ghi;
}

// Work item -> (u-tile, x-tile, slice range).  Two phases: every tile's first n1 slices in
// big chunks, then the remaining slices in small chunks, so the dynamic scheduler ends on
// short items (tail balance).  Within a phase u-tiles go centre-out (heaviest first).
// Projection-only launches (p.clip) split each tile's own slice range instead of [0, n): a
// long scan's tile is touched by ~(H + TU)/s of its slices, the rest would be empty stages.
template <int TU>
__device__ __forceinline__ void decode(int item, const Params &p, int &b, int &ut, int &xt, int64_t &s_begin,
                                       int64_t &s_end) {
    // phase 1 of every stack of a batch, then phase 2 of every stack (the tail stays short)
    const int per1 = p.UT * p.XT * p.S, per2 = p.UT * p.XT * p.S2;
    const int items1 = per1 * p.batch;
    const bool tail = item >= items1;
    if (tail) item -= items1;
    const int per = tail ? per2 : per1;
    b = item / per;
    item -= b * per;
    const int S = tail ? p.S2 : p.S;
    const int sc = item % S;
    const int rest = item / S;
    xt = rest % p.XT;
    const int k = rest / p.XT;
    const int mid = (p.UT - 1) / 2;
    const int d = (k + 1) >> 1;
    ut = (k & 1) ? mid + d : mid - d;
    int64_t chunk, base, stop;
    if (p.clip) {
        int64_t lo, hi;
        tile_slices<TU>(p, ut, lo, hi);
        const int64_t L = hi - lo;
        const int64_t n1 = p.S2 > 0 ? (L * p.big_pct) / 100 : L;
        base = tail ? lo + n1 : lo;
        stop = tail ? hi : lo + n1;
        chunk = (stop - base + S - 1) / S;
        if (chunk < 1) chunk = 1;
    } else {
        chunk = tail ? p.chunk2 : p.chunk;
        base = tail ? p.n1 : 0;
        stop = tail ? p.n : p.n1;
    }
    s_begin = min(stop, base + (int64_t)sc * chunk);
    s_end = min(stop, s_begin + chunk);
}

__device__ __forceinline__ double biased(uint32_t v16) { return __hiloint2double(0x43300000, (int)v16); }

template <int FORMULA>
__device__ __forceinline__ uint32_t voxel(uint32_t a, uint32_t b, const double c0, const double c1,
                                          const double n0, const double n1, const int kind) {
    if (FORMULA == SSB_FORMULA_CANVAS) {
        const double p0 = __fma_rn(c0, biased(a), n0);  // == fl(w0 * a)
        const double p1 = __fma_rn(c1, biased(b), n1);  // == fl(f * b)
        return (uint32_t)__double2loint(__dadd_rn(__dadd_rn(p0, p1), kRintMagic));
    } else {
        const double A = __dsub_rn(biased(a), kTwo52);
        if (kind == 3) {
            // dx == 1: slope = b - a exactly; fl(|d| * t) by the biased fma, sign restored
            // afterwards (round-to-nearest is symmetric)
            const int32_t d = (int32_t)b - (int32_t)a;
            double prod = __fma_rn(c0, biased((uint32_t)abs(d)), n0);
            if (d < 0) prod = -prod;
            return (uint32_t)__double2loint(__dadd_rn(__dadd_rn(prod, A), kRintMagic));
        }
        const double B = __dsub_rn(biased(b), kTwo52);
        const double slope = __ddiv_rn(__dsub_rn(B, A), c1);
        return (uint32_t)__double2loint(__dadd_rn(__dadd_rn(__dmul_rn(slope, c0), A), kRintMagic));
    }
}

// Exact fp64 evaluation of 8 voxels (the fallback of the fp32 bracket, see RowP): returns them
// as 2^23-biased fp32 bit patterns (0x4B000000 | v), the fast path's representation.
template <int FORMULA>
__device__ __forceinline__ void exact8(const uint4 a, const uint4 b, const double c0, const double c1, const int kind_,
                                       uint32_t (&bits)[8]) {
    const double n0 = __dmul_rn(c0, -kTwo52), n1 = __dmul_rn(c1, -kTwo52);  // exact
    const int kind = FORMULA == SSB_FORMULA_CANVAS ? 2 : kind_;
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
    const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        bits[2 * q] = 0x4B000000u | voxel<FORMULA>(aw[q] & 0xFFFFu, bw[q] & 0xFFFFu, c0, c1, n0, n1, kind);
        bits[2 * q + 1] = 0x4B000000u | voxel<FORMULA>(aw[q] >> 16, bw[q] >> 16, c0, c1, n0, n1, kind);
    }
}

constexpr uint32_t kBias = 0x4B000000u;  // fp32 bits of 2^23: a voxel v is carried as kBias | v

// ---- fp32x2 (FFMA2 / FADD2) helpers: a 64-bit register pair holds two fp32 lanes
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 f2pack(uint32_t lo, uint32_t hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}

__device__ __forceinline__ void f2unpack(f32x2 v, uint32_t &lo, uint32_t &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}

__device__ __forceinline__ f32x2 f2sub(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ f32x2 f2fma(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// 8 packed pixels -> 4 fp32 pairs holding 2^23 + pixel (one PRMT per pixel: 0x4B00 | pixel)
__device__ __forceinline__ void to_f23(const uint4 t, f32x2 (&o)[4]) {
    const uint32_t w4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = f2pack(__byte_perm(w4[q], 0x4B00u, 0x5410), __byte_perm(w4[q], 0x4B00u, 0x5432));
}

// rint(a + w*(b - a)) for 8 voxels at both ends of the weight bracket; bits = the w_lo results as
// 2^23-biased fp32 bit patterns.  Returns nonzero iff some voxel's two results differ.
__device__ __forceinline__ uint32_t lerp8_f32(const f32x2 (&A)[4], const f32x2 (&B)[4], const f32x2 wlo,
                                              const f32x2 whi, uint32_t (&bits)[8]) {
    uint32_t chk = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const f32x2 d = f2sub(B[q], A[q]);  // b - a, exact
        const f32x2 lo = f2fma(wlo, d, A[q]);
        const f32x2 hi = f2fma(whi, d, A[q]);
        uint32_t x0, x1;
        f2unpack(f2sub(hi, lo), x0, x1);  // 0 or +-1 per voxel
        chk |= x0 | x1;
        f2unpack(lo, bits[2 * q], bits[2 * q + 1]);
    }
    return chk;
}

// ---- fp64 chained lerp (sum mode with XZ / YZ: a per-slice CTA barrier would make every stage wait
// for the slowest warp's fp32-bracket fallback, so these kernels evaluate every voxel exactly in fp64)
// Tap conversion for the chained canvas path (SSB_CVT_MODE):
//   0  2^52 trick for every tap value: integer extract + constant high word, DFMA with -w*2^52;
//   1  native I2F.F64 for every value (one conversion-pipe op, ~16/clk/SM on B200) + DMUL;
//   2  mixed: low halves native (I2F.F64.U16 reads the half in place, no extract), high halves
//      by the trick -- 1.5 issue slots per value and half the conversion-pipe load of mode 1.
// All three give fl(w*a) exactly.  Measured on B200 (profiles/README.md): mode 2 is 2.6-3.4 %
// faster than mode 0 projection-only and equal with a volume; mode 1 is slowest (conversion pipe).
#ifndef SSB_CVT_MODE
#define SSB_CVT_MODE 2
#endif
template <int C>
__device__ __forceinline__ constexpr bool native_tap() {
    return SSB_CVT_MODE == 1 || (SSB_CVT_MODE == 2 && (C & 1) == 0);
}

// I2F.F64.U16 of the low half of a 32-bit register (no separate extract)
__device__ __forceinline__ double u16lo_to_f64(uint32_t w) {
    double r;
    asm("cvt.rn.f64.u16 %0, %1;" : "=d"(r) : "h"((unsigned short)w));
    return r;
}

__device__ __forceinline__ void to_biased8(const uint4 t, double (&o)[8]) {
    const uint32_t w4[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        o[2 * q] = (SSB_CVT_MODE != 0) ? u16lo_to_f64(w4[q]) : biased(w4[q] & 0xFFFFu);
        o[2 * q + 1] = (SSB_CVT_MODE == 1) ? __uint2double_rn(w4[q] >> 16) : biased(w4[q] >> 16);
    }
}

template <int C>
__device__ __forceinline__ double tap_prod(double c, double a, double n) {
    if (native_tap<C>()) return __dmul_rn(c, a);
    return __fma_rn(c, a, n);
}

// canvas lerp of 8 voxels from converted taps: rint(fl(fl(w0*a) + fl(f*b))) as 8 u32 values
template <int C>
__device__ __forceinline__ uint32_t lerp_one(const double a, const double b, const double c0, const double c1,
                                             const double n0, const double n1) {
    return (uint32_t)__double2loint(__dadd_rn(__dadd_rn(tap_prod<C>(c0, a, n0), tap_prod<C>(c1, b, n1)), kRintMagic));
}

__device__ __forceinline__ void lerp_biased8_raw(const double (&a)[8], const double (&b)[8], const double c0,
                                                 const double c1, const double n0, const double n1,
                                                 uint32_t (&r)[8]) {
    r[0] = lerp_one<0>(a[0], b[0], c0, c1, n0, n1);
    r[1] = lerp_one<1>(a[1], b[1], c0, c1, n0, n1);
    r[2] = lerp_one<2>(a[2], b[2], c0, c1, n0, n1);
    r[3] = lerp_one<3>(a[3], b[3], c0, c1, n0, n1);
    r[4] = lerp_one<4>(a[4], b[4], c0, c1, n0, n1);
    r[5] = lerp_one<5>(a[5], b[5], c0, c1, n0, n1);
    r[6] = lerp_one<6>(a[6], b[6], c0, c1, n0, n1);
    r[7] = lerp_one<7>(a[7], b[7], c0, c1, n0, n1);
}

__device__ __forceinline__ uint4 pack8(const uint32_t (&r)[8]) {
    return make_uint4(__byte_perm(r[0], r[1], 0x5410), __byte_perm(r[2], r[3], 0x5410),
                      __byte_perm(r[4], r[5], 0x5410), __byte_perm(r[6], r[7], 0x5410));
}

template <bool kMax>
__device__ __forceinline__ void red_u32(uint32_t *p, uint32_t v) {
    if (kMax) asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}

// 8 pixels from shared memory at a 2-byte aligned address known to be AC-byte aligned
template <int AC>
__device__ __forceinline__ uint4 lds8(uint32_t a) {
    if (AC == 16) return lds128(a);
    if (AC == 8) {
        const uint2 x = lds64(a), y = lds64(a + 8);
        return make_uint4(x.x, x.y, y.x, y.y);
    }
    if (AC == 4) return make_uint4(lds32(a), lds32(a + 4), lds32(a + 8), lds32(a + 12));
    // 2-byte aligned: five aligned words, shifted by 0 or 2 bytes (selector is warp-uniform per row)
    const uint32_t b = a & ~3u, sel = (a & 2u) ? 0x5432u : 0x3210u;
    const uint32_t w0 = lds32(b), w1 = lds32(b + 4), w2 = lds32(b + 8), w3 = lds32(b + 12), w4 = lds32(b + 16);
    return make_uint4(__byte_perm(w0, w1, sel), __byte_perm(w1, w2, sel), __byte_perm(w2, w3, sel),
                      __byte_perm(w3, w4, sel));
}

// a tap's 8 pixels from shared memory in the kernel's mode
// (row-class TMA, 4- / 2-byte aligned taps: two conflict-free 16-byte loads and a warp-uniform word
// shift instead were slower except for XY-only at W = 2047, profiles/r02_notes.md)
// 2- / 4-byte aligned taps: three 8-byte loads around the tap (12 shared-memory wavefronts, against 20 / 16
// for five / four 4-byte loads with the 4-way bank conflicts of a 16-byte lane stride), then a shift by a
// whole word (a & 4) and, for 2-byte alignment, a half word (a & 2) -- both warp-uniform (the row's)
// (projection-only kernels: W = 2046 / 2047 XY only 1.143 / 1.377 -> 1.095 / 1.323 ms, 3 MIPs 1.525 / 1.677
// -> 1.486 / 1.612; volume kernels: at 4-byte rows 1 % slower, so they keep the 4-byte loads there; at 2-byte
// rows, with the whole-sector stores below, 2.749 -> 2.686 ms, nearest 2.290 -> 2.188)
#ifndef SSB_RT_W64_LOADS
#define SSB_RT_W64_LOADS 2  // A/B knob: 0 off, 1 for 2-byte aligned taps, 2 also for 4-byte aligned taps
#endif
template <int A>
__device__ __forceinline__ uint4 lds8_w64(uint32_t a) {
    const uint32_t b = a & ~7u;
    const uint2 p = lds64(b), q = lds64(b + 8), r = lds64(b + 16);
    const bool w = (a & 4u) != 0;
    const uint32_t v0 = w ? p.y : p.x, v1 = w ? q.x : p.y, v2 = w ? q.y : q.x, v3 = w ? r.x : q.y;
    if (A == 4) return make_uint4(v0, v1, v2, v3);
    const uint32_t v4 = w ? r.y : r.x, sel = (a & 2u) ? 0x5432u : 0x3210u;
    return make_uint4(__byte_perm(v0, v1, sel), __byte_perm(v1, v2, sel), __byte_perm(v2, v3, sel),
                      __byte_perm(v3, v4, sel));
}

template <int AC, bool W64 = false>
__device__ __forceinline__ uint4 ldtap(uint32_t a) {
    if ((W64 || acl<AC>() == 2) && rt_mode<AC>() &&
        ((acl<AC>() == 2 && SSB_RT_W64_LOADS >= 1) || (acl<AC>() == 4 && SSB_RT_W64_LOADS >= 2)))
        return lds8_w64<acl<AC>()>(a);
    return lds8<smem_ac<AC>()>(a);
}

// 8 pixels to the volume (streaming stores) at an AC-byte aligned address
template <int AC>
__device__ __forceinline__ void stg8(uint16_t *p, const uint4 v) {
    if (AC == 16) {
        stg_cs_v4(p, v);
    } else if (AC == 8) {
#if SSB_ALIGNED_ROW_STORES
        if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {  // this row happens to be 16-byte aligned
            stg_cs_v4(p, v);
            return;
        }
#endif
        asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
        asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(p + 4), "r"(v.z), "r"(v.w) : "memory");
    } else if (AC == 4 || (reinterpret_cast<uintptr_t>(p) & 2u) == 0) {
        const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p + 2 * k), "r"(q[k]) : "memory");
    } else {
        // 2 mod 4: one pixel, three aligned words across pixel pairs, one pixel
        asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)(v.x & 0xFFFFu)) : "memory");
        asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p + 1), "r"(__byte_perm(v.x, v.y, 0x5432)) : "memory");
        asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p + 3), "r"(__byte_perm(v.y, v.z, 0x5432)) : "memory");
        asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p + 5), "r"(__byte_perm(v.z, v.w, 0x5432)) : "memory");
        asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p + 7), "h"((unsigned short)(v.w >> 16)) : "memory");
    }
}

// 8 pixels at the widest access this address allows (row-class TMA volume rows: the row alignment cycles
// with the canvas row, the same for every lane of a warp, so the branches are uniform)
#ifndef SSB_RT_DYN_STORES
#define SSB_RT_DYN_STORES 1  // A/B knob
#endif
__device__ __forceinline__ void stg8_any(uint16_t *p, const uint4 v) {
    const uint32_t a = (uint32_t)reinterpret_cast<uintptr_t>(p) & 15u;
    if (a == 0) stg8<16>(p, v);
    else if ((a & 7u) == 0) stg8<8>(p, v);
    else if ((a & 3u) == 0) stg8<4>(p, v);
    else stg8<2>(p, v);
}

// Row-class TMA volume rows that are 2- or 4-byte aligned: lane l's 16 bytes start r = (address & 15) past a
// 16-byte boundary (248-column tiles: lanes 0..30).  Lanes 1..30 store the aligned 16 bytes [q - r, q - r + 16)
// -- the left neighbour's last r bytes and their own first 16 - r -- as one 16-byte store; lanes 0 and 30 also
// store their own 16 bytes
// with narrow stores (covering the segment's unaligned head and tail; the overlap rewrites equal bytes).
// Narrow 2- / 4-byte stores at a 16-byte lane stride write every sector in 4-8 pieces; this writes whole
// sectors.  r is the same for every lane (lanes are 16 bytes apart), so the branch is uniform.
// (W = 2047, volume + 3 MIPs: 2.985 -> 2.750 ms; at 4-byte rows (W = 2046) 2.167 -> 2.227, so 2-byte rows only)
#ifndef SSB_RT_SHIFT_STORES
#define SSB_RT_SHIFT_STORES 1  // A/B knob
#endif
template <int A>
__device__ __forceinline__ void stg8_shift(uint16_t *q, const uint4 v, const uint32_t ln) {
    const uint32_t r = (uint32_t)reinterpret_cast<uintptr_t>(q) & 15u;
    if (r == 0) {
        if (ln < 31) stg_cs_v4(q, v);
        return;
    }
    const uint32_t W0 = __shfl_up_sync(0xffffffffu, v.x, 1), W1 = __shfl_up_sync(0xffffffffu, v.y, 1),
                   W2 = __shfl_up_sync(0xffffffffu, v.z, 1), W3 = __shfl_up_sync(0xffffffffu, v.w, 1);
    const uint32_t W[8] = {W0, W1, W2, W3, v.x, v.y, v.z, v.w};
    const uint32_t sft = 16u - r, m = sft >> 2;  // window (left 16 bytes, own 16 bytes) from byte sft
    uint32_t B[6], V[5];
#pragma unroll
    for (int j = 0; j < 6; ++j) B[j] = (m & 2u) ? W[j + 2] : W[j];
#pragma unroll
    for (int k = 0; k < 5; ++k) V[k] = (m & 1u) ? B[k + 1] : B[k];
    uint4 o;
    if (A == 4) {
        o = make_uint4(V[0], V[1], V[2], V[3]);
    } else {
        const uint32_t sel = (sft & 2u) ? 0x5432u : 0x3210u;
        o = make_uint4(__byte_perm(V[0], V[1], sel), __byte_perm(V[1], V[2], sel), __byte_perm(V[2], V[3], sel),
                       __byte_perm(V[3], V[4], sel));
    }
    if (ln >= 1 && ln <= 30) stg_cs_v4(reinterpret_cast<void *>(reinterpret_cast<uintptr_t>(q) - r), o);
    if (ln == 0 || ln == 30) stg8<A>(q, v);
}

// the first nv (< 8) pixels of a lane that straddles the right edge (row-copy mode only)
__device__ __forceinline__ void stg_partial(uint16_t *p, const uint4 v, const int nv) {
    const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if (c < nv) p[c] = (uint16_t)(q[c >> 1] >> (16 * (c & 1)));
}

// zero the pixels at and beyond column nv (0..8) of a lane
__device__ __forceinline__ uint4 mask_cols(const uint4 v, const int nv) {
    uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t keep = (2 * k < nv ? 0x0000FFFFu : 0u) | (2 * k + 1 < nv ? 0xFFFF0000u : 0u);
        q[k] &= keep;
    }
    return make_uint4(q[0], q[1], q[2], q[3]);
}

__device__ __forceinline__ uint4 max3_u16x8(const uint4 a, const uint4 b, const uint4 c) {
    // __vmaxu2(__vmaxu2(.)) pairs fuse into one VIMNMX3.U16x2 each
    return make_uint4(__vmaxu2(__vmaxu2(a.x, b.x), c.x), __vmaxu2(__vmaxu2(a.y, b.y), c.y),
                      __vmaxu2(__vmaxu2(a.z, b.z), c.z), __vmaxu2(__vmaxu2(a.w, b.w), c.w));
}

__device__ __forceinline__ uint32_t hmax8(const uint4 v) {
    const uint32_t m = __vmaxu2(__vmaxu2(__vmaxu2(v.x, v.y), v.z), v.w);  // ptxas fuses into VIMNMX3
    return max(m & 0xFFFFu, m >> 16);
}

// the same as a u16x2 word (both halves candidates)
__device__ __forceinline__ uint32_t hmax8w(const uint4 v) {
    return __vmaxu2(__vmaxu2(__vmaxu2(v.x, v.y), v.z), v.w);
}

__device__ __forceinline__ uint32_t redux_max(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}

__device__ __forceinline__ uint32_t redux_add(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.add.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}

// fp32 bracket [w_lo, w_hi] of the row weight w with a 2^-33 margin on either side: wider than the
// 2^-34.5 between the reference's fp64 result and a + w*(b - a) for any |b - a| >= 1
__device__ __forceinline__ void set_bracket(RowP &o, double w) {
    constexpr double kMargin = 1.1641532182693481e-10;  // 2^-33
    o.w_lo = o.w_lo2 = __double2float_rd(__dsub_rn(w, kMargin));
    o.w_hi = o.w_hi2 = __double2float_ru(__dadd_rn(w, kMargin));
}

// Row table entry of canvas row u for one slice (producer lanes).  Returns whether
// the row is live (inside the window and the slice's span).
// Row-copy mode: frame row j of the slice sits at byte (d0 + 2*j*rs) & 15 of its slot (d0: the
// alignment of row 0's first pixel of the tile); TMA mode: d0 = rs2 = 0.
// Shared address of frame row j's first tile pixel (no lane offset).  Row-class TMA: class c = (j - jb) mod P
// (jb = the class boxes' first frame row, a multiple of P), block row (j - jb) / P, B rows per class.
struct RtGeo {
    int64_t jb;
    uint32_t lp, B;  // log2(P), rows per class box
    uint32_t B31;    // rows per class in the lane-31 blocks (B rounded up to 4: 128-byte aligned boxes)
    uint32_t l31;    // shared address of the stage's lane-31 blocks
};
// lane 31's 8 pixels of frame row j: its class's lane-31 block, 32-byte rows, the row's byte offset
__device__ __forceinline__ uint32_t row_addr31(int64_t j, uint32_t d0, uint32_t rs2, const RtGeo &g) {
    const uint32_t q = (uint32_t)(j - g.jb);
    const uint32_t c = q & ((1u << g.lp) - 1u), r = q >> g.lp;
    return g.l31 + (c * g.B31 + r) * 32u + ((d0 + rs2 * (uint32_t)j) & 15u);
}
template <int AC>
__device__ __forceinline__ uint32_t row_addr(int64_t j, int64_t box_r0, uint32_t box_addr, uint32_t d0, uint32_t rs2,
                                             const RtGeo &g) {
    if (rt_mode<AC>()) {
        const uint32_t q = (uint32_t)(j - g.jb);
        const uint32_t c = q & ((1u << g.lp) - 1u), r = q >> g.lp;
        return box_addr + (c * g.B + r) * (2u * row_pitch<AC>()) + ((d0 + rs2 * (uint32_t)j) & 15u);
    }
    return box_addr + (uint32_t)(j - box_r0) * (2u * row_pitch<AC>()) + ((d0 + rs2 * (uint32_t)j) & 15u);
}

template <int INTERP, int FORMULA, int AC, bool F64>
__device__ __forceinline__ bool make_row(RowP &o, int64_t u, bool in_window, int64_t lo, int64_t hi, double off,
                                         int64_t h, int64_t box_r0, int64_t box_rows, uint32_t box_addr,
                                         uint32_t zero_addr, uint32_t d0, uint32_t rs2, const RtGeo &g) {
    o.c0 = 1.0;
    o.c1 = 0.0;
    o.off_a = o.off_b = zero_addr;
    o.kind = 3;
    o.pad = 0;
    // row-class TMA (canvas formula: `kind` unused): kind / pad carry lane 31's tap addresses
    if (lane31_boxes<AC>()) o.kind = o.pad = (int32_t)(zero_addr + 496u);
    if (FORMULA == SSB_FORMULA_NPINTERP) o.c0 = 0.0;  // t = 0: copy of tap a (the zero row)
    if (F64) {
        o.n0 = -(o.c0 * kTwo52);
        o.n1 = -0.0;
    } else {
        set_bracket(o, 0.0);
    }
    if (!in_window || u < lo || u > hi) return false;
    const RowParam rp = row_param<INTERP, FORMULA>(u, lo, off, h);
    // the box covers [box_r0, box_r0 + TU + 2*slack): a tap outside it would read another
    // stage's data -- fail loudly instead (cheap: once per row per slice, producer warp only)
    if (rp.j0 < box_r0 || rp.j1 < box_r0 || rp.j0 - box_r0 >= box_rows || rp.j1 - box_r0 >= box_rows) __trap();
    o.off_a = row_addr<AC>(rp.j0, box_r0, box_addr, d0, rs2, g);
    o.off_b = row_addr<AC>(rp.j1, box_r0, box_addr, d0, rs2, g);
    if (lane31_boxes<AC>()) {
        o.kind = (int32_t)row_addr31(rp.j0, d0, rs2, g);
        o.pad = (int32_t)row_addr31(rp.j1, d0, rs2, g);
    }
    if (rp.kind >= 2) {
        o.c0 = rp.c0;
        o.c1 = rp.c1;
        if (!lane31_boxes<AC>()) o.kind = rp.kind;
        // weight of a + w*(b - a): canvas f; np.interp t (dx == 1) or t/dx
        if (F64) {
            o.n0 = -(rp.c0 * kTwo52);  // exact: power-of-two scaling
            o.n1 = -(rp.c1 * kTwo52);
        } else {
            set_bracket(o, FORMULA == SSB_FORMULA_CANVAS ? rp.c1 : rp.kind == 3 ? rp.c0 : __ddiv_rn(rp.c0, rp.c1));
        }
    } else if (FORMULA == SSB_FORMULA_CANVAS) {
        // copy (only reachable for h == 1 paths): w0 = 1, f = 0
        o.off_b = o.off_a;
        o.pad = o.kind;
    }
    return true;
}

// One consumer warp's ROWS canvas rows of one slice: sample, store, fold into XY / XZ / YZ.
// FULL: all 8 columns of every lane and all rows are inside the output (no predicates).
// Max mode with 4 rows computes the voxels of all rows first and consumes them afterwards
// (the tap registers die before the accumulators are touched; XZ folds with 3-input maxes);
// with 8 rows, and always in sum mode, each row is consumed as soon as it is computed (sums
// take the u32 voxels straight from the rint, no pack/unpack: measured 2-5 % faster).
// Row-copy mode (AC < 16), !FULL: a lane may straddle the right edge (nv < 8 pixels inside); its
// outside pixels are zeroed before any reduction and never stored.
// REG: a regular stage (StageP): taps at fixed box rows (tap_base + k rows), one weight bracket,
// the fallback re-derives row k's exact weight from the slice offset (canvas row u0 + k, tap j0 + k).
template <int INTERP, int FORMULA, bool kMax, bool FULL, int ROWS, bool SIDE, bool CHAIN, int AC, bool REG,
          bool NOVOL>
__device__ __forceinline__ void rows_pass(const RowP *rg, const uint32_t lane_off, const uint32_t tap_base,
                                          const uint32_t *tad, const uint32_t *tad31, const StageP &sp,
                                          const int64_t u0,
                                          uint16_t *vrow, const int64_t w, const int rows_ok, const bool col_ok,
                                          const int nv, uint4 (&acc_max)[ROWS],
                                          uint32_t (&acc_sum)[kMax ? 1 : ROWS][8],
                                          uint4 &xz_max, uint32_t (&xz_sum)[8], uint32_t (&yzv)[ROWS]) {
#ifndef SSB_SIDE_STREAM
#define SSB_SIDE_STREAM 0  // A/B: 4-row max tiles with XZ/YZ consume each row as it is computed
#endif
    constexpr bool kStream = ROWS > 4 || !kMax || (SIDE && SSB_SIDE_STREAM);
    constexpr bool kFoldXz = kMax && SIDE && !kStream;  // XZ over the batch with 3-input maxes
    constexpr bool kPairXz = kMax && SIDE && kStream;   // XZ over row pairs with 3-input maxes
    uint4 xz_prev = make_uint4(0, 0, 0, 0);
    const bool store = vrow != nullptr;
    constexpr bool chain = (CHAIN || REG) && INTERP == SSB_INTERP_LINEAR;
    constexpr uint32_t kPitch = 2u * row_pitch<AC>();
    constexpr bool kRT = rt_mode<AC>();
    // row-class TMA: lane 31 reads its taps from the stage's lane-31 blocks (rows of 32 bytes)
    constexpr bool kL31 = lane31_boxes<AC>();
    constexpr bool kT248 = kRT && !kL31;  // 248-column tiles: lane 31 outside the tile
    const bool l31 = kL31 && (threadIdx.x & 31) == 31;
    // row-class TMA, regular stage: the rows' tap addresses from the stage's tables (consecutive rows
    // alternate between class boxes)
    uint32_t ta[ROWS + 1];
    if (kRT && REG) {
#pragma unroll
        for (int k = 0; k <= ROWS; ++k) ta[k] = kL31 && l31 ? tad31[k] : tad[k] + lane_off;
    }
    // tap addresses of row k (lane offset included; row-class TMA lane 31: the row table's kind / pad)
    auto tap_a = [&](const int k) {
        return REG ? (kRT ? ta[k] : tap_base + (uint32_t)k * kPitch)
                   : (l31 ? (uint32_t)rg[k].kind : rg[k].off_a + lane_off);
    };
    auto tap_b = [&](const int k) {
        return REG ? (kRT ? ta[k + 1] : tap_base + (uint32_t)(k + 1) * kPitch)
                   : (l31 ? (uint32_t)rg[k].pad : rg[k].off_b + lane_off);
    };
    // a lane may straddle the right edge; 248-column tiles in sum mode also mask lane 31 (max mode
    // duplicates lane 30)
    constexpr bool kEdge = (AC != 16 && !FULL) || (kT248 && !kMax);
    auto put = [&](const int k, const uint4 v) {
        if (kRT && SSB_RT_SHIFT_STORES && FULL && acl<AC>() == 2) {
            // every lane takes part in the shuffles (lane 31 lends nothing and stores nothing itself)
            if (store) stg8_shift<acl<AC>()>(vrow + k * w, v, threadIdx.x & 31);
            return;
        }
        if (!(store && (FULL ? (!kT248 || col_ok) : (k < rows_ok && col_ok)))) return;
        if (kEdge && nv < 8) stg_partial(vrow + k * w, v, nv);
        else if (kRT && SSB_RT_DYN_STORES && acl<AC>() == 8) stg8_any(vrow + k * w, v);
        else stg8<acl<AC>()>(vrow + k * w, v);
    };
    auto consume = [&](const int k, uint4 v) {
        if (kEdge) v = mask_cols(v, nv);
        put(k, v);
        if (kMax) {
            acc_max[k] = max_u16x8(acc_max[k], v);
            if (SIDE) {  // XZ / YZ requested (compile-time: XY-only views skip this work)
                if (kPairXz) {
                    if (k & 1) xz_max = max3_u16x8(xz_max, xz_prev, v);
                    else xz_prev = v;
                } else if (!kFoldXz) {
                    xz_max = max_u16x8(xz_max, v);
                }
                // staged YZ: the lane's u16x2 candidate word (folded across lanes after the pass)
                yzv[k] = staged_yz<ROWS, SIDE, AC>() ? hmax8w(v) : redux_max(hmax8(v));
            }
        } else {
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
            uint32_t rs = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t e = (w4[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                acc_sum[k][c] += e;
                if (SIDE) {  // XZ / YZ requested (compile-time: XY-only sums skip this work)
                    xz_sum[c] += e;
                    rs += e;
                }
            }
            if (SIDE) yzv[k] = redux_add(rs);
        }
    };
    uint4 vs[kStream ? 1 : ROWS];
    // batched fallback (rows computed before they are consumed): one branch per pass tests every row's
    // bracket check, so the rows' instructions form one basic block the scheduler can interleave
#ifndef SSB_ONE_FALLBACK
#define SSB_ONE_FALLBACK 1  // A/B knob
#endif
    // (XY-only views: 0.794 -> 0.789 ms at config 2; with XZ the longer block was 3 % slower)
    constexpr bool kOneFb = SSB_ONE_FALLBACK && !kStream && !SIDE;
    uint32_t chk[ROWS];
    constexpr bool kF64 = !kMax && SIDE && INTERP == SSB_INTERP_LINEAR;  // see lerp_biased8_raw
    constexpr bool chain32 = chain && !kF64, chain64 = chain && kF64 && FORMULA == SSB_FORMULA_CANVAS;
    // exact fp64 evaluation of row k (the fp32 bracket's fallback)
    auto exact_row = [&](const int k, uint32_t (&bits)[8]) {
        const uint4 ta = ldtap<AC, NOVOL>(tap_a(k)), tb = ldtap<AC, NOVOL>(tap_b(k));
        if (REG) {
            // canvas formula, unclamped taps j0+k, j0+k+1: f = fl(fl(u - off) - j0), w0 = 1 - f
            const double f = __dsub_rn(__dsub_rn((double)(u0 + k), sp.off), (double)(sp.j0 + k));
            exact8<FORMULA>(ta, tb, __dsub_rn(1.0, f), f, 2, bits);
        } else {
            exact8<FORMULA>(ta, tb, rg[k].c0, rg[k].c1, rg[k].kind, bits);
        }
    };
    f32x2 prev[4];
    double prevd[8];
    if (chain32) to_f23(ldtap<AC, NOVOL>(tap_a(0)), prev);
    if (chain64) to_biased8(ldtap<AC, NOVOL>(tap_a(0)), prevd);
    f32x2 wlo_s = 0, whi_s = 0;
    if (REG) {
        wlo_s = f2pack(__float_as_uint(sp.w_lo), __float_as_uint(sp.w_lo));
        whi_s = f2pack(__float_as_uint(sp.w_hi), __float_as_uint(sp.w_hi));
    }
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
        uint4 v;
        if (INTERP == SSB_INTERP_NEAREST) {
            v = ldtap<AC, NOVOL>(tap_a(k));
        } else if (kF64) {
            // the producer writes full row tables for these kernels (no regular stages)
            uint32_t bits[8];
            const double c0 = rg[k].c0, c1 = rg[k].c1;
            const int kind = rg[k].kind;
            if (chain64) {
                double cur[8];
                to_biased8(ldtap<AC, NOVOL>(tap_b(k)), cur);
                lerp_biased8_raw(prevd, cur, c0, c1, rg[k].n0, rg[k].n1, bits);
#pragma unroll
                for (int c = 0; c < 8; ++c) prevd[c] = cur[c];
            } else {
                exact8<FORMULA>(ldtap<AC, NOVOL>(tap_a(k)), ldtap<AC, NOVOL>(tap_b(k)), c0, c1, kind, bits);
#pragma unroll
                for (int c = 0; c < 8; ++c) bits[c] &= 0xFFFFu;  // unbiased: these kernels sum plain voxels
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (kEdge && c >= nv) bits[c] = 0u;
            put(k, pack8(bits));
            uint32_t rs = 0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                acc_sum[k][c] += bits[c];
                xz_sum[c] += bits[c];
                rs += bits[c];
            }
            yzv[k] = redux_add(rs);
            continue;
        } else {
            // fp32 bracket of the lerp (RowP); chained taps: tap row k+1 is tap b of row k and
            // tap a of row k+1, converted once
            f32x2 A[4], B[4];
            to_f23(ldtap<AC, NOVOL>(tap_b(k)), B);
            if (chain32) {
#pragma unroll
                for (int q = 0; q < 4; ++q) A[q] = prev[q];
            } else {
                to_f23(ldtap<AC, NOVOL>(tap_a(k)), A);
            }
            f32x2 wlo = wlo_s, whi = whi_s;
            if (!REG) {
                const uint4 wq = *reinterpret_cast<const uint4 *>(&rg[k].w_lo);
                wlo = f2pack(wq.x, wq.y);
                whi = f2pack(wq.z, wq.w);
            }
            uint32_t bits[8];
            chk[k] = lerp8_f32(A, B, wlo, whi, bits);
            if (!kOneFb && chk[k] != 0) exact_row(k, bits);
            if (chain32) {
#pragma unroll
                for (int q = 0; q < 4; ++q) prev[q] = B[q];
            }
            if (!kMax && kStream) {
                // sums add the 2^23-biased bits as they are (mod 2^32): the caller removes the
                // bias once per pass (XZ), per item (XY: live passes x kBias); a YZ row sums 256
                // biased values, whose bias is 0 mod 2^32.  Masked columns carry the bare bias.
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (kEdge && c >= nv) bits[c] = kBias;
                put(k, pack8(bits));
                uint32_t rs = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    acc_sum[k][c] += bits[c];
                    if (SIDE) {
                        xz_sum[c] += bits[c];
                        rs += bits[c];
                    }
                }
                if (SIDE) yzv[k] = redux_add(rs);
                continue;
            }
            v = pack8(bits);
        }
        if (kStream) consume(k, v);
        else vs[k] = kEdge ? mask_cols(v, nv) : v;
    }
    if (!kStream) {
        if (kOneFb && INTERP == SSB_INTERP_LINEAR && !kF64) {
            uint32_t any = 0;
#pragma unroll
            for (int k = 0; k < ROWS; ++k) any |= chk[k];
            if (any != 0) {
#pragma unroll
                for (int k = 0; k < ROWS; ++k) {
                    if (chk[k] != 0) {
                        uint32_t bits[8];
                        exact_row(k, bits);
                        vs[k] = kEdge ? mask_cols(pack8(bits), nv) : pack8(bits);
                    }
                }
            }
        }
        if (kFoldXz) {
#pragma unroll
            for (int k = 0; k + 1 < ROWS; k += 2) xz_max = max3_u16x8(xz_max, vs[k], vs[k + 1]);
        }
#pragma unroll
        for (int k = 0; k < ROWS; ++k) consume(k, vs[k < (kStream ? 1 : ROWS) ? k : 0]);
    }
}

// VOL = false: projection-only instantiation (no volume store code at all)
template <int INTERP, int FORMULA, int REDUCE, int ROWS, bool SIDE, int AC, bool VOL>
__global__ void __launch_bounds__(kThreads, 1)
    deskew_tma_kernel(const __grid_constant__ TmapSet maps, const Params p) {
    constexpr bool kMax = REDUCE == SSB_REDUCE_MAX;
    // sum mode with XZ / YZ evaluates voxels in fp64 (see lerp_biased8_raw) from full row tables
    constexpr bool kF64 = !kMax && SIDE && INTERP == SSB_INTERP_LINEAR;
    using C = Cfg<ROWS, SIDE>;
    constexpr int kTU = C::kTU;
    constexpr int kStages = stage_count<ROWS, SIDE, AC>();
    constexpr bool kRT = rt_mode<AC>();
    constexpr int kTW = tile_w<AC>();  // columns per tile
    const CUtensorMap &tmap = maps.m[0];
    // consumer-copy mode: stages copied ahead of the one processed; copying stage k + D needs every warp
    // done with stage k + D - kStages, so D < kStages - 1 leaves the warps room to drift apart
    constexpr int kLookahead = kStages - SSB_LOOKAHEAD_GAP > 0 ? kStages - SSB_LOOKAHEAD_GAP : 1;
    constexpr int kXzBatch = kMax ? xz_batch<ROWS, SIDE, AC>() : 1;
    static_assert(kXzBatch * (kTX / 2) <= kConsumerThreads, "one consumer thread per (slice, column pair)");
    static_assert(!(kMax && staged_yz<ROWS, SIDE, AC>()) ||
                      (kXzBatch <= 2 && kXzBatch * (kTX / 2 + kTU / 2) <= kConsumerThreads),
                  "staged YZ: one consumer thread per (slice, row pair) next to the XZ threads");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem<ROWS, AC, SIDE> &sm = *reinterpret_cast<Smem<ROWS, AC, SIDE> *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int k = 0; k < kStages; ++k) {
            // cp.async modes add one asynchronous arrival per producer lane (copies landed)
            // producer lanes (row table) + in consumer-copy mode every consumer lane's cp.async arrival
            mbar_init(&sm.full[k], consumer_copy<AC>() ? 32 + kConsumerThreads : 32);
            mbar_init(&sm.geo[k], 1);
            mbar_init(&sm.empty[k], kConsumerWarps);
        }
        for (int k = 0; k < kQueue; ++k) {
            mbar_init(&sm.qfull[k], 1);
            mbar_init(&sm.qempty[k], kConsumerWarps);
        }
        fence_mbar_init();
    }
    for (int k = tid; k < kTX + 8; k += kThreads) sm.zero_row[k] = 0;
    __syncthreads();

    if (warp == kConsumerWarps) {
        // ===================== producer warp =====================
        if (kRT ? (lane < p.rt_P || (lane31_boxes<AC>() && lane >= 8 && lane < 8 + p.rt_P)) : lane == 0)
            prefetch_tmap(&maps.m[lane]);
        // L2 policy of the frame loads: evict-normal in max mode (measured 2-3 % faster isolated:
        // halo rows shared by vertically adjacent tiles survive), evict-first in sum mode (whose u32
        // REDs into the caller's outputs want the L2 space; evict-normal was 2 % slower there)
        uint64_t policy;
        if (kMax && SSB_LOAD_EVICT_NORMAL == 2)
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy));
        else if (kMax && SSB_LOAD_EVICT_NORMAL)
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
        else
            policy = policy_evict_first();
        const uint32_t zero_addr = smem_addr(sm.zero_row);
        uint32_t stage = 0, sphase = 0, q = 0, qphase = 0;
        while (true) {
            int item = 0;
            if (lane == 0) item = (int)atomicAdd(&p.counters[0], 1u);
            item = __shfl_sync(0xffffffffu, item, 0);
            const bool done = item >= p.n_items;
            int b = 0, ut = 0, xt = 0;
            int64_t s_begin = 0, s_end = 0;
            if (!done) {
                decode<kTU>(item, p, b, ut, xt, s_begin, s_end);
                if (s_begin >= s_end) continue;  // items without slices (clipped tiles) are not handed over
            }
            if (lane == 0) {
                mbar_wait(&sm.qempty[q], qphase ^ 1);
                sm.queue[q] = done ? -1 : item;
                mbar_arrive(&sm.qfull[q]);
            }
            if (++q == kQueue) { q = 0; qphase ^= 1; }
            if (done) break;
            const int64_t tu0 = p.u_begin + (int64_t)ut * kTU;
            const int32_t frame0 = b * (int32_t)p.n;  // tensor-map frame of this stack's slice 0
            for (int64_t s = s_begin; s < s_end; ++s) {
                int64_t lo, hi;
                double off;
                slice_span(p.first + s, p.shear, p.h, INTERP, lo, hi, off);
                const bool hit = !(hi < tu0 || lo > tu0 + kTU - 1);
                const int64_t base = INTERP == SSB_INTERP_NEAREST ? lo : (int64_t)floor(off);
                const int64_t box_r0 = tu0 - base - box_slack<INTERP, FORMULA>();
                // the box load goes out as soon as the stage is free; the row table is built
                // while it is in flight (full completes on the bytes + all 32 lane arrivals)
                constexpr int kBoxRowsUsed = C::template box_rows<INTERP, FORMULA>();
                // row-class TMA: the class boxes start at frame row jb (the multiple of P at or below box_r0)
                RtGeo rg{0, 0, 0, 0, 0};
                if (kRT) {
                    rg.lp = (uint32_t)(__ffs(p.rt_P) - 1);
                    rg.B = (uint32_t)p.rt_B;
                    rg.B31 = (uint32_t)p.rt_B31;
                    rg.l31 = smem_addr(&sm.l31[stage][0][0]);
                    rg.jb = (box_r0 >> rg.lp) << rg.lp;  // floor (arithmetic shift)
                }
                if (lane == 0) {
                    mbar_wait(&sm.empty[stage], sphase ^ 1);
                    if (hit && AC == 16) {
                        mbar_expect_tx(&sm.full[stage], kBoxRowsUsed * kRowBytes);
                        tma_load_3d(&sm.box[stage][0][0], &tmap, &sm.full[stage], xt * kTX, (int32_t)box_r0,
                                    frame0 + (int32_t)s, policy);
                    }
                    if (hit && kRT) {
                        // per class: the 256-column box (and lane 31's 16-column box at map column x0 + 248)
                        mbar_expect_tx(&sm.full[stage],
                                       (uint32_t)(p.rt_P * p.rt_B) * (kRowBytes + (lane31_boxes<AC>() ? 32u : 0u)));
                        for (int c = 0; c < p.rt_P; ++c) {
                            tma_load_3d(&sm.box[stage][c * p.rt_B][0], &maps.m[c], &sm.full[stage], xt * kTW,
                                        (int32_t)(rg.jb >> rg.lp), (int32_t)s, policy);
                            if (lane31_boxes<AC>())
                                tma_load_3d(&sm.l31[stage][c * p.rt_B31][0], &maps.m[8 + c], &sm.full[stage],
                                            xt * kTW + kTW - 8, (int32_t)(rg.jb >> rg.lp), (int32_t)s, policy);
                        }
                    }
                }
                __syncwarp();
                // row-copy mode: tile row 0's first pixel, and per frame row the byte step
                uint32_t d0 = 0, rs2 = 0;
                if (kRT) {
                    d0 = p.rt_d0;
                    rs2 = (uint32_t)((2 * p.row_stride) & 15);
                }
                if (consumer_copy<AC>()) {
                    // publish what the consumers copy into this stage (they run kLookahead stages behind)
                    if (lane == 0) {
                        CopyRec rec;
                        rec.row0 = p.raw + s * p.frame_stride + box_r0 * p.row_stride + (int64_t)xt * kTX;
                        rec.r_lo = (int32_t)max((int64_t)0, -box_r0);
                        rec.r_hi = (int32_t)min((int64_t)kBoxRowsUsed, p.h - box_r0);
                        rec.x0 = xt * kTX;
                        rec.state = hit ? 1 : 0;
                        sm.cp[stage] = rec;
                        mbar_arrive(&sm.geo[stage]);
                    }
                }
                if (AC == 2) {
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p.raw) +
                                         2u * (uintptr_t)(s * p.frame_stride + (int64_t)xt * kTX);
                    d0 = (uint32_t)(a0 & 15u);
                    rs2 = (uint32_t)((2 * p.row_stride) & 15);
                    if (hit) {
                        // one bulk copy per frame row inside [0, H): the row's 16-byte-aligned superset
                        const int64_t ncols = min((int64_t)kTX, p.w - (int64_t)xt * kTX);
                        uint32_t bytes[(kBoxRowsUsed + 31) / 32];
                        uint64_t src[(kBoxRowsUsed + 31) / 32];
                        uint32_t total = 0;
#pragma unroll
                        for (int j = 0; j < (kBoxRowsUsed + 31) / 32; ++j) {
                            const int r = lane + 32 * j;
                            const int64_t jr = box_r0 + r;
                            bytes[j] = 0;
                            src[j] = 0;
                            if (r < kBoxRowsUsed && jr >= 0 && jr < p.h) {
                                const uintptr_t a = a0 + 2u * (uintptr_t)(jr * p.row_stride);
                                const uint32_t lead = (uint32_t)(a & 15u);
                                src[j] = (uint64_t)(a - lead);
                                bytes[j] = (lead + 2u * (uint32_t)ncols + 15u) & ~15u;
                                total += bytes[j];
                            }
                        }
                        total = redux_add(total);
                        if (lane == 0) mbar_expect_tx(&sm.full[stage], total);
                        __syncwarp();
#pragma unroll
                        for (int j = 0; j < (kBoxRowsUsed + 31) / 32; ++j) {
                            if (bytes[j] == 0) continue;
                            const int r = lane + 32 * j;
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                                " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(&sm.box[stage][r][0])),
                                "l"(src[j]), "r"(bytes[j]), "r"(smem_addr(&sm.full[stage])), "l"(policy)
                                : "memory");
                        }
                    }
                }
                // regular stage (StageP): the tile lies inside the span and the window and, for the
                // canvas lerp, RN(u - off) = u - base - 1 + (1 - phi) +- 2^-31 for every row (phi =
                // frac(off) away from 0 and 1 by 2^-30, |u - off| < 2^20): taps j0 + r, j0 + r + 1
                // unclamped and f = 1 - phi within (H + 2) * 2^-52
                bool regular = false;
                // (consumer-copy mode: the copies land in the same 16-byte-aligned rows as a TMA box)
                if ((AC == 16 || consumer_copy<AC>() || kRT) && FORMULA == SSB_FORMULA_CANVAS && hit &&
                    SSB_REGULAR_STAGES && !kF64 &&
                    (int64_t)(ut + 1) * kTU <= p.u_count && lo <= tu0 && tu0 + kTU - 1 <= hi && p.h < (1 << 20)) {
                    StageP spv;
                    spv.off = off;
                    if (INTERP == SSB_INTERP_NEAREST) {
                        regular = true;
                        spv.a0 = (int32_t)(tu0 - lo - box_r0);  // = 0
                        spv.j0 = (int32_t)(tu0 - lo);
                        spv.w_lo = spv.w_hi = 0.f;
                    } else {
                        const double phi = __dsub_rn(off, floor(off));  // exact (off >= 0)
                        const bool int_off = phi == 0.0;
                        const int64_t j0 = tu0 - base - (int_off ? 0 : 1);
                        if ((int_off || (phi > 0x1p-30 && phi < 1.0 - 0x1p-30)) && j0 >= 0 && j0 + kTU <= p.h - 1) {
                            regular = true;
                            const double f = int_off ? 0.0 : __dsub_rn(1.0, phi);
                            const double m = __dadd_rn(1.1641532182693481e-10, __dmul_rn((double)(p.h + 2), 0x1p-52));
                            spv.w_lo = __double2float_rd(__dsub_rn(f, m));
                            spv.w_hi = __double2float_ru(__dadd_rn(f, m));
                            spv.a0 = (int32_t)(j0 - box_r0);
                            spv.j0 = (int32_t)j0;
                        }
                    }
                    if (regular && kRT) {
                        // tap rows j0 .. j0 + kTU of the stage: their shared addresses (two per lane)
                        const uint32_t box_addr = smem_addr(&sm.box[stage][0][0]);
#pragma unroll
                        for (int j = 0; j < (kTU + 1 + 31) / 32; ++j) {
                            const int i = lane + 32 * j;
                            if (i <= kTU) {
                                const uint32_t a = row_addr<AC>(spv.j0 + i, box_r0, box_addr, d0, rs2, rg);
                                sm.taddr[stage][i] = a;
                                if (lane31_boxes<AC>()) sm.taddr31[stage][i] = row_addr31(spv.j0 + i, d0, rs2, rg);
                            }
                        }
                    }
                    if (regular && lane == 0) {
                        sm.sp[stage] = spv;
                        sm.hdr[stage] = 0x7FFFu | (1u << 15) | (1u << 16) | (0x7FFFu << 17);
                    }
                }
                if (!regular) {
                uint32_t live[C::kRowWords];
#pragma unroll
                for (int j = 0; j < C::kRowWords; ++j) live[j] = 0;
                if (hit) {
                    const uint32_t box_addr = smem_addr(&sm.box[stage][0][0]);
#pragma unroll
                    for (int j = 0; j < C::kRowWords; ++j) {
                        const int r = lane + 32 * j;
                        bool l = false;
                        if (r < kTU)
                            l = make_row<INTERP, FORMULA, AC, kF64>(sm.rows[stage][r], tu0 + r,
                                                              (int64_t)ut * kTU + r < p.u_count, lo, hi, off, p.h,
                                                              box_r0, C::template box_rows<INTERP, FORMULA>(),
                                                              box_addr, zero_addr, d0, rs2, rg);
                        live[j] = __ballot_sync(0xffffffffu, l);
                    }
                }
                __syncwarp();
                // per consumer warp: any live row (bits 0..14); all rows live with chained
                // taps, off_b(k) == off_a(k+1), so tap rows are converted once and reused by
                // the next row (bits 17..31, canvas formula only)
                bool any = false, chained = false;
                if (lane < kConsumerWarps) {
                    const int r0 = lane * ROWS;  // ROWS divides 32: a warp's rows share one word
                    const uint32_t bits = (live[r0 / 32] >> (r0 % 32)) & ((1u << ROWS) - 1);
                    any = bits != 0;
                    if (INTERP == SSB_INTERP_LINEAR && bits == (1u << ROWS) - 1) {
                        const RowP *g = &sm.rows[stage][r0];
                        chained = true;
#pragma unroll
                        for (int k = 0; k + 1 < ROWS; ++k) chained &= g[k].off_b == g[k + 1].off_a;
                    }
                }
                const uint32_t any_mask = __ballot_sync(0xffffffffu, any);
                const uint32_t chain_mask = __ballot_sync(0xffffffffu, chained);
                if (lane == 0) sm.hdr[stage] = any_mask | (hit ? (1u << 16) : 0u) | (chain_mask << 17);
                }
                __syncwarp();
                mbar_arrive(&sm.full[stage]);
                if (++stage == kStages) { stage = 0; sphase ^= 1; }
            }
        }
        if (consumer_copy<AC>()) {
            // the consumers look kLookahead stages ahead: mark the stages past the last one
            for (int d = 0; d < kLookahead; ++d) {
                if (lane == 0) {
                    mbar_wait(&sm.empty[stage], sphase ^ 1);
                    sm.cp[stage].state = 2;
                    mbar_arrive(&sm.geo[stage]);
                }
                if (++stage == kStages) { stage = 0; sphase ^= 1; }
            }
        }
        return;
    }

    // ===================== consumer warps =====================
    uint32_t stage = 0, sphase = 0, q = 0, qphase = 0, xz_batch = 0;
    const size_t plane = (size_t)p.u_count * p.w;
    constexpr bool kT248 = kRT && !lane31_boxes<AC>();  // 248-column tiles: lane 31 outside the tile
    // 248-column tiles, max mode: lane 31 duplicates lane 30's columns
    const uint32_t lane_off = (kT248 && kMax ? min(lane, 30) : lane) * 16;
    // consumer-copy mode: copy this warp's share (rows r with r % 15 == warp) of stage g's box rows,
    // then arrive on its `full` barrier when the copies have landed
    uint32_t g_next = 0;  // next stage (in the global stage sequence) to copy for
    auto copy_stage = [&]() {
        const uint32_t slot = g_next % kStages;
        mbar_wait(&sm.geo[slot], (g_next / kStages) & 1u);
        ++g_next;
        const CopyRec rec = sm.cp[slot];
        if (rec.state == 2) return;
        if (rec.state == 1) {
            const int64_t xl = (int64_t)rec.x0 + lane * 8;
            const int npix = (int)max((int64_t)0, min((int64_t)8, p.w - xl));
            int r = rec.r_lo + ((warp - rec.r_lo) % kConsumerWarps + kConsumerWarps) % kConsumerWarps;
            const char *src = reinterpret_cast<const char *>(rec.row0 + r * p.row_stride + lane * 8);
            const int64_t step = 2 * kConsumerWarps * p.row_stride;
            uint32_t dst = smem_addr(&sm.box[slot][r][0]) + 16u * lane;
            constexpr int kPiece = AC == 2 ? 8 : AC;  // (AC 2 never takes this path)
            for (; r < rec.r_hi; r += kConsumerWarps, src += step, dst += 2u * kTX * kConsumerWarps) {
#pragma unroll
                for (int q2 = 0; q2 < 16 / kPiece; ++q2) {
                    if (q2 * (kPiece / 2) < npix)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst + q2 * kPiece),
                                     "l"(src + q2 * kPiece), "n"(kPiece)
                                     : "memory");
                }
            }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&sm.full[slot]))
                     : "memory");
    };
    if (consumer_copy<AC>())
        for (int d = 0; d < kLookahead; ++d) copy_stage();
    while (true) {
        int item = 0;
        if (lane == 0) {
            mbar_wait(&sm.qfull[q], qphase);
            item = sm.queue[q];
        }
        item = __shfl_sync(0xffffffffu, item, 0);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.qempty[q]);
        if (++q == kQueue) { q = 0; qphase ^= 1; }
        if (item < 0) break;

        int b, ut, xt;
        int64_t s_begin, s_end;
        decode<kTU>(item, p, b, ut, xt, s_begin, s_end);
        const int64_t x = (int64_t)xt * kTW + lane * 8;
        const bool col_ok = x < p.w && (!kT248 || lane < 31);
        // this lane's pixels inside (248-column tiles: lane 31 has none)
        const int nv = (kT248 && lane == 31) ? 0 : (int)max((int64_t)0, min((int64_t)8, p.w - x));
        const int64_t r0 = (int64_t)ut * kTU + warp * ROWS;  // window row of k = 0
        const int64_t rows_left = p.u_count - r0;
        const int rows_ok = rows_left <= 0 ? 0 : (rows_left >= ROWS ? ROWS : (int)rows_left);
        uint16_t *vrow = (VOL && p.vol != nullptr)
                             ? p.vol + b * p.vol_bstride + (size_t)s_begin * plane + (size_t)r0 * p.w + x
                             : nullptr;
        // warp-uniform fast path: every lane's 8 columns and all rows inside the output
        const bool fast =
            __all_sync(0xffffffffu, AC == 16 ? col_ok : (nv == 8 || (kT248 && lane == 31))) && rows_ok == ROWS;
        // SIDE == false kernels run only without XZ / YZ outputs: their blocks compile away
        uint32_t *yzp = (SIDE && p.yz != nullptr) ? p.yz + b * p.yz_bstride + (size_t)s_begin * p.u_count + r0 + lane
                                                  : nullptr;
        const bool has_xz = SIDE && p.xz != nullptr;
        int g = 0;  // slice within the current XZ batch

        uint4 acc_max[ROWS];
        uint32_t acc_sum[kMax ? 1 : ROWS][8];
#pragma unroll
        for (int k = 0; k < ROWS; ++k) {
            acc_max[k] = make_uint4(0, 0, 0, 0);
            if (!kMax)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc_sum[k][c] = 0;
        }

        const int ns = (int)(s_end - s_begin);
        // linear sums carry 2^23-biased voxels (rows_pass): bias to remove per live pass
        constexpr bool kBiased = !kMax && INTERP == SSB_INTERP_LINEAR && !kF64;
        uint32_t n_live = 0;
        for (int si = 0; si < ns; ++si) {
            if (consumer_copy<AC>()) copy_stage();  // the stage kLookahead ahead of this one
            mbar_wait(&sm.full[stage], sphase);
            const uint32_t hdr = sm.hdr[stage];
            const bool live = (hdr >> 16) & (hdr >> warp) & 1u;
            n_live += live ? 1u : 0u;
            uint4 xz_max = make_uint4(0, 0, 0, 0);
            uint32_t xz_sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            uint32_t yzv[ROWS];
#pragma unroll
            for (int k = 0; k < ROWS; ++k) yzv[k] = 0;
            if (live) {
                const RowP *rg = &sm.rows[stage][warp * ROWS];
                const bool chained = (hdr >> (17 + warp)) & 1u;
                const int64_t u0 = p.u_begin + r0;  // canvas row of this warp's row 0
#define SSB_ROWS_PASS(F, CH, RG)                                                                             \
    rows_pass<INTERP, FORMULA, kMax, F, ROWS, SIDE, CH, AC, RG, !VOL>(rg, lane_off, tap_base, tad, tad31, spv, \
                                                                     u0, vrow, p.w, rows_ok, \
                                                            col_ok, nv, acc_max, acc_sum, xz_max, xz_sum, yzv)
                if ((AC == 16 || consumer_copy<AC>() || kRT) && FORMULA == SSB_FORMULA_CANVAS && !kF64 &&
                    ((hdr >> 15) & 1u)) {
                    // regular stage: taps at fixed box rows, one weight bracket (StageP)
                    StageP spv = sm.sp[stage];
                    spv.j0 += warp * ROWS;  // frame row of tap a of this warp's row 0
                    const uint32_t *tad = kRT ? &sm.taddr[stage][warp * ROWS] : nullptr;
                    const uint32_t *tad31 = lane31_boxes<AC>() ? &sm.taddr31[stage][warp * ROWS] : nullptr;
                    const uint32_t tap_base = smem_addr(&sm.box[stage][0][0]) +
                                              (uint32_t)(spv.a0 + warp * ROWS) * (2u * row_pitch<AC>()) + lane_off;
                    if (fast) SSB_ROWS_PASS(true, true, true);
                    else SSB_ROWS_PASS(false, true, true);
                } else {
                    const StageP spv{};
                    const uint32_t tap_base = 0;
                    const uint32_t *tad = nullptr, *tad31 = nullptr;
                    // four specialisations so the row loop has no per-row branches
                    if (fast) {
                        if (chained) SSB_ROWS_PASS(true, true, false);
                        else SSB_ROWS_PASS(true, false, false);
                    } else {
                        if (chained) SSB_ROWS_PASS(false, true, false);
                        else SSB_ROWS_PASS(false, false, false);
                    }
                }
#undef SSB_ROWS_PASS
            } else if (vrow != nullptr && col_ok) {
                const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int k = 0; k < ROWS; ++k) {
                    if (k >= rows_ok) continue;
                    if (AC != 16 && nv < 8) stg_partial(vrow + (size_t)k * p.w, z, nv);
                    else stg8<acl<AC>()>(vrow + (size_t)k * p.w, z);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[stage]);
            if (++stage == kStages) { stage = 0; sphase ^= 1; }
            if (vrow != nullptr) vrow += plane;

            constexpr bool kYS = kMax && staged_yz<ROWS, SIDE, AC>();
            if (!kYS && yzp != nullptr) {
#if SSB_YZ_LIVE_ONLY
                // dead passes have all-zero rows (neutral for max and sum): no RED, no lane select
                if (live && lane < rows_ok) {
                    uint32_t val = yzv[0];
#pragma unroll
                    for (int k = 1; k < ROWS; ++k)
                        if (lane == k) val = yzv[k];
                    red_u32<kMax>(yzp, val);
                }
#else
                if (lane < rows_ok) {
                    uint32_t val = yzv[0];
#pragma unroll
                    for (int k = 1; k < ROWS; ++k)
                        if (lane == k) val = yzv[k];
                    if (val != 0) red_u32<kMax>(yzp, val);
                }
#endif
                yzp += p.u_count;
            }

            if (has_xz || (kYS && yzp != nullptr)) {
                const int buf = xz_batch & 1;
                if (kYS && yzp != nullptr) {
                    // this warp's row pairs (4w, 4w+1) and (4w+2, 4w+3): u16x2 words (pair's first row low)
                    const uint32_t t01 = __vmaxu2(__byte_perm(yzv[0], yzv[1], 0x5410), __byte_perm(yzv[0], yzv[1], 0x7632));
                    const uint32_t t23 = __vmaxu2(__byte_perm(yzv[2], yzv[3], 0x5410), __byte_perm(yzv[2], yzv[3], 0x7632));
                    const int rp0 = warp * 2, rp1 = rp0 + 1;
                    sm.yzs[buf][g][rp0][lane ^ ((rp0 & 7) << 2)] = t01;
                    sm.yzs[buf][g][rp1][lane ^ ((rp1 & 7) << 2)] = t23;
                }
                if (kMax && has_xz) {
                    uint32_t *dst = &sm.xz[((buf * kXzBatch + g) * kConsumerWarps + warp) * (kTX / 2) + lane * 4];
                    *reinterpret_cast<uint4 *>(dst) = xz_max;
                } else if (!kMax) {
                    uint32_t *dst = &sm.xz[(buf * kConsumerWarps + warp) * kTX + lane * 8];
                    if (kBiased && live) {
#pragma unroll
                        for (int c = 0; c < 8; ++c) xz_sum[c] -= (uint32_t)ROWS * kBias;
                    }
                    *reinterpret_cast<uint4 *>(dst) = make_uint4(xz_sum[0], xz_sum[1], xz_sum[2], xz_sum[3]);
                    *reinterpret_cast<uint4 *>(dst + 4) = make_uint4(xz_sum[4], xz_sum[5], xz_sum[6], xz_sum[7]);
                }
                if (g == kXzBatch - 1 || si + 1 == ns) {
                    named_bar_sync(1, kConsumerThreads);
                    const int64_t s0 = s_begin + si - g;  // first slice of this batch
                    if (kYS && yzp != nullptr && tid >= kXzBatch * (kTX / 2) &&
                        tid < kXzBatch * (kTX / 2) + kXzBatch * (kTU / 2)) {
                        // thread -> (slice of batch, row pair): max over the pair's 32 lane words, read in
                        // the swizzled order (conflict-free across the reducing threads)
                        const int t2 = tid - kXzBatch * (kTX / 2), gg = t2 / (kTU / 2), rp = t2 % (kTU / 2);
                        if (gg <= g) {
                            const uint32_t base = smem_addr(&sm.yzs[buf][gg][rp][0]);
                            uint4 a = make_uint4(0, 0, 0, 0);
#pragma unroll
                            for (int q = 0; q < 8; ++q) a = max_u16x8(a, lds128(base + 16u * (uint32_t)(q ^ (rp & 7))));
                            const uint32_t m = __vmaxu2(__vmaxu2(a.x, a.y), __vmaxu2(a.z, a.w));
                            const int64_t wr = (int64_t)ut * kTU + 2 * rp;  // window row of the pair's first row
                            uint32_t *dst = p.yz + b * p.yz_bstride + (size_t)(s0 + gg) * p.u_count + wr;
                            if ((m & 0xFFFFu) && wr < p.u_count) red_u32<true>(dst, m & 0xFFFFu);
                            if ((m >> 16) && wr + 1 < p.u_count) red_u32<true>(dst + 1, m >> 16);
                        }
                    }
                    if (kMax && has_xz) {
                        // thread -> (slice of batch, word of 2 columns)
                        const int gg = tid / (kTX / 2), c2 = tid % (kTX / 2);
                        const int64_t col = (int64_t)xt * kTW + 2 * c2;
                        if (gg <= g && 2 * c2 < kTW && col < p.w) {
                            uint32_t red = 0;
#pragma unroll
                            for (int w2 = 0; w2 < kConsumerWarps; ++w2)
                                red = __vmaxu2(red, sm.xz[((buf * kXzBatch + gg) * kConsumerWarps + w2) * (kTX / 2) + c2]);
                            uint32_t *dst = p.xz + b * p.xz_bstride + (size_t)(s0 + gg) * p.w + col;
                            if (red & 0xFFFFu) red_u32<true>(dst, red & 0xFFFFu);
                            if (red >> 16) red_u32<true>(dst + 1, red >> 16);
                        }
                    } else if (!kMax && tid < kTW) {
                        const int64_t col = (int64_t)xt * kTW + tid;
                        if (col < p.w) {
                            uint32_t red = 0;
#pragma unroll
                            for (int w2 = 0; w2 < kConsumerWarps; ++w2) red += sm.xz[(buf * kConsumerWarps + w2) * kTX + tid];
                            if (red) red_u32<false>(p.xz + b * p.xz_bstride + (size_t)s0 * p.w + col, red);
                        }
                    }
                    ++xz_batch;
                    g = 0;
                } else {
                    ++g;
                }
            }
        }

        if (p.xy != nullptr && col_ok) {
            uint32_t *base = p.xy + b * p.xy_bstride + (size_t)r0 * p.w + x;
#pragma unroll
            for (int k = 0; k < ROWS; ++k) {
                if (k >= rows_ok) break;
                uint32_t *dst = base + (size_t)k * p.w;
                if (kMax) {
                    const uint32_t w4[4] = {acc_max[k].x, acc_max[k].y, acc_max[k].z, acc_max[k].w};
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint32_t e = (w4[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                        if (e && (AC == 16 || c < nv)) red_u32<true>(dst + c, e);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint32_t v = acc_sum[k][c] - (kBiased ? n_live * kBias : 0u);
                        if (v && (AC == 16 || c < nv)) red_u32<false>(dst + c, v);
                    }
                }
            }
        }
    }
}

// --------------------------------------------------------------------------- host

// cuTensorMapEncodeTiled is a driver entry point, the same for every device: resolved once per
// process.  (Tensor maps themselves are encoded per call, for the caller's buffer.)
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

template <int INTERP, int FORMULA, int REDUCE, int ROWS, bool SIDE, int AC, bool VOL>
int launch_kernel(const TmapSet &map, const Params &prm, int grid, cudaStream_t st) {
    auto kern = deskew_tma_kernel<INTERP, FORMULA, REDUCE, ROWS, SIDE, AC, VOL>;
    constexpr int smem = (int)sizeof(Smem<ROWS, AC, SIDE>);
    static_assert(smem <= 227 * 1024, "shared memory budget");
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, kThreads, smem, st>>>(map, prm);
    return check_launch("deskew_tma_kernel");
}

// projection-only calls (no volume) of the TMA mode get the instantiation without store code
template <int INTERP, int FORMULA, int REDUCE, int ROWS, bool SIDE, int AC>
int launch_one(const TmapSet &map, const Params &prm, int grid, cudaStream_t st) {
    if constexpr (lane31_boxes<AC>()) {  // chosen for projection-only launches only
        return launch_kernel<INTERP, FORMULA, REDUCE, ROWS, SIDE, AC, false>(map, prm, grid, st);
    }
    if ((AC == 16 || consumer_copy<AC>() || rt_mode<AC>()) && prm.vol == nullptr)
        return launch_kernel<INTERP, FORMULA, REDUCE, ROWS, SIDE, AC, false>(map, prm, grid, st);
    return launch_kernel<INTERP, FORMULA, REDUCE, ROWS, SIDE, AC, true>(map, prm, grid, st);
}

// Kernel instantiation for (reduce, tile height, side projections requested):
//   max: 4 rows {with, without XZ/YZ}, 8 rows with XZ/YZ (projection-only, TMA mode only)
//   sum: 4 rows {with, without}
template <int INTERP, int FORMULA, int AC>
int launch_variant(bool mx, bool tall, bool side, const TmapSet &map, const Params &prm, int grid,
                   cudaStream_t st) {
    if (mx) {
        if (side) {
            if (AC == 16 && tall) return launch_one<INTERP, FORMULA, SSB_REDUCE_MAX, 8, true, 16>(map, prm, grid, st);
            return launch_one<INTERP, FORMULA, SSB_REDUCE_MAX, 4, true, AC>(map, prm, grid, st);
        }
        return launch_one<INTERP, FORMULA, SSB_REDUCE_MAX, 4, false, AC>(map, prm, grid, st);
    }
    if (side) return launch_one<INTERP, FORMULA, SSB_REDUCE_SUM, 4, true, AC>(map, prm, grid, st);
    return launch_one<INTERP, FORMULA, SSB_REDUCE_SUM, 4, false, AC>(map, prm, grid, st);
}

}  // namespace tma_path
}  // namespace ssb
