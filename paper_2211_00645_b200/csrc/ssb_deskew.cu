// Fused deskew + XY/XZ/YZ projections (ssb_deskew) -- tiled path.
//
// Replaces the reference's per-frame numpy loop (ProjectionCanvas.place x N +
// finalize_global, ss/pipeline.py:316-336; _interp_slice_rows :229-236) and the
// batch oracle reference_deskew (ss/phantom.py:359-402) with one pass over HBM:
// every raw frame row is read once (+1 halo row per tile), every volume voxel is
// written once, and the projections are reduced on chip.
//
// Work decomposition: an item is (u-tile of TU canvas rows) x (x-tile of 256
// columns) x (chunk of slices).  A 256-thread CTA = 8 warps; warp w owns ROWS
// consecutive canvas rows, lane l owns 8 consecutive columns (16-byte vectors).
// For each slice of the chunk the CTA
//   * samples the frame (nearest copy or fp64 lerp, bit-exact with numpy),
//   * streams the voxels to the volume (st.global.cs, 512 B per warp-row),
//   * folds them into the XY accumulators held in registers (reduce over i),
//   * reduces each row over its 256 columns with REDUX (YZ partial per x-tile),
//   * reduces each column over its TU rows through shared memory (XZ partial
//     per u-tile).
// Partials of XY (per slice chunk), XZ (per u-tile) and YZ (per x-tile) land in
// the workspace and one small kernel folds them; when a dimension has a single
// partial the kernel writes the final projection directly.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ssb_common.cuh"
#include "ssb_host.h"
#include "ssb_plan.h"

namespace ssb {
namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kTX = 256;  // columns per tile: 32 lanes x 8

struct TileParams {
    const uint16_t *raw;
    uint16_t *vol;
    void *xy;  // base of XY planes (S planes of u_count*W), or final
    void *xz;  // base of XZ planes (UT planes of n*W), or final
    void *yz;  // base of YZ planes (XT planes of n*u_count), or final
    int64_t n, h, w, first, u_begin, u_count, chunk;
    int64_t row_stride, frame_stride;  // input strides (elements)
    double shear;
    int32_t UT, XT, S;
    int32_t xy_accumulate;
};

// 8 consecutive uint16 per lane.  VB = widest access the buffers' alignment allows (16, 8, 4 or
// 2 bytes): W % 8 == 0 stacks take 16-byte vectors, W % 4 == 0 (e.g. 4-pixel camera ROI steps) two
// 8-byte halves, even W four 4-byte words; lanes that straddle the row end go element by element.
template <int VB>
__device__ __forceinline__ uint4 load8(const uint16_t *row, int64_t x, int64_t w) {
    if (VB == 16) return ldg_nc_v4(row + x);
    uint32_t v[4] = {0, 0, 0, 0};
    if (VB > 2 && x + 8 <= w) {
        if (VB == 8) {
            const uint2 a = __ldg(reinterpret_cast<const uint2 *>(row + x));
            const uint2 b = __ldg(reinterpret_cast<const uint2 *>(row + x + 4));
            return make_uint4(a.x, a.y, b.x, b.y);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = __ldg(reinterpret_cast<const uint32_t *>(row + x + 2 * q));
        return make_uint4(v[0], v[1], v[2], v[3]);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if (x + c < w) v[c >> 1] |= (uint32_t)__ldg(row + x + c) << (16 * (c & 1));
    return make_uint4(v[0], v[1], v[2], v[3]);
}

template <int VB>
__device__ __forceinline__ void store8(uint16_t *row, int64_t x, int64_t w, uint4 v) {
    if (VB == 16) {
        stg_cs_v4(row + x, v);
        return;
    }
    const uint32_t q[4] = {v.x, v.y, v.z, v.w};
    if (VB > 2 && x + 8 <= w) {
        if (VB == 8) {
            asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(row + x), "r"(q[0]), "r"(q[1]) : "memory");
            asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(row + x + 4), "r"(q[2]), "r"(q[3]) : "memory");
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(row + x + 2 * k), "r"(q[k]) : "memory");
        }
        return;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if (x + c < w) row[x + c] = (uint16_t)(q[c >> 1] >> (16 * (c & 1)));
}

template <int ROWS, int INTERP, int FORMULA, int REDUCE, int VEC>
__global__ void __launch_bounds__(kThreads) deskew_tiles_kernel(const TileParams p) {
    constexpr int TU = kWarps * ROWS;
    constexpr bool kMax = REDUCE == SSB_REDUCE_MAX;
    __shared__ uint32_t xz_smem[kWarps][kTX];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int64_t item = blockIdx.x;
    const int sc = (int)(item % p.S);
    item /= p.S;
    const int xt = (int)(item % p.XT);
    const int ut = (int)(item / p.XT);

    const int64_t x = (int64_t)xt * kTX + lane * 8;
    const bool col_ok = x < p.w;
    const int64_t r0 = (int64_t)ut * TU + warp * ROWS;  // first row (within window) of this warp
    const int64_t tile_u0 = p.u_begin + (int64_t)ut * TU;
    const int64_t tile_u1 = tile_u0 + TU - 1;
    const int64_t s_begin = (int64_t)sc * p.chunk;
    const int64_t s_end = min(p.n, s_begin + p.chunk);
    const size_t frame_elems = (size_t)p.frame_stride;

    // XY accumulators: max -> 8 packed uint16 per row; sum -> 8 uint32 per row
    uint4 acc_max[ROWS];
    uint32_t acc_sum[kMax ? 1 : ROWS][8];
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
        acc_max[k] = make_uint4(0, 0, 0, 0);
        if (!kMax)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc_sum[k][c] = 0;
    }

    for (int64_t s = s_begin; s < s_end; ++s) {
        const int64_t gi = p.first + s;
        int64_t lo, hi;
        double off;
        slice_span(gi, p.shear, p.h, INTERP, lo, hi, off);
        const bool touches = !(hi < tile_u0 || lo > tile_u1);
        const uint16_t *frame = p.raw + (size_t)s * frame_elems;

        // lane k < ROWS derives the sampling parameters of row r0 + k
        RowParam mine;
        mine.kind = 0;
        mine.j0 = mine.j1 = 0;
        mine.c0 = 0.0;
        mine.c1 = 1.0;
        if (touches && lane < ROWS) {
            const int64_t r = r0 + lane;
            const int64_t u = p.u_begin + r;
            if (r < p.u_count && u >= lo && u <= hi) mine = row_param<INTERP, FORMULA>(u, lo, off, p.h);
        }

        uint4 xz_max = make_uint4(0, 0, 0, 0);
        uint32_t xz_sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};

#pragma unroll
        for (int k = 0; k < ROWS; ++k) {
            RowParam rp;
            rp.kind = __shfl_sync(0xffffffffu, mine.kind, k);
            rp.j0 = __shfl_sync(0xffffffffu, mine.j0, k);
            rp.j1 = __shfl_sync(0xffffffffu, mine.j1, k);
            if (INTERP == SSB_INTERP_LINEAR) {
                rp.c0 = __shfl_sync(0xffffffffu, mine.c0, k);
                rp.c1 = __shfl_sync(0xffffffffu, mine.c1, k);
            }
            const int64_t r = r0 + k;
            const bool row_ok = r < p.u_count;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (rp.kind != 0 && col_ok) {
                const uint4 a = load8<VEC>(frame + (size_t)rp.j0 * p.row_stride, x, p.w);
                if (rp.kind == 1) {
                    v = a;
                } else {
                    const uint4 b = load8<VEC>(frame + (size_t)rp.j1 * p.row_stride, x, p.w);
                    v = lerp8<FORMULA>(a, b, rp);
                }
            }
            if (p.vol != nullptr && row_ok && col_ok)
                store8<VEC>(p.vol + ((size_t)s * p.u_count + r) * p.w, x, p.w, v);
            if (kMax) {
                acc_max[k] = max_u16x8(acc_max[k], v);
                xz_max = max_u16x8(xz_max, v);
            } else {
                const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t e = (q[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                    acc_sum[k][c] += e;
                    xz_sum[c] += e;
                }
            }
            if (p.yz != nullptr) {
                const uint32_t part = kMax ? hmax_u16x8(v) : hsum_u16x8(v);
                const uint32_t red = kMax ? __reduce_max_sync(0xffffffffu, part)
                                          : __reduce_add_sync(0xffffffffu, part);
                if (lane == 0 && row_ok) {
                    const size_t idx = (size_t)xt * p.n * p.u_count + (size_t)s * p.u_count + r;
                    if (kMax) static_cast<uint16_t *>(p.yz)[idx] = (uint16_t)red;
                    else static_cast<uint32_t *>(p.yz)[idx] = red;
                }
            }
        }

        if (p.xz != nullptr) {
            // column partial over this warp's rows -> smem -> reduce over warps
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint32_t e;
                if (kMax) {
                    const uint32_t q[4] = {xz_max.x, xz_max.y, xz_max.z, xz_max.w};
                    e = (q[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                } else {
                    e = xz_sum[c];
                }
                xz_smem[warp][lane * 8 + c] = e;
            }
            __syncthreads();
            const int64_t col = (int64_t)xt * kTX + tid;
            if (col < p.w) {
                uint32_t red = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) red = kMax ? max(red, xz_smem[w][tid]) : red + xz_smem[w][tid];
                const size_t idx = (size_t)ut * p.n * p.w + (size_t)s * p.w + col;
                if (kMax) static_cast<uint16_t *>(p.xz)[idx] = (uint16_t)red;
                else static_cast<uint32_t *>(p.xz)[idx] = red;
            }
            __syncthreads();
        }
    }

    if (p.xy == nullptr || !col_ok) return;
    const size_t plane = (size_t)p.u_count * p.w;
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
        const int64_t r = r0 + k;
        if (r >= p.u_count) break;
        const size_t base = (size_t)sc * plane + (size_t)r * p.w + x;
        if (kMax) {
            uint16_t *dst = static_cast<uint16_t *>(p.xy) + base;
            uint4 v = acc_max[k];
            if (p.xy_accumulate) v = max_u16x8(v, load8<VEC>(dst, 0, p.w - x));
            store8<VEC>(dst, 0, p.w - x, v);
        } else {
            uint32_t *dst = static_cast<uint32_t *>(p.xy) + base;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (x + c >= p.w) break;
                dst[c] = p.xy_accumulate ? dst[c] + acc_sum[k][c] : acc_sum[k][c];
            }
        }
    }
}

// dst[m] = reduce_p src[p*M + m] (optionally also over the old dst[m])
template <typename T, bool kMax>
__global__ void reduce_planes_kernel(const T *__restrict__ src, T *__restrict__ dst, int64_t planes,
                                     int64_t m_total, int accumulate) {
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < m_total;
         m += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = accumulate ? (uint32_t)dst[m] : 0u;
        for (int64_t q = 0; q < planes; ++q) {
            const uint32_t e = (uint32_t)src[q * m_total + m];
            v = kMax ? max(v, e) : v + e;
        }
        dst[m] = (T)v;
    }
}

struct Plan {
    int64_t TU, UT, XT, S, chunk;
    size_t esz;                  // bytes per projection element
    size_t xy_ws, xz_ws, yz_ws;  // workspace bytes per partial kind (0 = written directly)
};

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }
constexpr size_t kCounterBytes = 256;  // scheduler counter at the head of the workspace

int64_t env_int(const char *name, int64_t dflt) {
    const char *v = getenv(name);
    return v ? atoll(v) : dflt;
}

// tu: canvas rows per work item of the kernel that will run.
Plan make_plan(const ssb_deskew_desc &d, bool want_xy, bool want_xz, bool want_yz, int64_t tu, bool persistent) {
    Plan pl{};
    pl.TU = tu;
    pl.UT = std::max<int64_t>(1, (d.u_count + tu - 1) / tu);
    pl.XT = std::max<int64_t>(1, (d.width + kTX - 1) / kTX);
    const int64_t tiles = pl.UT * pl.XT;
    // enough items for the scheduler to balance: ~4 per resident CTA slot
    const int64_t slots = (int64_t)num_sms() * (persistent ? 1 : 2);
    int64_t S = std::max<int64_t>(1, (env_int("SSB_ITEMS_PER_SLOT", 4) * slots + tiles - 1) / tiles);
    S = std::min<int64_t>(S, env_int("SSB_MAX_SLICE_CHUNKS", 8));
    S = std::min<int64_t>(S, std::max<int64_t>(1, d.n));
    pl.chunk = std::max<int64_t>(1, (d.n + S - 1) / S);
    pl.S = std::max<int64_t>(1, (d.n + pl.chunk - 1) / pl.chunk);
    pl.esz = d.reduce == SSB_REDUCE_MAX ? 2 : 4;
    pl.xy_ws = (want_xy && pl.S > 1) ? align_up((size_t)pl.S * d.u_count * d.width * pl.esz) : 0;
    pl.xz_ws = (want_xz && pl.UT > 1) ? align_up((size_t)pl.UT * d.n * d.width * pl.esz) : 0;
    pl.yz_ws = (want_yz && pl.XT > 1) ? align_up((size_t)pl.XT * d.n * d.u_count * pl.esz) : 0;
    return pl;
}

int64_t tiled_rows(const ssb_deskew_desc &d) { return kWarps * (d.reduce == SSB_REDUCE_MAX ? 8 : 4); }

int validate(const ssb_deskew_desc *d) {
    if (d == nullptr) return fail(SSB_ERR_PARAM, "null descriptor");
    if (d->n < 0 || d->height < 1 || d->width < 1)
        return fail(SSB_ERR_PARAM, "bad stack shape n=%lld H=%lld W=%lld", (long long)d->n,
                    (long long)d->height, (long long)d->width);
    if (!(d->shear_px >= 0.0)) return fail(SSB_ERR_PARAM, "shear_px must be >= 0, got %g", d->shear_px);
    if (d->interp != SSB_INTERP_NEAREST && d->interp != SSB_INTERP_LINEAR)
        return fail(SSB_ERR_PARAM, "interp must be nearest or linear");
    if (d->formula != SSB_FORMULA_CANVAS && d->formula != SSB_FORMULA_NPINTERP)
        return fail(SSB_ERR_PARAM, "unknown formula %d", d->formula);
    if (d->reduce != SSB_REDUCE_MAX && d->reduce != SSB_REDUCE_SUM)
        return fail(SSB_ERR_PARAM, "reduce must be max or sum");
    if (d->u_count < 0 || d->u_begin < 0) return fail(SSB_ERR_PARAM, "bad canvas row window");
    if (d->height > INT32_MAX) return fail(SSB_ERR_CAPACITY, "frame height too large");
    if (d->row_stride != 0 && d->row_stride < d->width) return fail(SSB_ERR_PARAM, "row_stride < width");
    if (d->frame_stride != 0 && d->frame_stride < row_stride_of(*d) * (d->height - 1) + d->width)
        return fail(SSB_ERR_PARAM, "frame_stride too small for the frame");
    return SSB_OK;
}

template <int ROWS, int INTERP, int FORMULA, int REDUCE>
void launch_tiles(const TileParams &tp, int64_t items, int vec, cudaStream_t st) {
    const unsigned g = (unsigned)items;
    if (vec == 16) deskew_tiles_kernel<ROWS, INTERP, FORMULA, REDUCE, 16><<<g, kThreads, 0, st>>>(tp);
    else if (vec == 8) deskew_tiles_kernel<ROWS, INTERP, FORMULA, REDUCE, 8><<<g, kThreads, 0, st>>>(tp);
    else if (vec == 4) deskew_tiles_kernel<ROWS, INTERP, FORMULA, REDUCE, 4><<<g, kThreads, 0, st>>>(tp);
    else deskew_tiles_kernel<ROWS, INTERP, FORMULA, REDUCE, 2><<<g, kThreads, 0, st>>>(tp);
}

template <int REDUCE>
void dispatch_interp(const ssb_deskew_desc &d, const TileParams &tp, int64_t items, int vec,
                     cudaStream_t st) {
    constexpr int R = REDUCE == SSB_REDUCE_MAX ? 8 : 4;
    if (d.interp == SSB_INTERP_NEAREST)
        launch_tiles<R, SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, REDUCE>(tp, items, vec, st);
    else if (d.formula == SSB_FORMULA_CANVAS)
        launch_tiles<R, SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, REDUCE>(tp, items, vec, st);
    else
        launch_tiles<R, SSB_INTERP_LINEAR, SSB_FORMULA_NPINTERP, REDUCE>(tp, items, vec, st);
}

void launch_reduce(const void *src, void *dst, int64_t planes, int64_t m, bool is_max, bool accumulate,
                   cudaStream_t st) {
    if (m <= 0) return;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((m + threads - 1) / threads, (int64_t)num_sms() * 8);
    if (is_max)
        reduce_planes_kernel<uint16_t, true><<<(unsigned)blocks, threads, 0, st>>>(
            static_cast<const uint16_t *>(src), static_cast<uint16_t *>(dst), planes, m, accumulate);
    else
        reduce_planes_kernel<uint32_t, false><<<(unsigned)blocks, threads, 0, st>>>(
            static_cast<const uint32_t *>(src), static_cast<uint32_t *>(dst), planes, m, accumulate);
    count_launches(1);
}

}  // namespace
}  // namespace ssb

using namespace ssb;

__global__ void fold_u16_into_u32_max(const uint16_t *__restrict__ src, uint32_t *__restrict__ dst, int64_t m) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = max(dst[k], (uint32_t)src[k]);
}

extern "C" size_t ssb_deskew_workspace_bytes(const ssb_deskew_desc *d) {
    if (validate(d) != SSB_OK) return 0;
    const Plan b = make_plan(*d, true, true, true, tiled_rows(*d), false);
    const size_t base = std::max(tma_workspace_bytes(*d), kCounterBytes + b.xy_ws + b.xz_ws + b.yz_ws);
    // SSB_FLAG_XY_U32 on the tiled path folds through a uint16 image kept after the scratch
    const bool xy_u32 = d->reduce == SSB_REDUCE_MAX && (d->flags & SSB_FLAG_XY_U32);
    return base + (xy_u32 ? align_up((size_t)d->u_count * d->width * 2) : 0);
}

extern "C" int ssb_deskew(const ssb_deskew_desc *d, const uint16_t *raw, uint16_t *vol, void *xy,
                          void *xz, void *yz, void *workspace, size_t workspace_bytes, void *stream) {
    if (int rc = validate(d)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (d->n == 0 || d->u_count == 0) {
        // nothing placed: projections of an empty window are zero (XY unless accumulating)
        // (and XZ (n, W) / YZ (n, u_count) of an empty window: all-zero rows)
        const size_t esz = d->reduce == SSB_REDUCE_MAX ? 2 : 4;
        if (xy && !(d->flags & (SSB_FLAG_XY_ACCUMULATE | SSB_FLAG_XY_U32)))
            cudaMemsetAsync(xy, 0, (size_t)d->u_count * d->width * esz, st);
        if (xz) cudaMemsetAsync(xz, 0, (size_t)d->n * d->width * esz, st);
        if (yz) cudaMemsetAsync(yz, 0, (size_t)d->n * d->u_count * esz, st);
        return check_launch("ssb_deskew(empty)");
    }
    if (raw == nullptr) return fail(SSB_ERR_PARAM, "raw frames pointer is null");
    // a handful of frames folded into XY only (ProjectionCanvas.place, ss/pipeline.py:316-323) is
    // one small launch of the tiled kernel: no scratch reset, no finalize pass
    const bool tiny = d->n <= 2 && xz == nullptr && yz == nullptr;
    const bool xy_u32 = d->reduce == SSB_REDUCE_MAX && (d->flags & SSB_FLAG_XY_U32);
    const int ac = (env_int("SSB_DISABLE_TMA", 0) == 0 && (!tiny || xy_u32)) ? persistent_access_class(*d, raw, vol, xy) : 0;
    if (ac) return launch_deskew_tma(*d, raw, vol, xy, xz, yz, workspace, workspace_bytes, st, ac);
    if (xy_u32) {
        // the other paths narrow XY to uint16: run the call into a uint16 image after the scratch,
        // then max-fold it into the caller's uint32 accumulator
        ssb_deskew_desc d2 = *d;
        d2.flags &= ~(SSB_FLAG_XY_U32 | SSB_FLAG_XY_ACCUMULATE);
        const size_t base = ssb_deskew_workspace_bytes(&d2), m = (size_t)d->u_count * d->width;
        if (workspace == nullptr || workspace_bytes < base + align_up(m * 2))
            return fail(SSB_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", base + align_up(m * 2),
                        workspace_bytes);
        uint16_t *xy16 = reinterpret_cast<uint16_t *>(static_cast<char *>(workspace) + base);
        if (int rc = ssb_deskew(&d2, raw, vol, xy16, xz, yz, workspace, base, stream)) return rc;
        const int blocks = (int)std::min<int64_t>(((int64_t)m + 255) / 256, (int64_t)num_sms() * 8);
        fold_u16_into_u32_max<<<std::max(blocks, 1), 256, 0, st>>>(xy16, static_cast<uint32_t *>(xy), (int64_t)m);
        count_launches(1);
        return check_launch("fold_u16_into_u32_max");
    }

    const Plan pl = make_plan(*d, xy != nullptr, xz != nullptr, yz != nullptr, tiled_rows(*d), false);
    const size_t need = kCounterBytes + pl.xy_ws + pl.xz_ws + pl.yz_ws;
    if (workspace == nullptr || workspace_bytes < need)
        return fail(SSB_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", need, workspace_bytes);

    char *ws = static_cast<char *>(workspace) + kCounterBytes;
    void *xy_dst = pl.xy_ws ? (void *)ws : xy;
    void *xz_dst = pl.xz_ws ? (void *)(ws + pl.xy_ws) : xz;
    void *yz_dst = pl.yz_ws ? (void *)(ws + pl.xy_ws + pl.xz_ws) : yz;
    const int xy_acc = (pl.xy_ws == 0 && (d->flags & SSB_FLAG_XY_ACCUMULATE)) ? 1 : 0;
    {
        TileParams tp{};
        tp.raw = raw;
        tp.vol = vol;
        tp.xy = xy_dst;
        tp.xz = xz_dst;
        tp.yz = yz_dst;
        tp.n = d->n;
        tp.h = d->height;
        tp.w = d->width;
        tp.row_stride = row_stride_of(*d);
        tp.frame_stride = frame_stride_of(*d);
        tp.first = d->first_slice;
        tp.u_begin = d->u_begin;
        tp.u_count = d->u_count;
        tp.chunk = pl.chunk;
        tp.shear = d->shear_px;
        tp.UT = (int32_t)pl.UT;
        tp.XT = (int32_t)pl.XT;
        tp.S = (int32_t)pl.S;
        tp.xy_accumulate = xy_acc;
        // widest access every buffer's alignment allows (element strides and base addresses)
        auto fits = [&](int vb) {
            const int64_t e = vb / 2;
            const uintptr_t m = (uintptr_t)vb - 1;
            return d->width % e == 0 && tp.row_stride % e == 0 && tp.frame_stride % e == 0 &&
                   ((uintptr_t)raw & m) == 0 && ((uintptr_t)vol & m) == 0 &&
                   (d->reduce != SSB_REDUCE_MAX || ((uintptr_t)tp.xy & m) == 0);
        };
        const int vec = fits(16) ? 16 : fits(8) ? 8 : fits(4) ? 4 : 2;
        const int64_t items = pl.UT * pl.XT * pl.S;
        if (items > INT32_MAX) return fail(SSB_ERR_CAPACITY, "too many tiles");
        profile_begin(st);
        if (d->reduce == SSB_REDUCE_MAX) dispatch_interp<SSB_REDUCE_MAX>(*d, tp, items, vec, st);
        else dispatch_interp<SSB_REDUCE_SUM>(*d, tp, items, vec, st);
        profile_end(st);
        count_launches(1);
        if (int rc = check_launch("deskew_tiles_kernel")) return rc;
    }

    const bool is_max = d->reduce == SSB_REDUCE_MAX;
    if (pl.xy_ws) launch_reduce(xy_dst, xy, pl.S, d->u_count * d->width, is_max,
                                (d->flags & SSB_FLAG_XY_ACCUMULATE) != 0, st);
    if (pl.xz_ws) launch_reduce(xz_dst, xz, pl.UT, d->n * d->width, is_max, false, st);
    if (pl.yz_ws) launch_reduce(yz_dst, yz, pl.XT, d->n * d->u_count, is_max, false, st);
    return check_launch("reduce_planes_kernel");
}

extern "C" size_t ssb_deskew_batch_workspace_bytes(const ssb_deskew_desc *d, int64_t batch) {
    if (validate(d) != SSB_OK || batch < 1) return 0;
    return std::max(ssb_deskew_workspace_bytes(d), tma_workspace_bytes(*d, batch));
}

extern "C" int ssb_deskew_batch(const ssb_deskew_desc *d, int64_t batch, const uint16_t *raw, uint16_t *vol,
                                void *xy, void *xz, void *yz, void *workspace, size_t workspace_bytes,
                                void *stream) {
    if (int rc = validate(d)) return rc;
    if (batch < 1) return fail(SSB_ERR_PARAM, "batch must be >= 1, got %lld", (long long)batch);
    if (batch == 1) return ssb_deskew(d, raw, vol, xy, xz, yz, workspace, workspace_bytes, stream);
    if (raw == nullptr && d->n > 0) return fail(SSB_ERR_PARAM, "raw frames pointer is null");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t fs = frame_stride_of(*d);
    // one persistent launch over every stack when the frames reach shared memory by TMA boxes
    // (stacks back to back: stack b's frame k is frame b*n + k of one tensor map)
    if (d->n > 0 && d->u_count > 0 && env_int("SSB_DISABLE_TMA", 0) == 0 &&
        persistent_access_class(*d, raw, vol, xy) == 16)
        return launch_deskew_tma(*d, raw, vol, xy, xz, yz, workspace, workspace_bytes, st, 16, batch);
    // otherwise stack by stack (same results, one launch each)
    const size_t esz = d->reduce == SSB_REDUCE_MAX ? 2 : 4;
    for (int64_t b = 0; b < batch; ++b) {
        const int rc = ssb_deskew(
            d, raw ? raw + b * d->n * fs : nullptr, vol ? vol + b * d->n * d->u_count * d->width : nullptr,
            xy ? static_cast<char *>(xy) + b * d->u_count * d->width * esz : nullptr,
            xz ? static_cast<char *>(xz) + b * d->n * d->width * esz : nullptr,
            yz ? static_cast<char *>(yz) + b * d->n * d->u_count * esz : nullptr, workspace, workspace_bytes, stream);
        if (rc) return rc;
    }
    return SSB_OK;
}
