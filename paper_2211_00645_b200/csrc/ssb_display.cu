// Display encode epilogue: the gray8 payload of the live-view wire format.
//
// Reference (skewstream/server.py:83-91, encode_frame_packet):
//     lo, hi = pixels.min(), pixels.max();  range = hi - lo
//     range == 0  ->  zero payload
//     else        ->  rint((pixels.astype(f64) - lo) * (255.0 / range)).astype(uint8)
// One cooperative launch: phase 1 reduces min/max (16-byte loads, warp REDUX, one partial
// per CTA), a grid barrier, phase 2 re-reads the image (L2-resident: a display image is
// ~10 MB against 126 MB of L2) and writes the bytes.  fl(p - lo) is exact, 255.0 / range is
// one correctly rounded fp64 division, the product is rounded once and rint is half-even,
// exactly numpy's sequence.
#include <algorithm>
#include <cooperative_groups.h>

#include "ssb_common.cuh"
#include "ssb_host.h"

namespace ssb {
namespace {

namespace cg = cooperative_groups;

constexpr int kEncThreads = 256;
constexpr int kMaxEncBlocks = 4 * 148 * 2;  // stats words: 2 + 2 per CTA

__device__ __forceinline__ uint32_t redux_min_u32(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}

__device__ __forceinline__ uint32_t redux_max_u32(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}

__device__ __forceinline__ uint8_t gray8(uint32_t p, uint32_t lo, double scale) {
    return (uint8_t)__double2uint_rn(__dmul_rn((double)(p - lo), scale));
}

__global__ void __launch_bounds__(kEncThreads) encode_gray8_kernel(const uint16_t *__restrict__ src, int64_t count,
                                                                   uint8_t *__restrict__ dst, uint32_t *stats,
                                                                   int vec) {
    __shared__ uint32_t s_min[kEncThreads / 32], s_max[kEncThreads / 32];
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t nvec = vec ? count / 8 : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // ---- phase 1: min / max ----
    uint32_t mn2 = 0xFFFFFFFFu, mx2 = 0u;  // u16x2 lanes
    for (int64_t k = tid; k < nvec; k += nthreads) {
        const uint4 v = ldg_nc_v4(src + 8 * k);
        mn2 = __vminu2(__vminu2(__vminu2(__vminu2(mn2, v.x), v.y), v.z), v.w);
        mx2 = __vmaxu2(__vmaxu2(__vmaxu2(__vmaxu2(mx2, v.x), v.y), v.z), v.w);
    }
    uint32_t mn = min(mn2 & 0xFFFFu, mn2 >> 16), mx = max(mx2 & 0xFFFFu, mx2 >> 16);
    for (int64_t k = 8 * nvec + tid; k < count; k += nthreads) {
        const uint32_t p = src[k];
        mn = min(mn, p);
        mx = max(mx, p);
    }
    mn = redux_min_u32(mn);
    mx = redux_max_u32(mx);
    if (lane == 0) {
        s_min[warp] = mn;
        s_max[warp] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kEncThreads / 32; ++w) {
            mn = min(mn, s_min[w]);
            mx = max(mx, s_max[w]);
        }
        stats[2 + 2 * blockIdx.x] = mn;
        stats[3 + 2 * blockIdx.x] = mx;
    }
    cg::this_grid().sync();

    // ---- phase 2: every CTA folds the partials (a few hundred words), then encodes ----
    mn = 0xFFFFFFFFu;
    mx = 0u;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        mn = min(mn, __ldcg(stats + 2 + 2 * b));
        mx = max(mx, __ldcg(stats + 3 + 2 * b));
    }
    mn = redux_min_u32(mn);
    mx = redux_max_u32(mx);
    __syncthreads();  // s_min / s_max reuse
    if (lane == 0) {
        s_min[warp] = mn;
        s_max[warp] = mx;
    }
    __syncthreads();
    uint32_t lo = s_min[0], hi = s_max[0];
    for (int w = 1; w < kEncThreads / 32; ++w) {
        lo = min(lo, s_min[w]);
        hi = max(hi, s_max[w]);
    }
    const uint32_t range = hi - lo;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        stats[0] = lo;
        stats[1] = range;
    }
    const double scale = range == 0 ? 0.0 : __ddiv_rn(255.0, (double)range);
    for (int64_t k = tid; k < nvec; k += nthreads) {
        const uint4 v = ldg_nc_v4(src + 8 * k);
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
        uint32_t o[2] = {0u, 0u};
        if (range != 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t p = (w4[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
                o[c >> 2] |= (uint32_t)gray8(p, lo, scale) << (8 * (c & 3));
            }
        }
        *reinterpret_cast<uint2 *>(dst + 8 * k) = make_uint2(o[0], o[1]);
    }
    for (int64_t k = 8 * nvec + tid; k < count; k += nthreads)
        dst[k] = range == 0 ? (uint8_t)0 : gray8(src[k], lo, scale);
}

int enc_grid() {
    static int grid = 0;
    if (grid == 0) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode_gray8_kernel, kEncThreads, 0);
        grid = std::max(1, std::min(per_sm, 4)) * num_sms();
        grid = std::min(grid, kMaxEncBlocks);
    }
    return grid;
}

}  // namespace
}  // namespace ssb

extern "C" size_t ssb_encode_gray8_stats_bytes(void) { return (size_t)(2 + 2 * ssb::kMaxEncBlocks) * 4; }

extern "C" int ssb_encode_gray8(const uint16_t *src, int64_t count, uint8_t *dst, uint32_t *stats,
                                size_t stats_bytes, void *stream) {
    using namespace ssb;
    if (count < 0) return fail(SSB_ERR_PARAM, "negative count");
    if (stats == nullptr || stats_bytes < ssb_encode_gray8_stats_bytes())
        return fail(SSB_ERR_CAPACITY, "stats buffer too small: need %zu bytes", ssb_encode_gray8_stats_bytes());
    if (count == 0) return SSB_OK;
    if (src == nullptr || dst == nullptr) return fail(SSB_ERR_PARAM, "null image pointer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int vec = aligned16(src) && (reinterpret_cast<uintptr_t>(dst) & 7u) == 0;
    const int grid = enc_grid();
    void *args[] = {(void *)&src, (void *)&count, (void *)&dst, (void *)&stats, (void *)&vec};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void *)encode_gray8_kernel, dim3(grid),
                                                      dim3(kEncThreads), args, 0, st);
    if (e != cudaSuccess) return fail(SSB_ERR_CUDA, "encode_gray8_kernel: %s", cudaGetErrorString(e));
    count_launches(1);
    return check_launch("encode_gray8_kernel");
}
