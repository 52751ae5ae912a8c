// Rolling-mode band recompute, display warp, projection combine, and the small
// library entry points (version, last error, launch counter).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "ssb_common.cuh"
#include "ssb_host.h"

namespace ssb {

namespace {
thread_local std::string g_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_error(const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
}

void count_launches(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

namespace {
struct Profiler {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t take() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
};
thread_local Profiler g_prof;
}  // namespace

void profile_begin(cudaStream_t st) {
    if (!g_prof.on) return;
    cudaEvent_t a = g_prof.take(), b = g_prof.take();
    cudaEventRecord(a, st);
    g_prof.pending.emplace_back(a, b);
}

void profile_end(cudaStream_t st) {
    if (!g_prof.on || g_prof.pending.empty()) return;
    cudaEventRecord(g_prof.pending.back().second, st);
}

namespace {

// Value ring slot k offers canvas row u, column x: the sample place() would use
// (canvas formula, ss/pipeline.py:283-290); 0 when the slot is empty or u is outside
// its span.
template <int INTERP>
__device__ __forceinline__ uint32_t ring_offer(const uint16_t *__restrict__ ring, const uint8_t *__restrict__ present,
                                               int64_t k, int64_t u, int64_t x, int64_t h, int64_t w, double s) {
    if (!present[k]) return 0;
    int64_t klo, khi;
    double off;
    slice_span(k, s, h, INTERP, klo, khi, off);
    if (u < klo || u > khi) return 0;
    const RowParam rp = row_param<INTERP, SSB_FORMULA_CANVAS>(u, klo, off, h);
    const uint16_t *frame = ring + (size_t)k * h * w;
    const uint32_t a = frame[(size_t)rp.j0 * w + x];
    return rp.kind == 2 ? lerp_voxel<SSB_FORMULA_CANVAS>(a, frame[(size_t)rp.j1 * w + x], rp) : a;
}

// Slots whose span can contain canvas row u: i*s within [u-H-1, u+1] (exact check in ring_offer).
__device__ __forceinline__ void ring_range(int64_t u, int64_t n_ring, int64_t h, double s, int64_t &k_lo,
                                           int64_t &k_hi) {
    k_lo = 0;
    k_hi = n_ring - 1;
    if (s > 0.0) {
        const double kl = floor(((double)(u - h) - 2.0) / s);
        const double kh = ceil(((double)u + 2.0) / s);
        k_lo = kl <= 0.0 ? 0 : (kl >= (double)n_ring ? n_ring : (int64_t)kl);
        k_hi = kh >= (double)(n_ring - 1) ? n_ring - 1 : (kh < 0.0 ? -1 : (int64_t)kh);
    }
}

// ss/pipeline.py:361-377, full recompute of a band.  One thread per (row, column).  Strict
// '>' in ring order keeps the first maximum; contributor -1 where every offer is 0.
template <int INTERP>
__global__ void rolling_full_kernel(const uint16_t *__restrict__ ring, const uint8_t *__restrict__ present,
                                    int64_t n_ring, int64_t h, int64_t w, double s, int64_t lo, int64_t hi,
                                    uint16_t *__restrict__ canvas, int16_t *__restrict__ contrib) {
    const int64_t total = (hi - lo + 1) * w;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = lo + e / w;
        const int64_t x = e % w;
        int64_t k_lo, k_hi;
        ring_range(u, n_ring, h, s, k_lo, k_hi);
        uint32_t best = 0;
        int32_t who = -1;
        for (int64_t k = k_lo; k <= k_hi; ++k) {
            const uint32_t v = ring_offer<INTERP>(ring, present, k, u, x, h, w, s);
            if (v > best) {
                best = v;
                who = (int32_t)k;
            }
        }
        canvas[(size_t)u * w + x] = (uint16_t)best;
        contrib[(size_t)u * w + x] = (int16_t)who;
    }
}

// Incremental pass (replaced = k, canvas exact before slot k changed): a voxel whose
// contributor is not k keeps its maximum unless the new offer v of slot k beats it -- v > best,
// or v == best > 0 with k earlier in ring order -- which is exactly the full re-max (every
// other slot's offer is unchanged and <= best, with ties only at later ring indices).  Voxels
// that k contributed to need the whole ring: they are appended to a list (a few per thousand:
// one slot of the ~H/s overlapping ones is each voxel's maximum) for rolling_remax_kernel, so
// no warp serialises a ring-long loop behind one lane.
template <int INTERP>
__global__ void rolling_incr_kernel(const uint16_t *__restrict__ ring, const uint8_t *__restrict__ present,
                                    int64_t n_ring, int64_t h, int64_t w, double s, int64_t lo, int64_t hi,
                                    uint16_t *__restrict__ canvas, int16_t *__restrict__ contrib, int32_t replaced,
                                    uint32_t *__restrict__ list, uint32_t *__restrict__ count) {
    const int64_t total = (hi - lo + 1) * w;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = lo + e / w;
        const int64_t x = e % w;
        const size_t idx = (size_t)u * w + x;
        const int32_t who = contrib[idx];
        if (who == replaced) {
            list[atomicAdd(count, 1u)] = (uint32_t)e;
            continue;
        }
        const uint32_t best = canvas[idx];
        const uint32_t v = ring_offer<INTERP>(ring, present, replaced, u, x, h, w, s);
        if (v > best || (v == best && v > 0 && replaced < who)) {
            canvas[idx] = (uint16_t)v;
            contrib[idx] = (int16_t)replaced;
        }
    }
}

// Full re-max of the listed voxels: one warp per voxel, lanes over ring slots (32 at a time),
// first maximum by a max then a min-index reduction.
template <int INTERP>
__global__ void rolling_remax_kernel(const uint16_t *__restrict__ ring, const uint8_t *__restrict__ present,
                                     int64_t n_ring, int64_t h, int64_t w, double s, int64_t lo,
                                     uint16_t *__restrict__ canvas, int16_t *__restrict__ contrib,
                                     const uint32_t *__restrict__ list, const uint32_t *__restrict__ count) {
    const int lane = threadIdx.x & 31;
    const uint32_t n = *count;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
        const int64_t e = list[i];
        const int64_t u = lo + e / w;
        const int64_t x = e % w;
        int64_t k_lo, k_hi;
        ring_range(u, n_ring, h, s, k_lo, k_hi);
        uint32_t best = 0;
        int32_t who = -1;
        for (int64_t k0 = k_lo; k0 <= k_hi; k0 += 32) {
            const int64_t k = k0 + lane;
            const uint32_t v = k <= k_hi ? ring_offer<INTERP>(ring, present, k, u, x, h, w, s) : 0u;
            const uint32_t m = __reduce_max_sync(0xffffffffu, v);
            if (m > best) {  // strict: an equal maximum in a later chunk keeps the earlier slot
                best = m;
                who = (int32_t)__reduce_min_sync(0xffffffffu, v == m ? (uint32_t)k : 0xFFFFFFFFu);
            }
        }
        if (lane == 0) {
            canvas[(size_t)u * w + x] = (uint16_t)best;
            contrib[(size_t)u * w + x] = (int16_t)who;
        }
    }
}

// ss/pipeline.py:451-457: m = clip(arange/scale, 0, rows-1); lerp rows m0, m1; rint.
__global__ void warp_rows_kernel(const uint16_t *__restrict__ proj, int64_t rows, int64_t cols,
                                 double scale, uint16_t *__restrict__ out, int64_t out_rows) {
    const int64_t total = out_rows * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = e / cols, c = e % cols;
        double mm = __ddiv_rn((double)m, scale);
        mm = fmin(fmax(mm, 0.0), (double)(rows - 1));
        const int64_t m0 = (int64_t)floor(mm);
        const int64_t m1 = m0 + 1 < rows - 1 ? m0 + 1 : rows - 1;
        RowParam rp;
        rp.c1 = __dsub_rn(mm, (double)m0);
        rp.c0 = __dsub_rn(1.0, rp.c1);
        rp.kind = 2;
        out[e] = (uint16_t)lerp_voxel<SSB_FORMULA_CANVAS>(proj[m0 * cols + c], proj[m1 * cols + c], rp);
    }
}

template <typename T, bool kMax>
__global__ void combine_kernel(const T *__restrict__ src, T *__restrict__ dst, int64_t count) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = dst[e], b = src[e];
        dst[e] = (T)(kMax ? max(a, b) : a + b);
    }
}

unsigned grid_for(int64_t total, int threads) {
    const int64_t b = (total + threads - 1) / threads;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 16));
}

}  // namespace
}  // namespace ssb

using namespace ssb;

extern "C" int ssb_version(void) { return SSB_VERSION; }

extern "C" const char *ssb_last_error(void) { return ssb::g_error.c_str(); }

extern "C" int64_t ssb_launch_count(void) { return ssb::g_launches.load(); }

extern "C" int ssb_profile_enable(int32_t on) {
    ssb::g_prof.on = on != 0;
    return SSB_OK;
}

extern "C" int ssb_profile_read(double *total_ms, int64_t *launches) {
    double sum = 0.0;
    int64_t k = 0;
    for (auto &pr : ssb::g_prof.pending) {
        if (cudaEventSynchronize(pr.second) != cudaSuccess) return fail(SSB_ERR_CUDA, "profile event sync failed");
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
            sum += ms;
            ++k;
        }
        ssb::g_prof.pool.push_back(pr.first);
        ssb::g_prof.pool.push_back(pr.second);
    }
    ssb::g_prof.pending.clear();
    if (total_ms) *total_ms = sum;
    if (launches) *launches = k;
    return SSB_OK;
}

extern "C" size_t ssb_rolling_workspace_bytes(int64_t band_rows, int64_t width) {
    return 256 + (size_t)std::max<int64_t>(0, band_rows) * (size_t)std::max<int64_t>(0, width) * 4;
}

extern "C" int ssb_rolling_band(const uint16_t *ring, const uint8_t *present, int64_t n_ring,
                                int64_t height, int64_t width, double shear_px, int32_t interp,
                                int64_t lo, int64_t hi, uint16_t *canvas, int16_t *contributor,
                                int64_t canvas_rows, int64_t replaced, void *workspace, size_t workspace_bytes,
                                void *stream) {
    if (n_ring < 1 || height < 1 || width < 1) return fail(SSB_ERR_PARAM, "bad ring shape");
    if (ring == nullptr || present == nullptr || canvas == nullptr || contributor == nullptr)
        return fail(SSB_ERR_PARAM, "ring, present, canvas and contributor must be device buffers");
    if (!(shear_px >= 0.0)) return fail(SSB_ERR_PARAM, "shear_px must be >= 0");
    if (interp != SSB_INTERP_NEAREST && interp != SSB_INTERP_LINEAR)
        return fail(SSB_ERR_PARAM, "interp must be nearest or linear");
    if (lo < 0 || hi >= canvas_rows) return fail(SSB_ERR_CAPACITY, "band %lld..%lld outside %lld-row canvas",
                                                (long long)lo, (long long)hi, (long long)canvas_rows);
    if (hi < lo) return SSB_OK;
    if (replaced >= n_ring || n_ring > 32767) return fail(SSB_ERR_PARAM, "ring index out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t total = (hi - lo + 1) * width;
    if (replaced < 0) {
        if (interp == SSB_INTERP_NEAREST)
            rolling_full_kernel<SSB_INTERP_NEAREST><<<grid_for(total, 256), 256, 0, st>>>(
                ring, present, n_ring, height, width, shear_px, lo, hi, canvas, contributor);
        else
            rolling_full_kernel<SSB_INTERP_LINEAR><<<grid_for(total, 256), 256, 0, st>>>(
                ring, present, n_ring, height, width, shear_px, lo, hi, canvas, contributor);
        count_launches(1);
        return check_launch("rolling_full_kernel");
    }
    if (total > (int64_t)UINT32_MAX) return fail(SSB_ERR_CAPACITY, "band too large");
    if (workspace == nullptr || workspace_bytes < ssb_rolling_workspace_bytes(hi - lo + 1, width))
        return fail(SSB_ERR_CAPACITY, "rolling workspace too small: need %zu bytes",
                    ssb_rolling_workspace_bytes(hi - lo + 1, width));
    uint32_t *count = static_cast<uint32_t *>(workspace);
    uint32_t *list = reinterpret_cast<uint32_t *>(static_cast<char *>(workspace) + 256);
    cudaMemsetAsync(count, 0, 4, st);
    const int remax_blocks = num_sms() * 8;
    if (interp == SSB_INTERP_NEAREST) {
        rolling_incr_kernel<SSB_INTERP_NEAREST><<<grid_for(total, 256), 256, 0, st>>>(
            ring, present, n_ring, height, width, shear_px, lo, hi, canvas, contributor, (int32_t)replaced, list,
            count);
        rolling_remax_kernel<SSB_INTERP_NEAREST><<<remax_blocks, 256, 0, st>>>(
            ring, present, n_ring, height, width, shear_px, lo, canvas, contributor, list, count);
    } else {
        rolling_incr_kernel<SSB_INTERP_LINEAR><<<grid_for(total, 256), 256, 0, st>>>(
            ring, present, n_ring, height, width, shear_px, lo, hi, canvas, contributor, (int32_t)replaced, list,
            count);
        rolling_remax_kernel<SSB_INTERP_LINEAR><<<remax_blocks, 256, 0, st>>>(
            ring, present, n_ring, height, width, shear_px, lo, canvas, contributor, list, count);
    }
    count_launches(2);
    return check_launch("rolling_incr_kernel / rolling_remax_kernel");
}

extern "C" int ssb_warp_rows(const uint16_t *proj, int64_t rows, int64_t cols, double warp_scale,
                             uint16_t *out, int64_t out_rows, void *stream) {
    if (!(warp_scale > 0.0)) return fail(SSB_ERR_PARAM, "warp_scale must be > 0, got %g", warp_scale);
    if (rows < 1 || cols < 0 || out_rows < 1) return fail(SSB_ERR_PARAM, "bad warp shape");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (warp_scale == 1.0) {
        if (out_rows != rows) return fail(SSB_ERR_PARAM, "identity warp must keep the row count");
        cudaMemcpyAsync(out, proj, (size_t)rows * cols * sizeof(uint16_t), cudaMemcpyDeviceToDevice, st);
        return check_launch("ssb_warp_rows(copy)");
    }
    const int64_t total = out_rows * cols;
    if (total == 0) return SSB_OK;
    warp_rows_kernel<<<grid_for(total, 256), 256, 0, st>>>(proj, rows, cols, warp_scale, out, out_rows);
    count_launches(1);
    return check_launch("warp_rows_kernel");
}

extern "C" int ssb_combine(const void *src, void *dst, int64_t count, int32_t reduce, int32_t elem_bits,
                           void *stream) {
    if (count < 0) return fail(SSB_ERR_PARAM, "negative count");
    if (count == 0) return SSB_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (elem_bits == 16 && reduce == SSB_REDUCE_MAX)
        combine_kernel<uint16_t, true><<<grid_for(count, 256), 256, 0, st>>>(
            static_cast<const uint16_t *>(src), static_cast<uint16_t *>(dst), count);
    else if (elem_bits == 32 && reduce == SSB_REDUCE_MAX)
        combine_kernel<uint32_t, true><<<grid_for(count, 256), 256, 0, st>>>(
            static_cast<const uint32_t *>(src), static_cast<uint32_t *>(dst), count);
    else if (elem_bits == 32 && reduce == SSB_REDUCE_SUM)
        combine_kernel<uint32_t, false><<<grid_for(count, 256), 256, 0, st>>>(
            static_cast<const uint32_t *>(src), static_cast<uint32_t *>(dst), count);
    else
        return fail(SSB_ERR_PARAM, "combine supports u16 max, u32 max, u32 sum");
    count_launches(1);
    return check_launch("combine_kernel");
}
