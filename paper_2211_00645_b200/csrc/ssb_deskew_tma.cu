// Persistent deskew kernel: host side (mode choice, tensor maps, scheduling, scratch, finalize); the
// kernel templates live in ssb_tma_kernel.cuh and are instantiated in ssb_tma_inst_*.cu.
#include "ssb_tma_kernel.cuh"

namespace ssb {
namespace tma_path {

extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 16>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 16>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_NPINTERP, 16>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 40>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 104>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 40>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 104>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 36>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 34>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 36>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 34>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 8>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 4>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 2>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 8>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 4>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
extern template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 2>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);

// u32 reduction scratch -> uint16 projections (max mode); dst = max(dst, src) when accumulating.
struct U16Seg {
    const uint32_t *src;
    uint16_t *dst;
    int64_t count;
    int32_t accumulate;
};

__device__ __forceinline__ void finalize_seg(const U16Seg &sg, int64_t tid, int64_t nthreads) {
    // 4 elements per step: one 16-byte load of u32, one 8-byte store of u16 (counts are multiples
    // of 8 on this path because W % 8 == 0; a scalar tail covers the rest)
    const int64_t n4 = (reinterpret_cast<uintptr_t>(sg.dst) & 7u) ? 0 : sg.count / 4;
    const uint4 *src = reinterpret_cast<const uint4 *>(sg.src);
    uint2 *dst = reinterpret_cast<uint2 *>(sg.dst);
    for (int64_t i = tid; i < n4; i += nthreads) {
        const uint4 v = src[i];
        uint32_t lo = v.x | (v.y << 16), hi = v.z | (v.w << 16);
        if (sg.accumulate) {
            const uint2 o = dst[i];
            lo = __vmaxu2(lo, o.x);
            hi = __vmaxu2(hi, o.y);
        }
        dst[i] = make_uint2(lo, hi);
    }
    for (int64_t i = 4 * n4 + tid; i < sg.count; i += nthreads) {
        uint32_t v = sg.src[i];
        if (sg.accumulate) v = max(v, (uint32_t)sg.dst[i]);
        sg.dst[i] = (uint16_t)v;
    }
}

__global__ void finalize_u16_kernel(U16Seg s0, U16Seg s1, U16Seg s2) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    finalize_seg(s0, tid, nthreads);
    finalize_seg(s1, tid, nthreads);
    finalize_seg(s2, tid, nthreads);
}

template <int INTERP, int FORMULA>
int launch_ac(int ac, bool mx, bool tall, bool side, const TmapSet &map, const Params &prm, int grid,
              cudaStream_t st) {
    if (ac == 16) return launch_variant<INTERP, FORMULA, 16>(mx, tall, side, map, prm, grid, st);
    if constexpr (FORMULA == SSB_FORMULA_CANVAS) {  // row-copy mode: canvas formula (ProjectionCanvas) only
        if (ac == 8) return launch_variant<INTERP, FORMULA, 8>(mx, false, side, map, prm, grid, st);
        if (ac == 4) return launch_variant<INTERP, FORMULA, 4>(mx, false, side, map, prm, grid, st);
        if (ac == 2) return launch_variant<INTERP, FORMULA, 2>(mx, false, side, map, prm, grid, st);
        // row-class TMA (AC = 32 + row alignment)
        if (ac == 40) return launch_variant<INTERP, FORMULA, 40>(mx, false, side, map, prm, grid, st);
        if (ac == 36) return launch_variant<INTERP, FORMULA, 36>(mx, false, side, map, prm, grid, st);
        if (ac == 34) return launch_variant<INTERP, FORMULA, 34>(mx, false, side, map, prm, grid, st);
        if (ac == 104) return launch_variant<INTERP, FORMULA, 104>(mx, false, side, map, prm, grid, st);
    }
    return fail(SSB_ERR_PARAM, "no persistent kernel for access class %d", ac);
}

}  // namespace tma_path

bool tma_eligible(const ssb_deskew_desc &d, const uint16_t *raw, const void *vol, const void *xy) {
    if (d.width % 8 != 0 || !aligned16(raw) || !aligned16(vol) || !aligned16(xy)) return false;
    if (row_stride_of(d) % 8 != 0 || frame_stride_of(d) % 8 != 0) return false;  // TMA: 16-byte strides
    if (d.n > INT32_MAX || d.height > INT32_MAX || d.width > INT32_MAX) return false;
    return tma_path::encode_fn() != nullptr;
}

int persistent_access_class(const ssb_deskew_desc &d, const uint16_t *raw, const void *vol, const void *xy) {
    if (tma_eligible(d, raw, vol, xy)) return 16;
    if (d.formula != SSB_FORMULA_CANVAS || getenv("SSB_DISABLE_ROWCOPY") != nullptr) return 0;
    if (d.n > INT32_MAX || d.height > INT32_MAX || d.width > INT32_MAX) return 0;
    if ((reinterpret_cast<uintptr_t>(xy) & 3u) != 0) return 0;  // u16 XY is written by the finalize pass
    // widest access every frame row (loads from the row slots) and every volume row (stores) allows
    const uintptr_t r = reinterpret_cast<uintptr_t>(raw), v = reinterpret_cast<uintptr_t>(vol);
    const int64_t rs = row_stride_of(d), fs = frame_stride_of(d), w = d.width;
    auto fits = [&](int ac) {
        const int64_t e = ac / 2;
        return (r % ac) == 0 && rs % e == 0 && fs % e == 0 && (vol == nullptr || ((v % ac) == 0 && w % e == 0));
    };
    const int ac = fits(8) ? 8 : fits(4) ? 4 : 2;
    const char *force = getenv("SSB_FORCE_AC");  // A/B and debugging: a narrower class than allowed
    return force && atoi(force) < ac && (atoi(force) == 4 || atoi(force) == 2) ? atoi(force) : ac;
}

namespace {
constexpr size_t kCounterBytes = 256;
size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
int64_t env_i64(const char *name, int64_t dflt) {
    const char *v = getenv(name);
    return v ? atoll(v) : dflt;
}
}  // namespace

size_t tma_workspace_bytes(const ssb_deskew_desc &d, int64_t batch) {
    // u32 reduction scratch for max mode (sum mode reduces straight into the caller's u32 outputs)
    size_t b = kCounterBytes;
    if (d.reduce == SSB_REDUCE_MAX)
        b += align256((size_t)batch * d.u_count * d.width * 4) + align256((size_t)batch * d.n * d.width * 4) +
             align256((size_t)batch * d.n * d.u_count * 4);
    return b;
}

int launch_deskew_tma(const ssb_deskew_desc &d, const uint16_t *raw, uint16_t *vol, void *xy, void *xz, void *yz,
                      void *workspace, size_t workspace_bytes, cudaStream_t st, int ac, int64_t batch) {
    using namespace tma_path;
    if (batch < 1 || (batch > 1 && ac != 16)) return fail(SSB_ERR_PARAM, "batched launches need TMA-mode stacks");
    if (batch * d.n > INT32_MAX) return fail(SSB_ERR_CAPACITY, "batch of %lld frames too large", (long long)(batch * d.n));
    if (workspace == nullptr || workspace_bytes < tma_workspace_bytes(d, batch))
        return fail(SSB_ERR_CAPACITY, "workspace too small: need %zu bytes, got %zu", tma_workspace_bytes(d, batch),
                    workspace_bytes);
    TmapSet maps;
    memset(&maps, 0, sizeof maps);
    CUtensorMap &map = maps.m[0];
    // a batch is one frame axis of batch * n frames (stacks back to back, frame stride apart)
    const cuuint64_t dims[3] = {(cuuint64_t)d.width, (cuuint64_t)d.height, (cuuint64_t)(batch * d.n)};
    const cuuint64_t strides[2] = {(cuuint64_t)row_stride_of(d) * 2, (cuuint64_t)frame_stride_of(d) * 2};
    const bool mx = d.reduce == SSB_REDUCE_MAX;
    const bool side = xz != nullptr || yz != nullptr;
    // 8-row tiles (A/B knob): since the fp32 lerp and the volume-free instantiations, 4-row tiles with
    // their deeper ring are faster for every projection-only variant too (3 MIPs 1.174 vs 1.202 ms,
    // XY+XZ 1.112 vs 1.166, XY+YZ 1.062 vs 1.122; profiles/r02_v4_tall_ab.txt)
    const int64_t tall_env = env_i64("SSB_TALL_TILES", 0);  // 0 never, 1 projection-only, 2 always
    const bool tall = (vol == nullptr || tall_env == 2) && tall_env != 0 && mx && side && ac == 16;
    const int kTU = tall ? Cfg<8>::kTU : Cfg<4>::kTU;
    const int slack = d.interp == SSB_INTERP_NEAREST ? box_slack<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS>()
                      : d.formula == SSB_FORMULA_CANVAS ? box_slack<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS>()
                                                        : box_slack<SSB_INTERP_LINEAR, SSB_FORMULA_NPINTERP>();
    const int rows = kTU + 2 * slack;
    const cuuint32_t box[3] = {(cuuint32_t)kTX, (cuuint32_t)rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (ac == 16) {  // row-copy mode (ac < 16) addresses the frames directly
        const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<uint16_t *>(raw), dims,
                                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       SSB_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SSB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
    // Rows that are not 16-byte aligned (canvas lerp, one stack, frames 16 bytes apart): one tensor map per
    // row class (see rt_mode) instead of the row-copy modes.  P = 16 / gcd(2 * row_stride, 16) classes.
    int32_t rt_P = 0, rt_B = 0, rt_B31 = 0;
    uint32_t rt_d0 = 0;
    {
        const int64_t rs = row_stride_of(d), fs = frame_stride_of(d);
        const int64_t rs16 = (2 * rs) % 16;
        const int P = rs16 == 0 ? 1 : 16 / (int)std::gcd<int64_t>(rs16, 16);
        if (ac < 16 && d.formula == SSB_FORMULA_CANVAS && batch == 1 &&
            (2 * fs) % 16 == 0 && d.height >= P && P <= 16 / ac && encode_fn() != nullptr &&
            env_i64("SSB_DISABLE_RT", 0) == 0) {
            const uintptr_t r0 = reinterpret_cast<uintptr_t>(raw);
            const int B = rt_class_rows(rows, P);
            bool ok = true;
            for (int c = 0; c < P && ok; ++c) {
                const uintptr_t a = r0 + 2u * (uintptr_t)(c * rs), dlt = a & 15u;
                const cuuint64_t cd[3] = {(cuuint64_t)(d.width + (int64_t)dlt / 2),
                                          (cuuint64_t)((d.height - c + P - 1) / P), (cuuint64_t)d.n};
                const cuuint64_t cs[2] = {(cuuint64_t)(2 * P * rs), (cuuint64_t)(2 * fs)};
                const cuuint32_t cb[3] = {(cuuint32_t)kTX, (cuuint32_t)B, 1};
                const cuuint32_t cb31[3] = {16, (cuuint32_t)B, 1};  // lane 31's box (16 columns)
                ok = encode_fn()(&maps.m[c], CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, reinterpret_cast<void *>(a - dlt), cd, cs,
                                 cb, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, SSB_L2_PROMO,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
                     (ac != 8 ||
                      encode_fn()(&maps.m[8 + c], CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, reinterpret_cast<void *>(a - dlt), cd,
                                 cs, cb31, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 SSB_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS);
            }
            if (ok) {
                rt_P = P;
                rt_B = B;
                rt_B31 = (B + 3) / 4 * 4;
                rt_d0 = (uint32_t)(r0 & 15u);
                ac += 32;
                if (ac == 40 && vol == nullptr) ac += 64;  // projection-only, 8-byte rows: lane-31 boxes
            }
        }
    }

    // work items: (u-tile, x-tile, slice chunk); ~kItemsPerCta items per persistent CTA keep the
    // dynamic scheduler's tail short (projections reduce in L2, so chunking costs no partial planes)
    const int sms = num_sms();
    const int64_t UT = std::max<int64_t>(1, (d.u_count + kTU - 1) / kTU);
    const int64_t tw = ac > 16 && ac < 64 ? kTX - 8 : kTX;  // tile width (row-class TMA: 248 unless lane-31 boxes)
    const int64_t XT = std::max<int64_t>(1, (d.width + tw - 1) / tw);
    const int64_t tiles = UT * XT * batch;  // tiles of every stack of the batch
    // phase 1: ~SSB_ITEMS_PER_CTA big items per CTA over the first SSB_BIG_PERCENT % of the
    // slices; phase 2: the rest in ~SSB_TAIL_ITEMS_PER_CTA small items
    auto split = [&](int64_t n_sl, int64_t per_cta, int64_t &S, int64_t &chunk) {
        S = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(n_sl, 1), (per_cta * sms + tiles - 1) / tiles));
        chunk = std::max<int64_t>(1, (n_sl + S - 1) / S);
        S = n_sl > 0 ? (n_sl + chunk - 1) / chunk : 0;
    };
    const int64_t big_pct = std::min<int64_t>(100, std::max<int64_t>(0, env_i64("SSB_BIG_PERCENT", 85)));
    // projection-only: tiles visit only the slices that can touch them (no volume zero fill
    // to write), so the chunking is planned on the longest per-tile slice range
    const bool clip = vol == nullptr && d.shear_px > 0.0 && env_i64("SSB_CLIP_SLICES", 1) != 0;
    const double span_slices = std::ceil((kTU + d.height + 4) / d.shear_px) + 2.0;
    const int64_t n_plan = clip && span_slices < (double)d.n ? (int64_t)span_slices : d.n;
    // small problems (few pipeline stages per SM, e.g. config 1) pay a fixed cost per item
    // (counter fetch, queue hand-off, pipeline fill): at most one item per ~16 stages of an SM's
    // share, and no tail phase below ~64 stages per SM
    const double stages_per_sm = (double)tiles * (double)n_plan / sms;
    const int64_t per1 = std::max<int64_t>(
        1, std::min<int64_t>(env_i64("SSB_ITEMS_PER_CTA", 2), (int64_t)(stages_per_sm / 16.0)));
    const bool tail = stages_per_sm >= 64.0;
    int64_t n1 = tail ? n_plan * big_pct / 100 : n_plan;
    if (n1 < 1) n1 = n_plan;
    int64_t S, chunk, S2, chunk2;
    split(n1, per1, S, chunk);
    split(n_plan - n1, env_i64("SSB_TAIL_ITEMS_PER_CTA", 3), S2, chunk2);
    const int64_t items = tiles * (S + S2);  // = batch * UT * XT * (S + S2), decode() order
    if (items > INT32_MAX / 2) return fail(SSB_ERR_CAPACITY, "too many tiles");

    char *ws = static_cast<char *>(workspace);
    unsigned int *counters = reinterpret_cast<unsigned int *>(ws);
    ws += kCounterBytes;
    const bool acc = (d.flags & SSB_FLAG_XY_ACCUMULATE) != 0;
    const bool xy_u32 = mx && (d.flags & SSB_FLAG_XY_U32) != 0;  // caller's u32 XY accumulator
    // per stack; the scratch / outputs of a batch hold `batch` of each back to back
    const size_t s_xy = (size_t)d.u_count * d.width, s_xz = (size_t)d.n * d.width, s_yz = (size_t)d.n * d.u_count;
    const size_t n_xy = s_xy * batch, n_xz = s_xz * batch, n_yz = s_yz * batch;
    uint32_t *xy32 = nullptr, *xz32 = nullptr, *yz32 = nullptr;
    if (mx) {
        xy32 = xy ? (xy_u32 ? static_cast<uint32_t *>(xy) : reinterpret_cast<uint32_t *>(ws)) : nullptr;
        ws += align256(n_xy * 4);
        xz32 = xz ? reinterpret_cast<uint32_t *>(ws) : nullptr;
        ws += align256(n_xz * 4);
        yz32 = yz ? reinterpret_cast<uint32_t *>(ws) : nullptr;
    } else {
        xy32 = static_cast<uint32_t *>(xy);
        xz32 = static_cast<uint32_t *>(xz);
        yz32 = static_cast<uint32_t *>(yz);
    }
    if (mx && !xy_u32) {
        // counter and the u32 scratch are contiguous in the workspace: one memset
        char *end = reinterpret_cast<char *>(counters) + sizeof(unsigned int);
        if (xy32) end = reinterpret_cast<char *>(xy32 + n_xy);
        if (xz32) end = reinterpret_cast<char *>(xz32 + n_xz);
        if (yz32) end = reinterpret_cast<char *>(yz32 + n_yz);
        cudaMemsetAsync(counters, 0, (size_t)(end - reinterpret_cast<char *>(counters)), st);
    } else if (mx) {  // the caller's XY accumulator keeps its contents
        cudaMemsetAsync(counters, 0, sizeof(unsigned int), st);
        if (xz32) cudaMemsetAsync(xz32, 0, n_xz * 4, st);
        if (yz32) cudaMemsetAsync(yz32, 0, n_yz * 4, st);
    } else {
        cudaMemsetAsync(counters, 0, sizeof(unsigned int), st);
        if (xy32 && !acc) cudaMemsetAsync(xy32, 0, n_xy * 4, st);
        if (xz32) cudaMemsetAsync(xz32, 0, n_xz * 4, st);
        if (yz32) cudaMemsetAsync(yz32, 0, n_yz * 4, st);
    }
    if (int rc = check_launch("ssb_deskew scratch reset")) return rc;

    Params prm{};
    prm.vol = vol;
    prm.xy = xy32;
    prm.xz = xz32;
    prm.yz = yz32;
    prm.counters = counters;
    prm.n = d.n;
    prm.h = d.height;
    prm.w = d.width;
    prm.first = d.first_slice;
    prm.u_begin = d.u_begin;
    prm.u_count = d.u_count;
    prm.chunk = chunk;
    prm.n1 = n1;
    prm.chunk2 = chunk2;
    prm.S2 = (int32_t)S2;
    prm.shear = d.shear_px;
    prm.UT = (int32_t)UT;
    prm.XT = (int32_t)XT;
    prm.S = (int32_t)S;
    prm.n_items = (int32_t)items;
    prm.xy_accumulate = acc;
    prm.clip = clip ? 1 : 0;
    prm.big_pct = (int32_t)big_pct;
    prm.raw = raw;
    prm.row_stride = row_stride_of(d);
    prm.frame_stride = frame_stride_of(d);
    prm.batch = (int32_t)batch;
    prm.vol_bstride = (int64_t)d.n * d.u_count * d.width;
    prm.xy_bstride = (int64_t)s_xy;
    prm.xz_bstride = (int64_t)s_xz;
    prm.yz_bstride = (int64_t)s_yz;
    prm.rt_P = rt_P;
    prm.rt_B = rt_B;
    prm.rt_B31 = rt_B31;
    prm.rt_d0 = rt_d0;
    const int grid = (int)std::min<int64_t>(items, sms);

    int rc;
    profile_begin(st);
    // one place decides the instantiation, consistent with the tile height planned above
    if (d.interp == SSB_INTERP_NEAREST)
        rc = launch_ac<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS>(ac, mx, tall, side, maps, prm, grid, st);
    else if (d.formula == SSB_FORMULA_CANVAS)
        rc = launch_ac<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS>(ac, mx, tall, side, maps, prm, grid, st);
    else
        rc = launch_ac<SSB_INTERP_LINEAR, SSB_FORMULA_NPINTERP>(ac, mx, tall, side, maps, prm, grid, st);
    profile_end(st);
    count_launches(1);
    if (rc) return rc;

    if (mx && ((xy32 && !xy_u32) || xz32 || yz32)) {
        U16Seg a{xy32, static_cast<uint16_t *>(xy), (xy32 && !xy_u32) ? (int64_t)n_xy : 0, acc ? 1 : 0};
        U16Seg b{xz32, static_cast<uint16_t *>(xz), xz32 ? (int64_t)n_xz : 0, 0};
        U16Seg c{yz32, static_cast<uint16_t *>(yz), yz32 ? (int64_t)n_yz : 0, 0};
        const int64_t total = (a.count + b.count + c.count) / 4;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sms * 8));
        finalize_u16_kernel<<<blocks, 256, 0, st>>>(a, b, c);
        count_launches(1);
        return check_launch("finalize_u16_kernel");
    }
    return SSB_OK;
}

}  // namespace ssb
