// Shared device helpers for libssb: exact fp64 index math and the bit-exact
// per-voxel arithmetic of the reference's numpy expressions.
//
// Bit-exactness rules:
//  * every product / sum is a separately rounded IEEE op (__dmul_rn/__dadd_rn/
//    __dsub_rn never contract into FMA), exactly like numpy element-wise float64;
//  * uint16 -> double uses the 2^52 magic (exact, one DADD instead of a slow
//    I2F.F64 conversion);
//  * rint (half to even) uses the 1.5*2^52 magic: fl(v + 1.5*2^52) rounds v to
//    the nearest integer with ties to even, identical to np.rint for |v| < 2^51.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ssb.h"

#ifndef SSB_STORE_WB
#define SSB_STORE_WB 0
#endif

namespace ssb {

constexpr double kEps = 1e-9;                      // ss/geometry.py:39
constexpr double kTwo52 = 4503599627370496.0;      // 2^52
constexpr double kRintMagic = 6755399441055744.0;  // 1.5 * 2^52

__device__ __forceinline__ double u16_to_f64(uint32_t v16) {
    return __dsub_rn(__hiloint2double(0x43300000, (int)v16), kTwo52);
}

__device__ __forceinline__ uint32_t rint_to_u16(double v) {
    return (uint32_t)__double2loint(__dadd_rn(v, kRintMagic)) & 0xFFFFu;
}

// Canvas span of global slice gi (ss/geometry.py:236-255, ss/pipeline.py:274-281).
__device__ __forceinline__ void slice_span(int64_t gi, double s, int64_t h, int interp,
                                           int64_t &lo, int64_t &hi, double &off) {
    off = __dmul_rn((double)gi, s);
    if (interp == SSB_INTERP_NEAREST) {
        lo = (int64_t)floor(__dadd_rn(off, 0.5));
        hi = lo + h - 1;
    } else {
        lo = (int64_t)ceil(__dsub_rn(off, kEps));
        // Python: off + H - 1 + eps, evaluated left to right
        hi = (int64_t)floor(__dadd_rn(__dsub_rn(__dadd_rn(off, (double)h), 1.0), kEps));
    }
}

// Per-canvas-row sampling parameters (amortised over all columns of the row).
struct RowParam {
    int32_t j0;   // first frame row read (or the copied row)
    int32_t j1;   // second frame row read
    double c0;    // canvas: 1-f        npinterp: t = x - xp[j]
    double c1;    // canvas: f          npinterp: dx = xp[j+1] - xp[j]
    int32_t kind; // 0: outside span (value 0); 1: copy row j0; 2: lerp; 3: lerp with dx == 1
};

// Row u of global slice gi (already known to be inside [lo, hi]).
// canvas:   ss/pipeline.py:229-236
// npinterp: ss/phantom.py:396-400 via numpy arr_interp
template <int INTERP, int FORMULA>
__device__ __forceinline__ RowParam row_param(int64_t u, int64_t lo, double off, int64_t h) {
    RowParam rp;
    rp.c0 = 0.0;
    rp.c1 = 1.0;
    if (INTERP == SSB_INTERP_NEAREST) {
        rp.kind = 1;
        rp.j0 = rp.j1 = (int32_t)(u - lo);
        return rp;
    }
    if (FORMULA == SSB_FORMULA_CANVAS) {
        const double j = __dsub_rn((double)u, off);
        int64_t j0 = (int64_t)floor(j);
        j0 = j0 < 0 ? 0 : (j0 > h - 1 ? h - 1 : j0);
        const int64_t j1 = j0 + 1 < h - 1 ? j0 + 1 : h - 1;
        const double f = __dsub_rn(j, (double)j0);
        rp.j0 = (int32_t)j0;
        rp.j1 = (int32_t)j1;
        rp.c0 = __dsub_rn(1.0, f);
        rp.c1 = f;
        rp.kind = 2;
        return rp;
    }
    // np.interp(u, xp = off + arange(h), fp = column)
    const double x = (double)u;
    rp.kind = 1;
    if (h == 1) {
        rp.j0 = rp.j1 = 0;
        return rp;
    }
    int64_t k = (int64_t)floor(__dsub_rn(x, off));
    k = k < -1 ? -1 : (k > h - 1 ? h - 1 : k);
    while (k + 1 <= h - 1 && __dadd_rn(off, (double)(k + 1)) <= x) ++k;
    while (k >= 0 && __dadd_rn(off, (double)k) > x) --k;
    const double xp_last = __dadd_rn(off, (double)(h - 1));
    if (k < 0) { rp.j0 = rp.j1 = 0; return rp; }                       // left value fp[0]
    if (x > xp_last || k == h - 1) { rp.j0 = rp.j1 = (int32_t)(h - 1); return rp; }
    const double xk = __dadd_rn(off, (double)k);
    if (xk == x) { rp.j0 = rp.j1 = (int32_t)k; return rp; }             // on a node
    const double xk1 = __dadd_rn(off, (double)(k + 1));
    rp.j0 = (int32_t)k;
    rp.j1 = (int32_t)(k + 1);
    rp.c0 = __dsub_rn(x, xk);
    rp.c1 = __dsub_rn(xk1, xk);
    rp.kind = rp.c1 == 1.0 ? 3 : 2;
    return rp;
}

// One voxel from the two frame samples a, b (uint16 held in uint32).
template <int FORMULA>
__device__ __forceinline__ uint32_t lerp_voxel(uint32_t a, uint32_t b, const RowParam &rp) {
    const double da = u16_to_f64(a);
    const double db = u16_to_f64(b);
    if (FORMULA == SSB_FORMULA_CANVAS) {
        // (1.0 - f) * a + f * b, each op rounded (numpy), then rint
        return rint_to_u16(__dadd_rn(__dmul_rn(rp.c0, da), __dmul_rn(rp.c1, db)));
    } else {
        // slope = (fp[j+1]-fp[j]) / dx ; v = slope * t + fp[j]
        const double d = __dsub_rn(db, da);
        const double slope = rp.kind == 3 ? d : __ddiv_rn(d, rp.c1);
        return rint_to_u16(__dadd_rn(__dmul_rn(slope, rp.c0), da));
    }
}

// Eight packed voxels (uint4 = 8 x uint16) of one canvas row.
template <int FORMULA>
__device__ __forceinline__ uint4 lerp8(const uint4 a, const uint4 b, const RowParam &rp) {
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
    const uint32_t bw[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t lo = lerp_voxel<FORMULA>(aw[q] & 0xFFFFu, bw[q] & 0xFFFFu, rp);
        const uint32_t hi = lerp_voxel<FORMULA>(aw[q] >> 16, bw[q] >> 16, rp);
        o[q] = lo | (hi << 16);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

__device__ __forceinline__ uint32_t max_u16x2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }

__device__ __forceinline__ uint4 max_u16x8(uint4 a, uint4 b) {
    return make_uint4(__vmaxu2(a.x, b.x), __vmaxu2(a.y, b.y), __vmaxu2(a.z, b.z), __vmaxu2(a.w, b.w));
}

__device__ __forceinline__ uint32_t hmax_u16x8(uint4 v) {
    const uint32_t m = __vmaxu2(__vmaxu2(v.x, v.y), __vmaxu2(v.z, v.w));
    return max(m & 0xFFFFu, m >> 16);
}

__device__ __forceinline__ uint32_t hsum_u16x8(uint4 v) {
    return (v.x & 0xFFFFu) + (v.x >> 16) + (v.y & 0xFFFFu) + (v.y >> 16) + (v.z & 0xFFFFu) +
           (v.z >> 16) + (v.w & 0xFFFFu) + (v.w >> 16);
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void stg_cs_v4(void *p, uint4 v) {
#if SSB_STORE_WB  // A/B knob: default write-back stores instead of streaming (.cs)
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
    return;
#endif
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

}  // namespace ssb
