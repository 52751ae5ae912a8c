// Micro-benchmark: issue throughput of the instructions the fp32 bracket lerp is built from
// (FFMA, FFMA2, FADD2, PRMT, LOP3, VIMNMX.U16x2, I2FP.F32.U32, IMAD), alone and mixed, on sm_100a.
// 8 independent chains per thread, 2048 threads per SM; prints warp-instructions / clk / SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
#define N 8
template <int OP>
__global__ void k(uint32_t *out, int iters, uint32_t seed) {
    uint32_t r[N];
    u64 q[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        r[i] = seed * (threadIdx.x + i + 1);
        q[i] = ((u64)r[i] << 32) | (r[i] ^ 0x3f800000u);
    }
    const u64 c2 = 0x3f8000003f800001ull;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(0x3f800001u), "r"(r[(i + 1) % N]));
            if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(q[i]) : "l"(c2), "l"(q[(i + 1) % N]));
            if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(q[i]) : "l"(q[(i + 1) % N]));
            if (OP == 3) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[i]) : "r"(r[(i + 1) % N]));
            if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0xfe;" : "+r"(r[i]) : "r"(r[(i + 1) % N]), "r"(r[(i + 2) % N]));
            if (OP == 5) asm volatile("vmax2.u32.u32.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(r[(i + 1) % N]), "r"(0));
            if (OP == 6) {
                float f;
                asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(r[i]));
                r[i] ^= __float_as_uint(f);
            }
            if (OP == 7) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(r[(i + 1) % N]), "r"(0x1234u));
            if (OP == 8) {  // mix: 1 FFMA2 + 1 PRMT
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(q[i]) : "l"(c2), "l"(q[(i + 1) % N]));
                asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[i]) : "r"(r[(i + 1) % N]));
            }
            if (OP == 9) {  // mix: 1 FFMA + 1 PRMT
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(0x3f800001u), "r"(r[(i + 1) % N]));
                asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[(i + 3) % N]) : "r"(r[(i + 1) % N]));
            }
            if (OP == 11) r[i] = __vmaxu2(r[i], r[(i + 1) % N]);
            if (OP == 12) {  // I2FP + FADD
                float f;
                asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(r[i]));
                asm volatile("add.rn.f32 %0, %0, %1;" : "+r"(r[(i + 3) % N]) : "f"(f));
            }
            if (OP == 13) {  // FFMA2 + LOP3 + PRMT
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(q[i]) : "l"(c2), "l"(q[(i + 1) % N]));
                asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[i]) : "r"(r[(i + 1) % N]));
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xfe;" : "+r"(r[(i + 4) % N]) : "r"(r[(i + 1) % N]), "r"(r[(i + 2) % N]));
            }
            if (OP == 14) {  // IMAD + PRMT
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(r[(i + 1) % N]), "r"(0x1234u));
                asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[(i + 4) % N]) : "r"(r[(i + 1) % N]));
            }
            if (OP == 15) {  // FFMA2 + FFMA2 + PRMT + PRMT (pipes balanced)
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(q[i]) : "l"(c2), "l"(q[(i + 1) % N]));
                asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(r[i]) : "r"(r[(i + 1) % N]));
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(q[(i + 4) % N]) : "l"(q[(i + 5) % N]));
                asm volatile("prmt.b32 %0, %0, %1, 0x5432;" : "+r"(r[(i + 4) % N]) : "r"(r[(i + 5) % N]));
            }
            if (OP == 10) {  // cvt.rn.f32.u16 (half-register source)
                float f;
                asm volatile("cvt.rn.f32.u16 %0, %1;" : "=f"(f) : "h"((unsigned short)r[i]));
                r[i] ^= __float_as_uint(f);
            }
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) acc ^= r[i] ^ (uint32_t)q[i] ^ (uint32_t)(q[i] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
void run(const char *name, int per_iter) {
    const int sms = 148, blocks = sms * 8, threads = 256, iters = 4096;
    uint32_t *out;
    cudaMalloc(&out, blocks * threads * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<OP><<<blocks, threads>>>(out, 16, 3);
    cudaEventRecord(a);
    k<OP><<<blocks, threads>>>(out, iters, 3);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warp_ins = (double)blocks * threads / 32 * iters * N * per_iter;
    printf("%-28s %.3f ms  %.2f warp-instr/clk/SM (at %.0f MHz)\n", name, ms, warp_ins / (ms * 1e-3) / (clk * 1e3) / sms,
           clk / 1e3);
    cudaFree(out);
}

int main() {
    run<0>("FFMA (3 regs)", 1);
    run<1>("FFMA2", 1);
    run<2>("FADD2", 1);
    run<3>("PRMT", 1);
    run<4>("LOP3", 1);
    run<5>("VIMNMX.U16x2", 1);
    run<6>("I2FP.F32.U32 + LOP3", 2);
    run<7>("IMAD", 1);
    run<8>("FFMA2 + PRMT", 2);
    run<9>("FFMA + PRMT", 2);
    run<10>("cvt.f32.u16 + LOP3", 2);
    run<11>("VIMNMX.U16x2 (__vmaxu2)", 1);
    run<12>("I2FP.F32.U32 + FADD", 2);
    run<13>("FFMA2 + PRMT + LOP3", 3);
    run<14>("IMAD + PRMT", 2);
    run<15>("FFMA2+FADD2+2 PRMT", 4);
    return 0;
}
