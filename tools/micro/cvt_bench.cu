// Microbenchmark: uint16 -> double conversion throughput on sm_100a.
//  a) I2F.F64 (native conversion) + DMUL
//  b) 2^52 magic (extract + constant high word) + DFMA
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void conv_native(const uint32_t* in, double* out, int iters, double c) {
    uint32_t w = in[threadIdx.x + blockIdx.x * blockDim.x];
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    #pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        w = w * 1664525u + 1013904223u;
        acc0 = __dadd_rn(acc0, __dmul_rn(c, (double)(w & 0xFFFF)));
        acc1 = __dadd_rn(acc1, __dmul_rn(c, (double)(w >> 16)));
        acc2 = __dadd_rn(acc2, __dmul_rn(c, (double)((w >> 8) & 0xFFFF)));
        acc3 = __dadd_rn(acc3, __dmul_rn(c, (double)((w ^ 0x5555) & 0xFFFF)));
    }
    out[threadIdx.x + blockIdx.x * blockDim.x] = acc0 + acc1 + acc2 + acc3;
}

__device__ __forceinline__ double biased(uint32_t v) { return __hiloint2double(0x43300000, (int)v); }

__global__ void conv_magic(const uint32_t* in, double* out, int iters, double c) {
    uint32_t w = in[threadIdx.x + blockIdx.x * blockDim.x];
    const double n = -c * 4503599627370496.0;
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    #pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        w = w * 1664525u + 1013904223u;
        acc0 = __dadd_rn(acc0, __fma_rn(c, biased(w & 0xFFFF), n));
        acc1 = __dadd_rn(acc1, __fma_rn(c, biased(w >> 16), n));
        acc2 = __dadd_rn(acc2, __fma_rn(c, biased((w >> 8) & 0xFFFF), n));
        acc3 = __dadd_rn(acc3, __fma_rn(c, biased((w ^ 0x5555) & 0xFFFF), n));
    }
    out[threadIdx.x + blockIdx.x * blockDim.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    uint32_t* in; double* out;
    cudaMalloc(&in, blocks * threads * 4); cudaMalloc(&out, blocks * threads * 8);
    cudaMemset(in, 1, blocks * threads * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a); conv_native<<<blocks, threads>>>(in, out, iters, 0.3); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        double conv = 4.0 * iters * blocks * threads;
        printf("native I2F.F64: %.3f ms  %.1f Gconv/s  %.2f conv/clk/SM@1.9GHz\n", ms, conv / ms / 1e6, conv / ms / 1e6 / 148 / 1.9);
        cudaEventRecord(a); conv_magic<<<blocks, threads>>>(in, out, iters, 0.3); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("magic  2^52   : %.3f ms  %.1f Gconv/s  %.2f conv/clk/SM@1.9GHz\n", ms, conv / ms / 1e6, conv / ms / 1e6 / 148 / 1.9);
    }
    return 0;
}
