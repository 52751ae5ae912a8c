// Microbenchmark: FP64 vs FP32 pipe throughput on sm_100a (independent DFMA / FFMA chains).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_chains(T* out, int iters, T c) {
    T a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
        a0 = a0 * c + c; a1 = a1 * c + c; a2 = a2 * c + c; a3 = a3 * c + c;
        a4 = a4 * c + c; a5 = a5 * c + c; a6 = a6 * c + c; a7 = a7 * c + c;
    }
    out[threadIdx.x + blockIdx.x * blockDim.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
    const int blocks = 148 * 4, threads = 512, iters = 8192;
    void* out;
    cudaMalloc(&out, blocks * threads * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    for (int rep = 0; rep < 3; ++rep) {
        float ms;
        double ops = 8.0 * iters * blocks * threads;
        cudaEventRecord(a); fma_chains<double><<<blocks, threads>>>((double*)out, iters, 0.999); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("DFMA: %.3f ms  %.2f TFMA/s  %.1f /clk/SM @1.9GHz\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.9e9);
        cudaEventRecord(a); fma_chains<float><<<blocks, threads>>>((float*)out, iters, 0.999f); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("FFMA: %.3f ms  %.2f TFMA/s  %.1f /clk/SM @1.9GHz\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / 148 / 1.9e9);
    }
    printf("clock rate attr %d kHz\n", clk_khz);
    return 0;
}
