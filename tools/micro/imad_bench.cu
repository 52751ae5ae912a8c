// Microbenchmark: IMAD.WIDE.U32 / IMAD / IADD3 throughput on sm_100a (independent chains).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void wide_chains(uint64_t* out, int iters, uint32_t m) {
    uint64_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = (uint64_t)(uint32_t)a[k] * m + a[k];
    }
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}

__global__ void imad_chains(uint32_t* out, int iters, uint32_t m) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = a[k] * m + (uint32_t)k;
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}

__global__ void hi_chains(uint32_t* out, int iters, uint32_t m) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
#pragma unroll 8
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __umulhi(a[k], m) + a[k];
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}

int main() {
    const int blocks = 148 * 4, threads = 512, iters = 8192;
    void* out;
    cudaMalloc(&out, blocks * threads * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const double ops = 8.0 * iters * blocks * threads;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a); wide_chains<<<blocks, threads>>>((uint64_t*)out, iters, 2654435761u); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("IMAD.WIDE.U32+add64: %.3f ms  %.1f /clk/SM @1.9GHz\n", ms, ops / (ms * 1e-3) / 148 / 1.9e9);
        cudaEventRecord(a); imad_chains<<<blocks, threads>>>((uint32_t*)out, iters, 2654435761u); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("IMAD: %.3f ms  %.1f /clk/SM @1.9GHz\n", ms, ops / (ms * 1e-3) / 148 / 1.9e9);
        cudaEventRecord(a); hi_chains<<<blocks, threads>>>((uint32_t*)out, iters, 2654435761u); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("IMAD.HI+add: %.3f ms  %.1f /clk/SM @1.9GHz\n", ms, ops / (ms * 1e-3) / 148 / 1.9e9);
    }
    return 0;
}
