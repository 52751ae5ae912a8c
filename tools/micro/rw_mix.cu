// Microbenchmark: HBM read+write mix ceiling for the deskew's traffic shape
// (read 4.29 GB, write 5.22 GB per launch), linear addresses, 16-byte accesses.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rw(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t nr, size_t nw) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    const size_t n = nr > nw ? nr : nw;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (i < nr) {
            uint4 v;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        if (i < nw) {
            uint4 o = make_uint4(acc, (uint32_t)i, 0, 0);
            asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dst + i), "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w) : "memory");
        }
    }
}

int main() {
    const size_t rb = 4294967296ull, wb = 5224005632ull;
    uint4 *src, *dst;
    cudaMalloc(&src, rb); cudaMalloc(&dst, wb);
    cudaMemset(src, 1, rb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocks_per_sm : {2, 4, 8}) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            rw<<<148 * blocks_per_sm, 512>>>(src, dst, rb / 16, wb / 16);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("rw mix %d CTAs/SM: %.3f ms  %.0f GB/s\n", blocks_per_sm, ms, (rb + wb) / (ms * 1e-3) / 1e9);
        }
    }
    // pure copy of the same write size for reference
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(dst, src, rb, cudaMemcpyDeviceToDevice);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("cudaMemcpy D2D 4.29 GB: %.3f ms  %.0f GB/s (r+w)\n", ms, 2.0 * rb / (ms * 1e-3) / 1e9);
    }
    return 0;
}
