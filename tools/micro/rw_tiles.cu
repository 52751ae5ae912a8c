// Microbenchmark: does the deskew's access shape cost DRAM efficiency?  Same bytes as the
// headline (read 4.29 GB, write 5.22 GB), two shapes:
//   linear : grid-stride 16-byte accesses over flat arrays
//   tiles  : items of 60 rows x 512 B (rows 4 KB apart), one warp per 4 rows, like the kernel
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void stcs(uint4* p, uint4 o) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w) : "memory");
}

// rows of 256 uint4 (4 KB); tile = 60 rows x 32 uint4; read rows_r rows, write rows_w rows
__global__ void tiles(const uint4* __restrict__ src, uint4* __restrict__ dst, int rows_r, int rows_w) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_w = (rows_w + 59) / 60 * 8;
    uint32_t acc = 0;
    for (int t = blockIdx.x; t < tiles_w; t += gridDim.x) {
        const int rb = (t / 8) * 60, xs = (t % 8) * 32;
        for (int k = 0; k < 4; ++k) {
            const int r = rb + warp * 4 + k;
            if (warp < 15) {
                // read ~0.82 of the rows (4.29 / 5.22)
                const long rr = (long)r * 4294967296l / 5224005632l;
                if (rr < rows_r && (r * 4294967296l) / 5224005632l != ((long)(r - 1) * 4294967296l) / 5224005632l) {
                    const uint4 v = ldnc(src + rr * 256 + xs + lane);
                    acc ^= v.x ^ v.w;
                }
                if (r < rows_w) stcs(dst + (long)r * 256 + xs + lane, make_uint4(acc, r, 0, 0));
            }
        }
    }
}

__global__ void linear(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t nr, size_t nw) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += stride) {
        const size_t j = i * 4294967296ull / 5224005632ull;
        if (j < nr && (i == 0 || (i - 1) * 4294967296ull / 5224005632ull != j)) {
            const uint4 v = ldnc(src + j);
            acc ^= v.x ^ v.w;
        }
        stcs(dst + i, make_uint4(acc, (uint32_t)i, 0, 0));
    }
}

int main() {
    const size_t rb = 4294967296ull, wb = 5224005632ull;
    uint4 *src, *dst;
    cudaMalloc(&src, rb); cudaMalloc(&dst, wb);
    cudaMemset(src, 1, rb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int cps : {2, 4}) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            tiles<<<148 * cps, 512>>>(src, dst, (int)(rb / 4096), (int)(wb / 4096));
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        }
        printf("tiles  %d CTA/SM: %.3f ms  %.0f GB/s\n", cps, ms, (rb + wb) / (ms * 1e-3) / 1e9);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            linear<<<148 * cps, 512>>>(src, dst, rb / 16, wb / 16);
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        }
        printf("linear %d CTA/SM: %.3f ms  %.0f GB/s\n", cps, ms, (rb + wb) / (ms * 1e-3) / 1e9);
    }
    return 0;
}
