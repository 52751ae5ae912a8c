#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, int c0, int c1, int use_g, uint16_t* out) {
  __shared__ __align__(128) uint16_t box[8][256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(8*256*2));
    const CUtensorMap* mp = use_g ? gm : &m;
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(sa(&box[0][0])), "l"((uint64_t)mp), "r"(c0), "r"(c1), "r"(sa(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8*256; i += blockDim.x) out[i] = box[i/256][i%256];
}
int main(int argc, char** argv) {
  int W = argc > 1 ? atoi(argv[1]) : 2044, H = 64, P = 2; int off = argc > 2 ? atoi(argv[2]) : 0;
  while ((P * 2 * W) % 16) P *= 2; if (argc > 3) P = atoi(argv[3]);
  size_t n = (size_t)W * H + 64;
  uint16_t* d; cudaMalloc(&d, n * 2);
  uint16_t* h = (uint16_t*)malloc(n * 2); for (size_t i = 0; i < n; ++i) h[i] = (uint16_t)i;
  cudaMemcpy(d, h, n * 2, cudaMemcpyHostToDevice);
  void* fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fnp, 12000, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  uint16_t* raw = d + off;
  int r = argc > 4 ? atoi(argv[4]) : 1;
  uintptr_t a = (uintptr_t)raw + r * W * 2, a16 = a & ~uintptr_t(15);
  int c = (int)((a - a16) / 2);
  CUtensorMap m; memset(&m, 0, sizeof m);
  cuuint64_t dims[2] = {(cuuint64_t)(W + c), (cuuint64_t)((H - r + P - 1) / P)};
  cuuint64_t str[1] = {(cuuint64_t)(P * W * 2)};
  cuuint32_t box[2] = {256, 8}, es[2] = {1, 1};
  CUresult e = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)a16, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("W=%d P=%d c=%d encode=%d\n", W, P, c, (int)e);
  CUtensorMap* gm; cudaMalloc(&gm, sizeof m); cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice);
  uint16_t* out; cudaMalloc(&out, 8 * 256 * 2);
  for (int use_g = 0; use_g < 2; ++use_g) {
    k<<<1, 128>>>(m, gm, c + 0, 1, use_g, out);
    cudaError_t err = cudaDeviceSynchronize();
    uint16_t ho[8 * 256]; cudaMemcpy(ho, out, sizeof ho, cudaMemcpyDeviceToHost);
    // row 1 of the map = global row r + P*1; col 0 = pixel 0
    int R = r + P * 1; printf("use_g=%d err=%s got %d want %d\n", use_g, cudaGetErrorString(err), ho[0], (int)(uint16_t)(off + R * W));
    if (err) return 1;
  }
}
