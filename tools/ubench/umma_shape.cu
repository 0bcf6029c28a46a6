// Cycles per tcgen05.mma kind::i8 (SS) for M in {64, 128} and N in {32..256} with the
// certified scan's descriptor walk (16 K-steps; A: LBO 256 / SBO 128 overlapping
// cores, B: LBO 128 / SBO = bsbo).  One CTA per SM, one issuing warp.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o umma_shape umma_shape.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__global__ void __launch_bounds__(128) k(int R, int M, int N, int bsbo, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int t = threadIdx.x;
  for (int i = t; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "r"(256) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  long long t0 = clock64(), t1 = 0;
  if (t < 32) {
    uint64_t da = sdesc(base, 256, 128), db = sdesc(base + 32768, 128, bsbo);
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_base),
                   "l"(da), "l"(db), "r"(idesc), "r"(r));
      da += 512 >> 4; db += 256 >> 4;
      if ((r & 15) == 15) { da -= (16 * 512) >> 4; db -= (16 * 256) >> 4; }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(0) : "memory");
    t1 = clock64();
  }
  __syncthreads();
  if (t == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256) : "memory");
}
int main() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int R = 4096;
  const int shapes[][3] = {{128, 64, 1024}, {128, 128, 1024}, {128, 256, 1024}, {128, 32, 1024},
                           {64, 64, 512}, {64, 128, 512}, {64, 256, 512}, {64, 128, 1024}};
  for (auto& sh : shapes) {
    long long h = 0;
    k<<<nsm, 128, 96 * 1024>>>(64, sh[0], sh[1], sh[2], d);
    k<<<nsm, 128, 96 * 1024>>>(R, sh[0], sh[1], sh[2], d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double macs = (double)sh[0] * sh[1] * 32;
    printf("M=%3d N=%3d (B SBO %4d): %.1f cycles/MMA  %.0f MAC/cycle/SM  %s\n", sh[0], sh[1], sh[2],
           (double)h / R, macs * R / h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
