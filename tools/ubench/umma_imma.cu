// Do tcgen05 kind::i8 MMAs (issued by warp 0) and mma.sync m16n8k32 IMMAs (warps
// 1-15) share the SM's tensor pipe?  Times each stream alone and both together.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o umma_imma umma_imma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__global__ void __launch_bounds__(512) k(int R, int M, int mode, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "r"(128) : "memory");
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
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  const long long t0 = clock64();
  long long tu = 0, ti = 0;
  if (w == 0 && (mode & 1)) {
    uint64_t da = sdesc(base, 256, 128), db = sdesc(base + 40960, 128, 1024);
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
    tu = clock64() - t0;
  }
  if (w > 0 && (mode & 2)) {
    uint32_t a0 = 0x01010101u * t, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = ~a0;
    int d[4][4] = {};
#pragma unroll 1
    for (int r = 0; r < M; ++r) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(d[q][0]), "+r"(d[q][1]), "+r"(d[q][2]), "+r"(d[q][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      a0 += 1;
    }
    int s = 0;
    for (int q = 0; q < 4; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3];
    if (s == 0x7fffffff) out[100] = s;
    ti = clock64() - t0;
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    if (t == 0) out[0] = tu;
    if (t == 32) out[1] = ti;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(128) : "memory");
}
int main() {
  long long* d; cudaMalloc(&d, 8192);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int R = 4096, M = 1024;   // 4096 UMMAs vs 15 warps x 4096 IMMAs
  for (int mode : {1, 2, 3}) {
    long long h[2] = {0, 0};
    k<<<nsm, 512, 96 * 1024>>>(R, M, mode, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<nsm, 512, 96 * 1024>>>(R, M, mode, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): umma stream %lld cyc (%.1f cyc/umma), imma stream %lld cyc (%.2f cyc/imma/SM), kernel %.3f ms  %s\n",
           mode, mode == 1 ? "umma only" : mode == 2 ? "imma only" : "both", h[0], (double)h[0] / R, h[1],
           (double)h[1] / (15.0 * 4 * M), ms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
