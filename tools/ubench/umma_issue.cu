// How long does one thread block in tcgen05.mma issue, and how long do R
// back-to-back kind::i8 M128 x N x K32 MMAs (SS mode, the certified scan's
// descriptor strides) take to complete?  One CTA per SM, all SMs.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o umma_issue umma_issue.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__global__ void __launch_bounds__(512) k(int n, int R, int ldsw, long long* out, int nis, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int t = threadIdx.x;
  for (int i = t; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "r"(512) : "memory");
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
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
  long long t0 = 0, t1 = 0, t2 = 0;
  if (mode == 1 && t < 32) {
    // whole warp, uniform descriptors, one lane elected inside the asm
    uint64_t da = sdesc(base, 256, 128), db = sdesc(base + 40960, 128, 1024);
    t0 = clock64();
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_base),
                   "l"(da), "l"(db), "r"(idesc), "r"(r));
      da += 512 >> 4; db += 256 >> 4;
      if ((r & 15) == 15) { da -= (16 * 512) >> 4; db -= (16 * 256) >> 4; }
    }
    t1 = clock64();
    if (t == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    uint32_t done = 0;
    for (int it = 0; !done && it < 2000000; ++it)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(0) : "memory");
    t2 = clock64();
  } else if (mode == 0 && (t & 31) == 0 && (t >> 5) < nis) {
    uint64_t da = sdesc(base, 256, 128), db = sdesc(base + 40960, 128, 1024);
    t0 = clock64();
    for (int r = 0; r < R / nis; ++r) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_base),
                   "l"(da), "l"(db), "r"(idesc), "r"(r));
      da += 512 >> 4; db += 256 >> 4;
      if ((r & 15) == 15) { da -= (16 * 512) >> 4; db -= (16 * 256) >> 4; }
    }
    t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    uint32_t done = 0;
    for (int it = 0; !done && it < 2000000; ++it)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(0) : "memory");
    t2 = clock64();
  }
  if (ldsw && t >= 32) {
    // other warps hammer shared memory (LDS.128, conflict-free) meanwhile
    uint32_t acc = 0, a = base + 16 * (t & 31) + 512 * ((t >> 5) & 7);
    for (int i = 0; i < ldsw; ++i) {
      uint4 v;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a + ((i * 4096) & 32767)));
      acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345) out[1023] = acc;
  }
  __syncthreads();
  if (t == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
}
int main(int argc, char** argv) {
  const int only_nis = argc > 1 ? atoi(argv[1]) : 0;
  long long* d; cudaMalloc(&d, 8192);
  long long h[2];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int mode : {1})
  for (int nis : {1}) if (!only_nis || nis == only_nis)
  for (int thr : {128, 512})
  for (int ldsw : {0, 20000})
    for (int n : {64})
      for (int R : {32, 64}) {
        k<<<nsm, thr, 96 * 1024>>>(n, R, ldsw, d, nis, mode);
        k<<<nsm, thr, 96 * 1024>>>(n, R, ldsw, d, nis, mode);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("thr=%d mode=%d issuers=%d lds=%d N=%2d R=%2d issue %6lld cyc  complete %6lld cyc  (%.1f cyc/mma)  %s\n", thr, mode, nis, ldsw, n, R, h[0], h[1],
               (double)h[1] / R, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
