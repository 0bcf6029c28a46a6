// tcgen05.mma kind::i8 with Hankel-core A and shifted-digit-core B descriptors:
// Out[r][(g,d)] = sum_kappa A[r][kappa] * B[kappa][(g,d)],
//   A[r][kappa] = S[r + kappa]                   (sequence bytes, Hankel)
//   B[kappa][(g,d)] = D[d][kappa + 16*8*g']      (digit rows, shifted per N-group)
// A is stored as "cores": Core[m] = 8 rows x 16 bytes, row i = S[8m + i .. 8m + i + 15];
// the A descriptor for K-step s starts at Core[4s] with SBO = 128 B (next 8 rows)
// and LBO = 256 B (next 16 k).  B cores: DC[q] = 8 digit rows x 16 k-bytes at
// k = 16q..16q+15; the N-group g starts 8 cores further (SBO = 1024 B), LBO = 128 B.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, NG = 10, N = 8 * NG, KSTEPS = 16;      // K = 32 * KSTEPS
constexpr int KTOT = 32 * KSTEPS;
constexpr int NPOS = M + KTOT + 64;                           // sequence bytes used
constexpr int NCORE_A = NPOS / 8;
constexpr int KB = KTOT + 128 * NG + 64;                      // digit k-range
constexpr int NCORE_B = KB / 16;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;             // version (Blackwell)
  return d;                            // base_offset 0, lbo_mode 0, SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)        // D format S32
       | (1u << 7)        // A signed 8-bit
       | (1u << 10)       // B signed 8-bit
       | ((uint32_t)(n >> 3) << 17)
       | ((uint32_t)(m >> 4) << 24);
}

__global__ void __launch_bounds__(128) umma_kernel(const int8_t* S, const int8_t* Dg, int32_t* out, int reps) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* coreA = smem;                                   // NCORE_A * 128
  unsigned char* coreB = smem + NCORE_A * 128;                   // NCORE_B * 128
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int t = threadIdx.x;
  for (int m = t; m < NCORE_A; m += blockDim.x)
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 16; ++j) coreA[m * 128 + i * 16 + j] = (unsigned char)S[8 * m + i + j];
  for (int q = t; q < NCORE_B; q += blockDim.x)
    for (int d = 0; d < 8; ++d)
      for (int j = 0; j < 16; ++j) coreB[q * 128 + d * 16 + j] = (unsigned char)Dg[d * KB + 16 * q + j];
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)), "r"(128) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t aA = (uint32_t)__cvta_generic_to_shared(coreA);
  const uint32_t aB = (uint32_t)__cvta_generic_to_shared(coreB);
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (t == 0) {
      for (int s = 0; s < KSTEPS; ++s) {
        // A: rows r, k = 32s + kk -> S[r + 32 s + kk]: start core 4s
        const uint64_t da = sdesc(aA + 128 * (4 * s), 256, 128);
        // B: N-group g (= sigma reversed), k = 32 s + kk: digit cores start at 2s + 8g
        const uint64_t db = sdesc(aB + 128 * (2 * s), 128, 1024);
        const uint32_t acc = (s > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc_i8(M, N)), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    }
    // wait for the MMAs
    {
      const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
      uint32_t done = 0;
      while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(mb), "r"(phase) : "memory");
      }
      phase ^= 1;
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // TMEM -> registers: warp w reads lanes 32w..32w+31, 8 columns at a time
  const int w = t >> 5;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + ((uint32_t)(32 * w) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[t * N + c0 + j] = (int32_t)v[j];
  }
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
}

int main() {
  int8_t* hS = (int8_t*)malloc(NPOS + 64);
  int8_t* hD = (int8_t*)malloc(8 * KB);
  srand(7);
  for (int i = 0; i < NPOS + 64; ++i) hS[i] = (rand() & 1) ? 1 : -1;
  for (int i = 0; i < 8 * KB; ++i) hD[i] = (int8_t)((rand() & 255) - 128);
  int8_t *dS, *dD;
  int32_t* dO;
  cudaMalloc(&dS, NPOS + 64); cudaMalloc(&dD, 8 * KB); cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dS, hS, NPOS + 64, cudaMemcpyHostToDevice);
  cudaMemcpy(dD, hD, 8 * KB, cudaMemcpyHostToDevice);
  const int smem = NCORE_A * 128 + NCORE_B * 128;
  cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_kernel<<<1, 128, smem>>>(dS, dD, dO, 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  int32_t* hO = (int32_t*)malloc(M * N * 4);
  cudaMemcpy(hO, dO, M * N * 4, cudaMemcpyDeviceToHost);
  // reference: column n = 8 g + d ; B[kappa][n] = D[d][kappa + 128 g]... (core q = 2s + 8g -> k offset 16*8g = 128 g)
  int bad = 0;
  for (int r = 0; r < M; ++r)
    for (int g = 0; g < NG; ++g)
      for (int d = 0; d < 8; ++d) {
        long long acc = 0;
        for (int k = 0; k < KTOT; ++k) acc += (long long)hS[r + k] * hD[d * KB + k + 128 * g];
        const int32_t got = hO[r * N + 8 * g + d];
        if (got != acc) { if (bad < 10) printf("mismatch r=%d g=%d d=%d got=%d want=%lld\n", r, g, d, got, acc); ++bad; }
      }
  printf("%s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  // timing: many reps on all SMs
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int reps = 2000;
  cudaEventRecord(a);
  umma_kernel<<<sms, 128, smem>>>(dS, dD, dO, reps);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double macs = (double)sms * reps * KSTEPS * M * N * 32;
  printf("throughput: %.1f TMAC/s  (%.0f MAC/clk/SM at 1.9 GHz)\n", macs / (ms * 1e-3) / 1e12,
         macs / (ms * 1e-3) / sms / 1.9e9);
  return bad ? 1 : 0;
}
