// mma.sync m16n8k32 s8 throughput vs resident warps per SM and independent accumulators.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int NACC>
__global__ void kern(int reps, int* out) {
  uint32_t a0 = 0x01010101u * (threadIdx.x + 1), a1 = a0 ^ 0x5a5a5a5au, a2 = ~a0, a3 = a0 + 7;
  const uint32_t b0 = 0x03030303u * threadIdx.x, b1 = ~b0;
  int d[NACC][4] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < NACC; ++q)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[q][0]), "+r"(d[q][1]), "+r"(d[q][2]), "+r"(d[q][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    a0 += 1;
  }
  int s = 0;
  for (int q = 0; q < NACC; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3];
  if (s == 0x7fffffff) out[0] = s;
}
template <int NACC>
void run(int sms, int warps_per_sm, int* dout) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 4096 * 8 / NACC;
  kern<NACC><<<sms, 32 * warps_per_sm>>>(16, dout);
  cudaEventRecord(e0);
  kern<NACC><<<sms, 32 * warps_per_sm>>>(reps, dout);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)sms * warps_per_sm * reps * NACC;
  printf("warps/SM %2d  acc %2d  %.3f mma/clk/SM\n", warps_per_sm, NACC, mmas / (ms * 1e-3) / sms / 1.9e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* d; cudaMalloc(&d, 64);
  for (int w : {4, 8, 16, 32}) { run<1>(sms, w, d); run<2>(sms, w, d); run<4>(sms, w, d); run<8>(sms, w, d); }
  return 0;
}
