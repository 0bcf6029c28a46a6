// mma.sync throughput vs warps/SM and independent accumulator chains (B200).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o imma_rate imma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int CH, int KIND>
__global__ void k(int reps, int* out) {
  uint32_t a[CH][4];
  for (int q = 0; q < CH; ++q) for (int i = 0; i < 4; ++i) a[q][i] = 0x01010101u * (threadIdx.x + q + i);
  const uint32_t b0 = 0x03030303u * threadIdx.x, b1 = ~b0;
  int d[CH][4] = {};
  float f[CH][4] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(d[q][0]), "+r"(d[q][1]), "+r"(d[q][2]), "+r"(d[q][3])
                     : "r"(a[q][0]), "r"(a[q][1]), "r"(a[q][2]), "r"(a[q][3]), "r"(b0), "r"(b1));
      else if (KIND == 1)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(f[q][0]), "+f"(f[q][1]), "+f"(f[q][2]), "+f"(f[q][3])
                     : "r"(a[q][0]), "r"(a[q][1]), "r"(a[q][2]), "r"(a[q][3]), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(f[q][0]), "+f"(f[q][1]), "+f"(f[q][2]), "+f"(f[q][3])
                     : "r"(a[q][0]), "r"(a[q][1]), "r"(a[q][2]), "r"(a[q][3]), "r"(b0), "r"(b1));
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) a[q][0] += 1;
  }
  int s = 0;
  for (int q = 0; q < CH; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3] + (int)f[q][0] + (int)f[q][3];
  if (s == 0x7fffffff) out[0] = s;
}
template <int CH, int KIND>
void run(int warps, const char* name) {
  int* out; cudaMalloc(&out, 64);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 4096;
  k<CH, KIND><<<nsm, 32 * warps>>>(8, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH, KIND><<<nsm, 32 * warps>>>(reps, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_sm = (double)warps * reps * CH / (ms * 1e-3);   // mma per s per SM
  printf("%s warps=%2d chains=%d : %.2f cyc/mma/SM (at %.0f MHz)  err=%s\n", name, warps, CH,
         clk * 1e3 / per_sm, clk / 1e3, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<4, 0>(16, "imma m16n8k32"); run<8, 0>(16, "imma m16n8k32"); run<4, 0>(32, "imma m16n8k32");
  run<8, 0>(32, "imma m16n8k32"); run<2, 0>(16, "imma m16n8k32"); run<4, 0>(8, "imma m16n8k32");
  run<4, 1>(16, "hmma m16n8k16"); run<8, 1>(32, "hmma m16n8k16");
  run<4, 2>(16, "e4m3 m16n8k32"); run<8, 2>(32, "e4m3 m16n8k32");
  return 0;
}
