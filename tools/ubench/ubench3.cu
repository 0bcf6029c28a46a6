// Microbenchmarks for the certified (decision-exact) scan design:
//   b1 mma.sync (AND/XOR + popc) and s8 mma.sync throughput on sm_100a,
//   POPC throughput, the latency of one serial DADD chain, and the fp32
//   select+add cell rate of the both-sides cross term.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void mma_b1_and(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_b1_xor(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_s8(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

constexpr int NACC = 8;

template <int MODE>
__global__ void kern(int reps, int* out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x9E3779B9u * (threadIdx.x + 7 * i + 1);
  for (int i = 0; i < 2; ++i) b[i] = 0x85EBCA6Bu * (threadIdx.x + 3 * i + 1);
  int d[NACC][4] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      if (MODE == 0) mma_b1_and(d[q], a, b);
      else if (MODE == 1) mma_b1_xor(d[q], a, b);
      else mma_s8(d[q], a, b);
    }
    a[0] += 1;
  }
  int s = 0;
  for (int q = 0; q < NACC; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3];
  if (s == 0x12345) out[0] = s;
}

__global__ void popc_kern(int reps, int* out) {
  uint32_t x[8];
  for (int i = 0; i < 8; ++i) x[i] = 0x9E3779B9u * (threadIdx.x + i + 1);
  uint32_t acc[8] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i] += __popc(x[i] ^ acc[(i + 1) & 7]); }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 0x12345) out[0] = s;
}

__global__ void chain_kern(int n, double* out, long long* cyc) {
  double s = 0.0, t = 1.0 + threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < n; i += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dadd_rn(s, t);
  }
  const long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// cross term: acc += bit ? R_k : 0 in fp32, R uniform per k, bit per lane (4 neighbours/lane)
__global__ void cross_kern(int reps, const float* R, float* out) {
  __shared__ float rs[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) rs[i] = R[i];
  __syncthreads();
  uint32_t w[4];
  for (int m = 0; m < 4; ++m) w[m] = 0x9E3779B9u * (threadIdx.x * 4 + m + 1);
  float acc[4] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int kb = 0; kb < 512; kb += 32) {
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const float rv = rs[kb + q];
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[m] += ((w[m] >> q) & 1u) ? rv : 0.0f;
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) w[m] = w[m] * 0x2545F491u + 1u;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  int* dout; CK(cudaMalloc(&dout, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double ghz = 1.965;
  auto run_mma = [&](auto kfn, const char* name, double ops_per_mma) {
    const int reps = 4096, threads = 256, blocks = sms * 4;
    kfn<<<blocks, threads>>>(16, dout);
    cudaEventRecord(e0);
    kfn<<<blocks, threads>>>(reps, dout);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = (double)blocks * (threads / 32) * reps * NACC;
    printf("%-12s %.3f ms  %.3e mma/s  %.2f mma/clk/SM  %.1f Tops/s\n", name, ms, mmas / (ms * 1e-3),
           mmas / (ms * 1e-3) / sms / (ghz * 1e9), mmas * ops_per_mma / (ms * 1e-3) / 1e12);
  };
  run_mma(kern<0>, "b1.and.popc", 2.0 * 16 * 8 * 256);
  run_mma(kern<1>, "b1.xor.popc", 2.0 * 16 * 8 * 256);
  run_mma(kern<2>, "s8 k32", 2.0 * 16 * 8 * 32);
  {
    const int reps = 8192, threads = 256, blocks = sms * 8;
    popc_kern<<<blocks, threads>>>(16, dout);
    cudaEventRecord(e0);
    popc_kern<<<blocks, threads>>>(reps, dout);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * reps * 8;
    printf("%-12s %.3f ms  %.2f popc/clk/SM\n", "popc", ms, ops / (ms * 1e-3) / sms / (ghz * 1e9));
  }
  {
    double* dd; long long* dc; CK(cudaMalloc(&dd, 4096)); CK(cudaMalloc(&dc, 64));
    const int n = 1 << 20;
    chain_kern<<<1, 1>>>(1024, dd, dc);
    cudaEventRecord(e0);
    chain_kern<<<1, 1>>>(n, dd, dc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%-12s n=%d  %.3f ms  %.2f clk/add\n", "dadd chain", n, ms, (double)c / n);
  }
  {
    float* R; float* o; CK(cudaMalloc(&R, 512 * 4)); CK(cudaMalloc(&o, sms * 2 * 256 * 4));
    cudaMemset(R, 0, 512 * 4);
    const int reps = 256, threads = 256, blocks = sms * 2;
    cross_kern<<<blocks, threads>>>(4, R, o);
    cudaEventRecord(e0);
    cross_kern<<<blocks, threads>>>(reps, R, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double cells = (double)blocks * threads * 4 * reps * 512;
    printf("%-12s %.3f ms  %.2f cells/clk/SM\n", "cross fp32", ms, cells / (ms * 1e-3) / sms / (ghz * 1e9));
  }
  CK(cudaGetLastError());
  return 0;
}
