// Microbenchmarks for the scan-kernel design decisions (B200, sm_100a).
// Measures cells/clk/SM for candidate inner loops: per-cell slot lookup in a
// 64 B/k smem record + serial DADD chain, the tail (broadcast) path, raw
// LDS.64 throughput and DADD throughput/latency.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int KC = 512;          // k records per smem buffer
constexpr int REC = 64;          // bytes per k record

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr)); return v;
}
__device__ __forceinline__ void lds_f64x2(uint32_t addr, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr));
}

// Variant A: general per-cell path. offset = ((W >> s) & mask) | base.
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_cells(int reps, double* out, long long* cyc) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* tab = reinterpret_cast<double*>(smem);
  for (int i = threadIdx.x; i < KC * REC / 8; i += blockDim.x) tab[i] = 1.0 + (i & 7) * 0.25;
  __syncthreads();
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  uint32_t wlo = 0x9E3779B9u * (threadIdx.x + 1), whi = 0x85EBCA6Bu * (threadIdx.x + 7);
  const uint32_t mask = 0x18u, base = 0u;
  double sum = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int kb = 0; kb < KC; kb += 32) {
      const uint32_t rec = sbase + kb * REC;
      if (MODE == 0) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t off = (q == 0 ? (wlo << 3) : (q == 1 ? (wlo << 1) : (wlo >> (2 * q - 3)))) & mask | base;
          sum = __dadd_rn(sum, lds_f64(rec + q * REC + off));
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t off = (q == 0 ? (whi << 3) : (q == 1 ? (whi << 1) : (whi >> (2 * q - 3)))) & mask | base;
          sum = __dadd_rn(sum, lds_f64(rec + (16 + q) * REC + off));
        }
      } else if (MODE == 1) {
        // tail path: dense array of doubles, uniform address, LDS.128 broadcast
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          double a, b; lds_f64x2(sbase + (kb + q) * 8, a, b);
          sum = __dadd_rn(sum, a); sum = __dadd_rn(sum, b);
        }
      } else if (MODE == 2) {
        // LDS.64 throughput only (no DADD): xor the low words
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t off = (q == 0 ? (wlo << 3) : (q == 1 ? (wlo << 1) : (wlo >> (2 * q - 3)))) & mask | base;
          double v = lds_f64(rec + q * REC + off);
          acc ^= __double2loint(v);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t off = (q == 0 ? (whi << 3) : (q == 1 ? (whi << 1) : (whi >> (2 * q - 3)))) & mask | base;
          double v = lds_f64(rec + (16 + q) * REC + off);
          acc ^= __double2loint(v);
        }
        sum += (double)acc;
      } else if (MODE == 3) {
        // DADD throughput: 4 independent chains per thread, operands in registers
        double s1 = sum, s2 = sum * 0.5, s3 = sum * 0.25, s4 = 1.0;
        const double x = 1.0000001 + threadIdx.x * 1e-9;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          s1 = __dadd_rn(s1, x); s2 = __dadd_rn(s2, x); s3 = __dadd_rn(s3, x); s4 = __dadd_rn(s4, x);
        }
        sum = s1 + s2 + s3 + s4;
      } else if (MODE == 4) {
        // DADD latency: one chain per thread
        const double x = 1.0000001 + threadIdx.x * 1e-9;
#pragma unroll
        for (int q = 0; q < 32; ++q) sum = __dadd_rn(sum, x);
      } else if (MODE == 5) {
        // pair path: 16-slot table per k-pair (256 B), LDS.128 gives terms for k and k+1.
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = ((q == 0 ? (wlo << 4) : (wlo >> (4 * q - 4))) & 0xF0u);
          double a, b; lds_f64x2(sbase + (kb / 2 + q) * 256 % (KC * REC) + off, a, b);
          sum = __dadd_rn(sum, a); sum = __dadd_rn(sum, b);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = ((q == 0 ? (whi << 4) : (whi >> (4 * q - 4))) & 0xF0u);
          double a, b; lds_f64x2(sbase + (kb / 2 + 8 + q) * 256 % (KC * REC) + off, a, b);
          sum = __dadd_rn(sum, a); sum = __dadd_rn(sum, b);
        }
      }

      if (MODE == 6) {  // LDS.64 per-lane 4-slot, integer consume of both words
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t off = (qq == 0 ? (w << 3) : (qq == 1 ? (w << 1) : (w >> (2 * qq - 3)))) & mask | base;
          uint32_t lo, hi; asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(rec + q * REC + off));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      } else if (MODE == 7) {  // LDS.64 uniform address, integer consume
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          uint32_t lo, hi; asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(rec + q * REC + ((wlo >> 30) & 0) ));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      } else if (MODE == 8) {  // LDS.32 per-lane 4-slot
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t off = (qq == 0 ? (w << 3) : (qq == 1 ? (w << 1) : (w >> (2 * qq - 3)))) & mask | base;
          uint32_t lo; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(rec + q * REC + off));
          acc = acc + lo;
        }
        sum += (double)acc;
      } else if (MODE == 9) {  // DADD with SEL-chosen register operand (no LDS)
        const double x0 = 1.0 + threadIdx.x, x1 = 2.0 + threadIdx.x, x2 = 3.0, x3 = 5.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t b = (w >> (2 * qq)) & 3u;
          const double t = b == 0 ? x0 : (b == 1 ? x1 : (b == 2 ? x2 : x3));
          sum = __dadd_rn(sum, t);
        }
      } else if (MODE == 10) {  // general path, 2 chains per thread (q even / odd)
        double s2 = 0.0;
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t off = (qq == 0 ? (w << 3) : (qq == 1 ? (w << 1) : (w >> (2 * qq - 3)))) & mask | base;
          const uint32_t off2 = ((w << 1) >> (2 * qq)) & mask | base;
          sum = __dadd_rn(sum, lds_f64(rec + q * REC + off));
          s2 = __dadd_rn(s2, lds_f64(rec + (q + 1) * REC + off2));
        }
        sum += s2;
      } else if (MODE == 11) {  // general path but uniform address (mask 0)
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t off = (qq == 0 ? (w << 3) : (qq == 1 ? (w << 1) : (w >> (2 * qq - 3)))) & (mask & 0u) | base;
          sum = __dadd_rn(sum, lds_f64(rec + q * REC + off));
        }
      } else if (MODE == 12) {  // LDS.128 uniform, integer consume
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          uint32_t a, b, c, d; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(sbase + (kb + q) * 8));
          acc = acc + a + b + c + d;
        }
        sum += (double)acc;
      } else if (MODE == 13) {  // two LDS.32 (lo/hi split tables) per cell + DADD
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t off = (qq == 0 ? (w << 2) : (w >> (2 * qq - 2))) & 0xCu;
          uint32_t lo, hi;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(rec + q * 32 + off));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(rec + q * 32 + 16 + off));
          sum = __dadd_rn(sum, __hiloint2double(hi, lo));
        }
      }

      if (MODE == 14) {  // LDS.64: lanes 0-15 addr X, 16-31 addr Y
        uint32_t acc = 0;
        const uint32_t off = (threadIdx.x & 16) ? 8u : 0u;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          uint32_t lo, hi; asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(rec + q * REC + off));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      } else if (MODE == 15) {  // LDS.64: even lanes X, odd lanes Y
        uint32_t acc = 0;
        const uint32_t off = (threadIdx.x & 1) ? 8u : 0u;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          uint32_t lo, hi; asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(rec + q * REC + off));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      } else if (MODE == 16) {  // predicated divergent LDS.64, ~half lanes active, predicated DADDs
        const double e2 = 3.0 + threadIdx.x * 1e-9;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t off = (qq == 0 ? (w << 3) : (qq == 1 ? (w << 1) : (w >> (2 * qq - 3)))) & mask | base;
          const bool x = (w >> (2 * qq)) & 1u;
          double t;
          asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0;\n"
                       "  @!p ld.shared.f64 %0, [%1];\n"
                       "  @p mov.f64 %0, %3; }" : "=d"(t) : "r"(rec + q * REC + off), "r"((uint32_t)x), "d"(e2));
          sum = __dadd_rn(sum, t);
        }
      } else if (MODE == 17) {  // predicated uniform LDS.64 half lanes
        uint32_t acc = 0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t x = (w >> (2 * qq)) & 1u;
          uint32_t lo = 0, hi = 0;
          asm volatile("{ .reg .pred p; setp.ne.u32 p, %3, 0;\n"
                       "  @p ld.shared.v2.u32 {%0,%1}, [%2]; }" : "+r"(lo), "+r"(hi) : "r"(rec + q * REC), "r"(x));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      } else if (MODE == 18) {  // ALU select (x ? e2 : y ? e0 : e4) from registers + DADD
        const uint32_t e4lo = 11u + threadIdx.x, e4hi = 0x40100000u, e2lo = 7u, e2hi = 0x40200000u, e0lo = 3u, e0hi = 0x40300000u;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t b = w >> (2 * qq);
          uint32_t lo, hi;
          asm volatile("{ .reg .pred px, py; .reg .b32 t;\n"
                       "  and.b32 t, %2, 1; setp.ne.u32 px, t, 0;\n"
                       "  and.b32 t, %2, 2; setp.ne.u32 py, t, 0;\n"
                       "  selp.b32 %0, %5, %3, py; selp.b32 %1, %6, %4, py;\n"
                       "  selp.b32 %0, %7, %0, px; selp.b32 %1, %8, %1, px; }"
                       : "=r"(lo), "=r"(hi) : "r"(b), "r"(e4lo), "r"(e4hi), "r"(e0lo), "r"(e0hi), "r"(e2lo), "r"(e2hi));
          sum = __dadd_rn(sum, __hiloint2double(hi, lo));
        }
      }

      if (MODE >= 20 && MODE < 40) {
        uint32_t acc = 0;
        const uint32_t l = threadIdx.x & 31;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          const uint32_t r2 = (w >> (2 * qq)) & 3u;
          uint32_t off;
          if (MODE == 20) off = (l % 3) * 8;
          else if (MODE == 21) off = (l % 4) * 8;
          else if (MODE == 22) off = (l / 8) * 8;
          else if (MODE == 23) off = (l & 1) * 16;
          else if (MODE == 24) off = (l & 1) * 24;
          else if (MODE == 25) off = (l & 1) * 128 % 64 + (l & 1) * 0;
          else if (MODE == 26) off = l * 8;
          else if (MODE == 27) off = (l % 16) * 8;
          else if (MODE == 28) off = (r2 & 1) * 8;
          else if (MODE == 29) off = (r2 == 3 ? 1 : r2) * 8;
          else if (MODE == 30) off = r2 * 8;
          else if (MODE == 31) off = (l % 4) * 4;   // 32-bit-aligned 8-byte? (4-byte stride -> misaligned for 64b) use u32 below
          else off = 0;
          uint32_t lo, hi;
          if (MODE == 31) { asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(rec + q * REC + off)); hi = 0; }
          else asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(rec + q * REC + off));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      }

      if (MODE >= 40 && MODE < 60) {
        uint32_t acc = 0;
        const uint32_t l = threadIdx.x & 31;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const uint32_t w = q < 16 ? wlo : whi; const int qq = q & 15;
          // per-lane random bit for this q, then forced structure
          auto rb = [&](uint32_t lane) { return (__shfl_sync(0xffffffffu, w, lane) >> (2 * qq)) & 1u; };
          uint32_t off;
          if (MODE == 40) off = ((l >> 1) & 1) * 8;
          else if (MODE == 41) off = ((l >> 2) & 1) * 8;
          else if (MODE == 42) off = rb(l & ~1u) * 8;          // pair-uniform random
          else if (MODE == 43) off = rb(l & 15u) * 8;          // l and l+16 equal
          else if (MODE == 44) off = rb(l & ~3u) * 8;          // quad-uniform random
          else if (MODE == 45) off = rb(l & ~7u) * 8;          // octet-uniform random
          else if (MODE == 46) off = rb(l) * 16;               // random X / X+16
          else if (MODE == 47) off = rb(l) * 64;               // random X / X+64 (next record)
          else if (MODE == 48) off = rb(l) * 8 + (l & 16) * 2; // random within half-warp-specific pairs
          else off = rb(l) * 8;                                 // random (T9)
          uint32_t lo, hi;
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(rec + q * REC + off));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      }

      if (MODE >= 60 && MODE < 80) {
        uint32_t acc = 0;
        const uint32_t l = threadIdx.x & 31;
        // per-block patterns prepared once (shuffles outside the cell loop)
        const uint32_t wpair = __shfl_sync(0xffffffffu, wlo, l & ~1u);
        const uint32_t wquad = __shfl_sync(0xffffffffu, wlo, l & ~3u);
        const uint32_t whalf = __shfl_sync(0xffffffffu, wlo, l & 15u);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int qq = q & 15;
          uint32_t off;
          if (MODE == 60) off = ((wlo >> (2 * qq)) & 1u) * 8;            // random 0/8
          else if (MODE == 61) off = ((wpair >> (2 * qq)) & 1u) * 8;     // pair-uniform random 0/8
          else if (MODE == 62) off = ((wquad >> (2 * qq)) & 1u) * 8;     // quad-uniform random
          else if (MODE == 63) off = ((whalf >> (2 * qq)) & 1u) * 8;     // lane l == lane l+16
          else if (MODE == 64) off = ((wlo >> (2 * qq)) & 3u) * 8;       // random 4 slots
          else if (MODE == 65) off = ((wpair >> (2 * qq)) & 3u) * 8;     // pair-uniform 4 slots
          else if (MODE == 66) off = ((wlo >> (2 * qq)) & 1u) * 8 + (l & 1u) * 16; // random, pair parity picks half
          else if (MODE == 67) off = ((wlo >> (2 * qq)) & 1u) * 16 + (l & 1u) * 8; // (X|X+16)+parity*8
          else off = 0;
          uint32_t lo, hi;
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(rec + q * REC + off));
          acc = acc + lo + hi;
        }
        sum += (double)acc;
      }
      // rotate W so the pattern changes per block
      const uint32_t t = wlo; wlo = whi ^ (wlo << 7); whi = t ^ (whi >> 3);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
int run(const char* name, int nsm, int threads, int reps, double cells_per_block_iter) {
  double* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(double) * nsm * 1024));
  CK(cudaMalloc(&cyc, sizeof(long long) * nsm));
  const int smem = KC * REC + 1024;
  CK(cudaFuncSetAttribute(k_cells<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_cells<MODE><<<nsm, threads, smem>>>(2, out, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_cells<MODE><<<nsm, threads, smem>>>(reps, out, cyc);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long c0; CK(cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost));
  const double cells = (double)nsm * threads * reps * (KC / 32) * cells_per_block_iter;
  const double cps_sm = cells / nsm / (double)c0;
  printf("%-28s threads=%4d  %.3f ms  %.3e cells/s  %.2f cells/clk/SM  (clk %.0f MHz)\n",
         name, threads, ms, cells / (ms * 1e-3), cps_sm, c0 / (ms * 1e-3) / 1e6);
  cudaFree(out); cudaFree(cyc);
  return 0;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("%s SMs=%d cc=%d.%d\n", p.name, p.multiProcessorCount, p.major, p.minor);
  const int nsm = p.multiProcessorCount;
  for (int th : {1024}) {
    run<60>("R0 random 0/8", nsm, th, 100, 32);
    run<61>("R1 pair-uniform 0/8", nsm, th, 100, 32);
    run<62>("R2 quad-uniform 0/8", nsm, th, 100, 32);
    run<63>("R3 l==l+16 0/8", nsm, th, 100, 32);
    run<64>("R4 random 4 slots", nsm, th, 100, 32);
    run<65>("R5 pair-uniform 4 slots", nsm, th, 100, 32);
    run<66>("R6 random + parity*16", nsm, th, 100, 32);
    run<67>("R7 random*16 + parity*8", nsm, th, 100, 32);
    run<7>("H uniform", nsm, th, 100, 32);
  }
  return 0;
}
