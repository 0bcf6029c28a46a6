// Microbenchmark for the J-neighbours-per-thread scan design (J = 4):
// ONE class via uniform candidate loads + predicated select, TAIL via uniform
// loads shared by J chains, BOTH via per-cell divergent LDS.64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
constexpr int KC = 512, REC = 64, J = 4;

__device__ __forceinline__ double lds_f64(uint32_t a) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a)); return v; }
__device__ __forceinline__ void lds_f64x2(uint32_t a, double& x, double& y) { asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(x), "=d"(y) : "r"(a)); }

template <int MODE>
__global__ void kern(int reps, double* out, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* tab = reinterpret_cast<double*>(smem);
  for (int i = threadIdx.x; i < KC * REC / 8 + 64; i += blockDim.x) tab[i] = 1.0 + (i & 7) * 0.25 + (i >> 3) * 1e-3;
  __syncthreads();
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  uint32_t P[J];
  for (int m = 0; m < J; ++m) P[m] = 0x9E3779B9u * (threadIdx.x * J + m + 1);
  double s[J];
  for (int m = 0; m < J; ++m) s[m] = 0.0;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int kb = 0; kb < KC; kb += 32) {
      const uint32_t rec = sbase + kb * REC;
      if (MODE == 0) {          // ONE: candidates (e3,e1) uniform per k, select per neighbour
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          double e3, e1; lds_f64x2(rec + q * REC + 32, e3, e1);
#pragma unroll
          for (int m = 0; m < J; ++m) {
            const double t = (P[m] >> q) & 1u ? e1 : e3;
            s[m] = __dadd_rn(s[m], t);
          }
        }
      } else if (MODE == 1) {   // TAIL: e2 pairs uniform, shared by J chains
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          double a, b; lds_f64x2(sbase + (kb + q) * 8, a, b);
#pragma unroll
          for (int m = 0; m < J; ++m) { s[m] = __dadd_rn(s[m], a); s[m] = __dadd_rn(s[m], b); }
        }
      } else if (MODE == 2) {   // BOTH: per-cell divergent LDS.64 (4 slots), J chains
#pragma unroll
        for (int q = 0; q < 32; ++q) {
#pragma unroll
          for (int m = 0; m < J; ++m) {
            const uint32_t w = P[m];
            const int sh = (2 * q - 3) & 31;
            const uint32_t v = q < 2 ? (w << (3 - 2 * q)) : (w >> sh);
            s[m] = __dadd_rn(s[m], lds_f64(((v & 0x18u) | rec) + q * REC));
          }
        }
      } else if (MODE == 4) {   // ONE: predicated DADD pair per cell
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          double e3, e1; lds_f64x2(rec + q * REC + 32, e3, e1);
#pragma unroll
          for (int m = 0; m < J; ++m) {
            asm("{ .reg .pred p; setp.ne.b32 p, %1, 0;\n @p add.rn.f64 %0, %0, %2;\n @!p add.rn.f64 %0, %0, %3; }"
                : "+d"(s[m]) : "r"(P[m] & (1u << q)), "d"(e1), "d"(e3));
          }
        }
      } else if (MODE == 5) {   // BOTH: 3 predicated DADDs per cell
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          double e4, e2, e0, ex; lds_f64x2(rec + q * REC, e4, e2); lds_f64x2(rec + q * REC + 16, ex, e0);
#pragma unroll
          for (int m = 0; m < J; ++m) {
            const uint32_t X = P[m], A = P[m] * 3u;
            asm("{ .reg .pred px, pa, pb;\n"
                " setp.ne.b32 px, %1, 0;\n setp.ne.b32 pa, %2, 0;\n setp.ne.b32 pb, %3, 0;\n"
                " @px add.rn.f64 %0, %0, %4;\n @pa add.rn.f64 %0, %0, %5;\n @pb add.rn.f64 %0, %0, %6; }"
                : "+d"(s[m]) : "r"(X & (1u << q)), "r"(~X & A & (1u << q)), "r"(~X & ~A & (1u << q)),
                  "d"(e2), "d"(e0), "d"(e4));
          }
        }
      } else if (MODE == 6) {   // ONE: 2 FSEL + 2 IMAD-select neighbours, d computed per k
        uint32_t R2 = __brev(P[2]), R3 = __brev(P[3]);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          double e3, e1; lds_f64x2(rec + q * REC + 32, e3, e1);
          const uint32_t e3l = __double2loint(e3), e3h = __double2hiint(e3);
          const uint32_t dl = __double2loint(e1) - e3l, dh = __double2hiint(e1) - e3h;
          s[0] = __dadd_rn(s[0], (P[0] & (1u << q)) ? e1 : e3);
          s[1] = __dadd_rn(s[1], (P[1] & (1u << q)) ? e1 : e3);
          uint64_t w2, w3;
          asm("mul.wide.u32 %0, %1, 2;" : "=l"(w2) : "r"(R2)); R2 = (uint32_t)w2; const uint32_t b2 = w2 >> 32;
          asm("mul.wide.u32 %0, %1, 2;" : "=l"(w3) : "r"(R3)); R3 = (uint32_t)w3; const uint32_t b3 = w3 >> 32;
          s[2] = __dadd_rn(s[2], __hiloint2double((int)(b2 * dh + e3h), (int)(b2 * dl + e3l)));
          s[3] = __dadd_rn(s[3], __hiloint2double((int)(b3 * dh + e3h), (int)(b3 * dl + e3l)));
        }
      } else if (MODE == 7) {   // ONE: 4 IMAD-select neighbours, (e3, d) from the record
        uint32_t R[J]; for (int m = 0; m < J; ++m) R[m] = P[m];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          uint32_t e3l, e3h, dl, dh;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(e3l), "=r"(e3h), "=r"(dl), "=r"(dh) : "r"(rec + q * REC + 32));
#pragma unroll
          for (int m = 0; m < J; ++m) {
            uint64_t w; asm("mul.wide.u32 %0, %1, 2;" : "=l"(w) : "r"(R[m])); R[m] = (uint32_t)w; const uint32_t b = w >> 32;
            s[m] = __dadd_rn(s[m], __hiloint2double((int)(b * dh + e3h), (int)(b * dl + e3l)));
          }
        }
      } else if (MODE == 8) {   // ONE: 2 FSEL + 2 IMAD, d from the record (LDS.128 + LDS.64)
        uint32_t R2 = P[2], R3 = P[3];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          double e3, e1; lds_f64x2(rec + q * REC + 32, e3, e1);
          uint32_t dl, dh; asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(dl), "=r"(dh) : "r"(rec + q * REC + 48));
          const uint32_t e3l = __double2loint(e3), e3h = __double2hiint(e3);
          s[0] = __dadd_rn(s[0], (P[0] & (1u << q)) ? e1 : e3);
          s[1] = __dadd_rn(s[1], (P[1] & (1u << q)) ? e1 : e3);
          uint64_t w2, w3;
          asm("mul.wide.u32 %0, %1, 2;" : "=l"(w2) : "r"(R2)); R2 = (uint32_t)w2; const uint32_t b2 = w2 >> 32;
          asm("mul.wide.u32 %0, %1, 2;" : "=l"(w3) : "r"(R3)); R3 = (uint32_t)w3; const uint32_t b3 = w3 >> 32;
          s[2] = __dadd_rn(s[2], __hiloint2double((int)(b2 * dh + e3h), (int)(b2 * dl + e3l)));
          s[3] = __dadd_rn(s[3], __hiloint2double((int)(b3 * dh + e3h), (int)(b3 * dl + e3l)));
        }
      } else if (MODE == 9) {   // ONE: 4xFSEL with predicates from R2P (7 bits per group)
#pragma unroll
        for (int g = 0; g < 5; ++g) {
          uint32_t x[J];
#pragma unroll
          for (int m = 0; m < J; ++m) x[m] = P[m] >> (7 * g);
#pragma unroll
          for (int qq = 0; qq < 7; ++qq) {
            const int q = 7 * g + qq;
            if (q >= 32) break;
            double e3, e1; lds_f64x2(rec + q * REC + 32, e3, e1);
#pragma unroll
            for (int m = 0; m < J; ++m) {
              const bool b = (x[m] >> qq) & 1u;
              s[m] = __dadd_rn(s[m], b ? e1 : e3);
            }
          }
        }
      } else if (MODE == 10) {  // ONE: R2P-friendly order: per group, terms per neighbour, then chains
#pragma unroll
        for (int g = 0; g < 5; ++g) {
          constexpr int G = 7;
          double e3[G], e1[G];
#pragma unroll
          for (int qq = 0; qq < G; ++qq) { const int q = G * g + qq; if (q < 32) lds_f64x2(rec + q * REC + 32, e3[qq], e1[qq]); }
          double tm[J][G];
#pragma unroll
          for (int m = 0; m < J; ++m) {
            const uint32_t x = P[m] >> (G * g);
#pragma unroll
            for (int qq = 0; qq < G; ++qq) tm[m][qq] = ((x >> qq) & 1u) ? e1[qq] : e3[qq];
          }
#pragma unroll
          for (int qq = 0; qq < G; ++qq) {
            if (G * g + qq >= 32) break;
#pragma unroll
            for (int m = 0; m < J; ++m) s[m] = __dadd_rn(s[m], tm[m][qq]);
          }
        }
      } else if (MODE == 11 || MODE == 12) {  // ONE: NF FSEL (R2P order) + rest IMAD select, d from record
        constexpr int NF = (MODE == 11) ? 3 : 2;
        uint32_t R[J];
#pragma unroll
        for (int m = NF; m < J; ++m) R[m] = __brev(P[m]);
#pragma unroll
        for (int g = 0; g < 5; ++g) {
          constexpr int G = 7;
          double e3[G], e1[G];
          uint32_t dl[G], dh[G];
#pragma unroll
          for (int qq = 0; qq < G; ++qq) {
            const int q = G * g + qq;
            if (q < 32) {
              lds_f64x2(rec + q * REC + 32, e3[qq], e1[qq]);
              asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(dl[qq]), "=r"(dh[qq]) : "r"(rec + q * REC + 48));
            }
          }
          double tm[J][G];
#pragma unroll
          for (int m = 0; m < NF; ++m) {
            const uint32_t x = P[m] >> (G * g);
#pragma unroll
            for (int qq = 0; qq < G; ++qq) tm[m][qq] = ((x >> qq) & 1u) ? e1[qq] : e3[qq];
          }
#pragma unroll
          for (int qq = 0; qq < G; ++qq) {
            if (G * g + qq >= 32) break;
#pragma unroll
            for (int m = NF; m < J; ++m) {
              uint64_t w; asm("mul.wide.u32 %0, %1, 2;" : "=l"(w) : "r"(R[m])); R[m] = (uint32_t)w; const uint32_t b = w >> 32;
              tm[m][qq] = __hiloint2double((int)(b * dh[qq] + (uint32_t)__double2hiint(e3[qq])),
                                           (int)(b * dl[qq] + (uint32_t)__double2loint(e3[qq])));
            }
#pragma unroll
            for (int m = 0; m < J; ++m) s[m] = __dadd_rn(s[m], tm[m][qq]);
          }
        }
      } else if (MODE == 13 || MODE == 14) {  // ONE: predicated DADD pairs (NP neighbours), FSEL for the rest
        constexpr int NP = (MODE == 13) ? 4 : 2;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          constexpr int G = 4;
          double e3[G], e1[G];
#pragma unroll
          for (int qq = 0; qq < G; ++qq) lds_f64x2(rec + (G * g + qq) * REC + 32, e3[qq], e1[qq]);
          double tm[J][G];
#pragma unroll
          for (int m = NP; m < J; ++m) {
            const uint32_t x = P[m] >> (G * g);
#pragma unroll
            for (int qq = 0; qq < G; ++qq) tm[m][qq] = ((x >> qq) & 1u) ? e1[qq] : e3[qq];
          }
#pragma unroll
          for (int qq = 0; qq < G; ++qq) {
#pragma unroll
            for (int m = 0; m < NP; ++m) {
              const uint32_t bit = (P[m] >> (G * g + qq)) & 1u;
              asm volatile("{ .reg .pred p; setp.ne.u32 p, %1, 0;\n"
                           "  @p add.rn.f64 %0, %0, %2;\n"
                           "  @!p add.rn.f64 %0, %0, %3; }" : "+d"(s[m]) : "r"(bit), "d"(e1[qq]), "d"(e3[qq]));
            }
#pragma unroll
            for (int m = NP; m < J; ++m) s[m] = __dadd_rn(s[m], tm[m][qq]);
          }
        }
      } else if (MODE == 15) {  // ONE: 3 FSEL (R2P order) + 1 divergent-LDS neighbour
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          constexpr int G = 4;
          double e3[G], e1[G];
#pragma unroll
          for (int qq = 0; qq < G; ++qq) lds_f64x2(rec + (G * g + qq) * REC + 32, e3[qq], e1[qq]);
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const uint32_t x = P[m] >> (G * g);
#pragma unroll
            for (int qq = 0; qq < G; ++qq) s[m] = __dadd_rn(s[m], ((x >> qq) & 1u) ? e1[qq] : e3[qq]);
          }
#pragma unroll
          for (int qq = 0; qq < G; ++qq) {
            const int q = G * g + qq;
            const uint32_t v = q < 3 ? (P[3] << (3 - q)) : (P[3] >> (q - 3));
            uint32_t a; asm("lop3.b32 %0, %1, 8, %2, 0xEA;" : "=r"(a) : "r"(v), "r"(rec + 32));
            s[3] = __dadd_rn(s[3], lds_f64(a + q * REC));
          }
        }
      } else if (MODE == 16) {  // BOTH: 2 LDS neighbours + 2 FSEL 2-level neighbours
        uint32_t X[J], Y[J];
#pragma unroll
        for (int m = 0; m < J; ++m) { X[m] = P[m]; Y[m] = P[m] * 2654435761u; }
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          constexpr int G = 4;
          double e4[G], e2[G], e0[G];
#pragma unroll
          for (int qq = 0; qq < G; ++qq) { lds_f64x2(rec + (G * g + qq) * REC, e4[qq], e2[qq]); e0[qq] = lds_f64(rec + (G * g + qq) * REC + 24); }
#pragma unroll
          for (int m = 2; m < 4; ++m) {
            const uint32_t x = X[m] >> (G * g), y = Y[m] >> (G * g);
#pragma unroll
            for (int qq = 0; qq < G; ++qq)
              s[m] = __dadd_rn(s[m], ((x >> qq) & 1u) ? e2[qq] : (((y >> qq) & 1u) ? e0[qq] : e4[qq]));
          }
#pragma unroll
          for (int qq = 0; qq < G; ++qq) {
            const int q = G * g + qq;
#pragma unroll
            for (int m = 0; m < 2; ++m) {
              const uint32_t w = P[m];
              const int sh = (2 * q - 3) & 31;
              const uint32_t v = q < 2 ? (w << (3 - 2 * q)) : (w >> sh);
              uint32_t a; asm("lop3.b32 %0, %1, 0x18, %2, 0xEA;" : "=r"(a) : "r"(v), "r"(rec));
              s[m] = __dadd_rn(s[m], lds_f64(a + q * REC));
            }
          }
        }
      } else if (MODE == 3) {   // BOTH via select: candidates (e4,e2),(e0,x) uniform
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          double e4, e2, e0, ex; lds_f64x2(rec + q * REC, e4, e2); lds_f64x2(rec + q * REC + 16, ex, e0);
#pragma unroll
          for (int m = 0; m < J; ++m) {
            const uint32_t x = (P[m] >> q) & 1u, y = (P[m] >> ((q + 7) & 31)) & 1u;
            const double t = x ? e2 : (y ? e0 : e4);
            s[m] = __dadd_rn(s[m], t);
          }
        }
      }
      for (int m = 0; m < J; ++m) P[m] = P[m] * 1664525u + 1013904223u;
    }
  }
  const long long t1 = clock64();
  double acc = 0; for (int m = 0; m < J; ++m) acc += s[m];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
int run(const char* name, int nsm, int threads, int ctas_per_sm, int reps) {
  double* out; long long* cyc;
  const int grid = nsm * ctas_per_sm;
  CK(cudaMalloc(&out, sizeof(double) * grid * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * grid));
  const int smem = KC * REC + 1024;
  CK(cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  kern<MODE><<<grid, threads, smem>>>(2, out, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE><<<grid, threads, smem>>>(reps, out, cyc);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double cells = (double)grid * threads * J * reps * KC;
  printf("%-26s thr=%4d ctas/SM=%d  %.3f ms  %.3e cells/s  %.2f cells/clk/SM @1.965GHz\n", name, threads,
         ctas_per_sm, ms, cells / (ms * 1e-3), cells / (ms * 1e-3) / nsm / 1.965e9);
  cudaFree(out); cudaFree(cyc);
  return 0;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int nsm = p.multiProcessorCount;
  for (int cps = 2; cps <= 2; ++cps) {
    const int th = 256;
    run<10>("ONE 4xFSEL R2P v2", nsm, th, cps, 100);
    run<15>("ONE 3 FSEL + 1 LDS", nsm, th, cps, 100);
    run<2>("BOTH 4 LDS", nsm, th, cps, 100);
    run<16>("BOTH 2 LDS + 2 FSEL", nsm, th, cps, 100);
  }
  return 0;
}
