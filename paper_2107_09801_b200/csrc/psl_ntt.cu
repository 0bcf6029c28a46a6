// psl_ntt.cu -- SidelobeTable::build (sequence.cpp:46-60) for many walks by an
// exact number-theoretic transform.
//
// C_k = sum_i s_i s_{i+k} is the correlation of the +-1 sequence with itself:
// C_k = (x * y)[L-1-k] with y_i = x_{L-1-i}.  Over Z_p with p = 998244353 =
// 119 * 2^23 + 1 (3 is a primitive root) the cyclic convolution of length
// N = 2^ceil(log2(2L)) is exact, and |C_k| <= L < p/2 recovers the signed value.
// O(L log L) per walk instead of the O(L^2) popcount kernel (which stays for
// small L and the single-table C-ABI call).
//
// Only x is transformed: Y(k) = sum_m x_m w^{(L-1-m)k} = w^{(L-1)k} X(-k), so
// the spectrum of the correlation is X(k) X(N-k) w^{(L-1)k}.
//
// Layout: each walk's N values as R rows x C columns (i = m C + col, R C = N),
// transformed by the four-step scheme: R-point DIF down every column (column
// pass: a CTA holds 8 adjacent columns in shared memory, generated straight
// from the packed bits), the twiddle w_N^{k1 col} on the way out, then C-point
// DIF along every row (row pass: a CTA holds a row).  The result sits at the
// full bit-reversed position of k = k1 + R k2, as a radix-2 DIF over N would
// leave it.  Pointwise product on the bit-reversed spectrum.  Inverse
// (bit-reversed -> natural): C-point DIT rows, the inverse twiddle, R-point DIT
// columns, which also scale by N^-1, write C_k (pivot and local tables) and
// reduce the walk's PSL and energy.  Four passes over HBM; inside a pass the
// stages run three at a time in registers (radix-8 rounds).
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "psl_internal.h"

namespace pslb {
namespace {

constexpr uint32_t kP = 998244353u;
constexpr uint32_t kPinv = 998244351u;   // -p^{-1} mod 2^32 (Montgomery)
constexpr uint32_t kOne = 301989884u;    // 2^32 mod p (Montgomery 1)
constexpr int kCols = 8;                 // columns per column-pass CTA (one 32 B sector per row)
constexpr int kMaxRows = 1024;           // R <= 1024, C <= 2048 (N <= 2^21)
constexpr int kMaxRowLen = 2048;
constexpr uint32_t kRowsPerCta = 4;
constexpr uint32_t kNttThreads = 256;       // threads per NTT CTA     // rows per row-pass CTA (amortises the twiddle copy)

// Montgomery product: returns a*b*2^-32 mod p for a, b < p.
__device__ __forceinline__ uint32_t mmul(uint32_t a, uint32_t b) {
  const uint64_t t = (uint64_t)a * b;
  const uint32_t m = (uint32_t)t * kPinv;
  const uint64_t u = (t + (uint64_t)m * kP) >> 32;
  return u >= kP ? (uint32_t)(u - kP) : (uint32_t)u;
}
__device__ __forceinline__ uint32_t madd(uint32_t a, uint32_t b) {
  const uint32_t s = a + b;
  return s >= kP ? s - kP : s;
}
__device__ __forceinline__ uint32_t msub(uint32_t a, uint32_t b) {
  return a >= b ? a - b : a + kP - b;
}
// Shoup product for the butterflies (Harvey's lazy reduction): w < p in normal
// form with wq = floor(w 2^32 / p); for any a < 2^32 returns a w mod p + {0, p}
// (< 2p) in three integer multiplies.  Butterfly values stay below 2p (DIF) or
// 4p (DIT) < 2^32 and are reduced only where a consumer needs it.
__device__ __forceinline__ uint32_t shoup(uint32_t a, uint32_t w, uint32_t wq) {
  return a * w - __umulhi(a, wq) * kP;
}
// Montgomery form of a stage twiddle from its Shoup pair: w 2^32 mod p = -wq p mod 2^32
__device__ __forceinline__ uint32_t pair_mont(uint2 t) { return 0u - t.y * kP; }
// w^e for any e (mod N) from the half table tw[j] = w^j, j < N/2 (w^{N/2} = -1)
__device__ __forceinline__ uint32_t wpow(const uint32_t* tw, uint32_t e, uint32_t N) {
  e &= N - 1;
  const uint32_t h = N >> 1;
  return e < h ? tw[e] : (kP - tw[e - h]) % kP;
}

// ---- radix-8 register rounds -------------------------------------------------
// An n-point transform (n = 2^logn) of each of `cols` interleaved columns is
// held in shared memory, element (i, c) at phys(i, c).  A round performs RB
// consecutive radix-2 stages in registers: every work item loads the 2^RB
// elements base + k u (k < 2^RB), runs the stages of spans u 2^q, stores them
// back: one shared-memory round trip and one barrier per three stages instead
// of per stage.  Stage twiddles: tws[h + j] = w_n^{j n / 2h} (j < h).
//
// Layouts (bank-conflict free for every round, checked by simulation):
//   cols == 1 (row pass):  phys = i ^ (((i >> 5) & 7) << 2); the u == 1 round
//                          moves its 8 contiguous elements as two 16-byte words
//   cols == 8 (column pass): row i sits at row (i & ~3) | ((i + (i >> 3)) & 3)
template <int kColsLog>
__device__ __forceinline__ uint32_t phys(uint32_t i, uint32_t c) {
  if (kColsLog == 0) return i ^ (((i >> 5) & 7u) << 2);
  return ((((i & ~3u) | ((i + (i >> 3)) & 3u))) << kColsLog) + c;
}

// Sizes are template parameters so the index arithmetic folds into immediate
// shared-memory offsets.  GIN / GOUT: the round reads its inputs from / writes
// its outputs to the row in global memory gm (natural order) instead of s.
template <int RB, bool kFwd, int kColsLog, int LOGN, int ULOG, bool GIN = false, bool GOUT = false>
__device__ __forceinline__ void ntt_round(uint32_t* __restrict__ s, const uint2* __restrict__ tws,
                                          uint32_t* __restrict__ gm = nullptr) {
  constexpr int E = 1 << RB;
  constexpr uint32_t cols = 1u << kColsLog, ulog = ULOG;
  constexpr uint32_t u = 1u << ulog;
  constexpr uint32_t items = (1u << (LOGN - RB)) << kColsLog;
#pragma unroll
  for (uint32_t it = threadIdx.x; it < items; it += kNttThreads) {
    const uint32_t c = it & (cols - 1), g = it >> kColsLog;
    const uint32_t off = g & (u - 1), base = ((g >> ulog) << (ulog + RB)) + off;
    uint32_t v[E];
    constexpr bool vec = kColsLog == 0 && RB == 3 && ulog == 0;
    // spans that are multiples of the swizzle period keep the base's swizzle:
    // element k sits at phys(base) + k u cols (immediate offsets)
    constexpr bool lin = kColsLog == 3 ? (u % 32 == 0) : (u % 256 == 0);
    const uint32_t p0 = phys<kColsLog>(base, c);
    if constexpr (vec) {
      const uint4 a = *reinterpret_cast<const uint4*>(GIN ? gm + base : s + phys<kColsLog>(base, 0));
      const uint4 b = *reinterpret_cast<const uint4*>(GIN ? gm + base + 4 : s + phys<kColsLog>(base + 4, 0));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4 % E] = b.x; v[5 % E] = b.y; v[6 % E] = b.z; v[7 % E] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k)
        v[k] = GIN ? gm[base + k * u] : s[lin ? p0 + k * u * cols : phys<kColsLog>(base + k * u, c)];
    }
#pragma unroll
    for (int qq = 0; qq < RB; ++qq) {
      const int q = kFwd ? RB - 1 - qq : qq;                   // DIF: wide spans first
      const uint32_t h = u << q;
      uint2 w[1 << (RB - 1)];
#pragma unroll
      for (int k = 0; k < (1 << q); ++k) w[k] = tws[h + off + k * u];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << q)) continue;
        const uint32_t a = v[k], b = v[k + (1 << q)];
        const uint2 ww = w[k & ((1 << q) - 1)];
        if (kFwd) {                                            // in, out < 2p
          const uint32_t t = a + b;
          v[k] = t >= 2 * kP ? t - 2 * kP : t;
          v[k + (1 << q)] = shoup(a + 2 * kP - b, ww.x, ww.y);
        } else {                                               // in, out < 4p
          const uint32_t ar = a >= 2 * kP ? a - 2 * kP : a;
          const uint32_t bw = shoup(b, ww.x, ww.y);
          v[k] = ar + bw;
          v[k + (1 << q)] = ar + 2 * kP - bw;
        }
      }
    }
    if constexpr (vec) {
      *reinterpret_cast<uint4*>(GOUT ? gm + base : s + phys<kColsLog>(base, 0)) = make_uint4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<uint4*>(GOUT ? gm + base + 4 : s + phys<kColsLog>(base + 4, 0)) =
          make_uint4(v[4 % E], v[5 % E], v[6 % E], v[7 % E]);
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (GOUT) gm[base + k * u] = v[k];
        else s[lin ? p0 + k * u * cols : phys<kColsLog>(base + k * u, c)] = v[k];
      }
    }
  }
  __syncthreads();
}

// All LOGN stages: rounds of three from the narrow end, the remainder (1 or 2
// stages) at the wide end.  Forward DIF runs wide -> narrow, inverse DIT the reverse.
template <bool kFwd, int CL, int LOGN>
__device__ __forceinline__ void ntt_smem(uint32_t* s, const uint2* tws) {
  constexpr int top = LOGN % 3, nf = LOGN / 3;
  static_assert(nf >= 1 && nf <= 3, "7 <= LOGN <= 11");
  if constexpr (kFwd && top) ntt_round<top, true, CL, LOGN, LOGN - top>(s, tws);
  ntt_round<3, kFwd, CL, LOGN, kFwd ? 3 * (nf - 1) : 0>(s, tws);
  if constexpr (nf >= 2) ntt_round<3, kFwd, CL, LOGN, kFwd ? 3 * (nf - 2) : 3>(s, tws);
  if constexpr (nf >= 3) ntt_round<3, kFwd, CL, LOGN, kFwd ? 3 * (nf - 3) : 6>(s, tws);
  if constexpr (!kFwd && top) ntt_round<top, false, CL, LOGN, LOGN - top>(s, tws);
}

// The same for one row in global memory g: the first round reads g, the last
// writes g (two shared-memory round trips fewer per row).
template <bool kFwd, int LOGN>
__device__ __forceinline__ void ntt_row_g(uint32_t* s, const uint2* tws, uint32_t* g) {
  constexpr int top = LOGN % 3, nf = LOGN / 3;
  static_assert(top != 0 && nf >= 2 && nf <= 3, "LOGN in {7, 8, 10, 11}");
  if constexpr (kFwd) {
    ntt_round<top, true, 0, LOGN, LOGN - top, true, false>(s, tws, g);
    if constexpr (nf == 3) ntt_round<3, true, 0, LOGN, 6>(s, tws);
    ntt_round<3, true, 0, LOGN, 3>(s, tws);
    ntt_round<3, true, 0, LOGN, 0, false, true>(s, tws, g);
  } else {
    ntt_round<3, false, 0, LOGN, 0, true, false>(s, tws, g);
    ntt_round<3, false, 0, LOGN, 3>(s, tws);
    if constexpr (nf == 3) ntt_round<3, false, 0, LOGN, 6>(s, tws);
    ntt_round<top, false, 0, LOGN, LOGN - top, false, true>(s, tws, g);
  }
}

// Stage twiddles of an n-point transform, tws[h + j] = w_N^{j N / 2h}
// (j < h < n), precomputed once per build by ntt_stage_table_kernel (the
// strided gather tw[j N / 2h] would cost a sector per entry in every CTA);
// each CTA copies its table with coalesced loads.
__device__ __forceinline__ void stage_twiddles(const uint2* tab, uint32_t n, uint2* tws) {
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) tws[j] = tab[j];
}

// Four-step twiddle w_N^{k1 col} (Montgomery form) with k1 < R, col < C:
// k1 col = q C + r, w_N^{qC} = w_R^q from the R-point stage table
// (w_R^{R/2} = -1), w_N^r from tlo (Montgomery).
__device__ __forceinline__ uint32_t four_step_tw(uint32_t k1, uint32_t col, uint32_t logC, uint32_t R,
                                                 const uint2* tws, const uint32_t* tlo) {
  const uint32_t e = k1 * col, q = e >> logC, r = e & ((1u << logC) - 1);
  const uint32_t hm = pair_mont(tws[q < R / 2 ? R / 2 + q : q]);
  return mmul(q < R / 2 ? hm : kP - hm, tlo[r]);
}

// Forward column pass (four-step): R-point DIF of 8 adjacent columns in
// shared memory, inputs generated from the packed bits (x_i = +-1 for i < L,
// 0 past L), then the twiddle w_N^{k1 col} for the column spectrum entry
// k1 = brev_R(row) on the way out.
template <int LOGR>
__global__ void __launch_bounds__(256) ntt_col_fwd_kernel(const uint32_t* bits, size_t w_stride,
                                                          uint32_t L, uint32_t R, uint32_t C,
                                                          const uint32_t* tw, const uint2* tabR,
                                                          uint32_t* x) {
  __shared__ __align__(16) uint32_t s[kMaxRows * kCols];
  __shared__ uint2 tws[kMaxRows];
  __shared__ uint32_t tlo[kMaxRowLen];
  const uint32_t walk = blockIdx.y, col0 = blockIdx.x * kCols;
  const uint32_t N = R * C, logR = LOGR, logC = 31 - __clz(C);
  const uint32_t* S = bits + (size_t)walk * w_stride;
  stage_twiddles(tabR, R, tws);
  for (uint32_t j = threadIdx.x; j < C; j += blockDim.x) tlo[j] = tw[j];
  // work items = (row, half row of 4 columns): one bit word, one 16-byte store
  for (uint32_t e = threadIdx.x; e < 2 * R; e += blockDim.x) {
    const uint32_t m = e >> 1, c0 = (e & 1) * 4, i0 = m * C + col0 + c0;   // 4 | i0: one word
    const uint32_t b = i0 < L ? S[i0 >> 5] >> (i0 & 31) : 0u;          // no reads past the bits
    uint32_t v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      v[c] = i0 + c < L ? (((b >> c) & 1u) ? kP - 1u : 1u) : 0u;          // normal form
    *reinterpret_cast<uint4*>(s + phys<3>(m, c0)) = make_uint4(v[0], v[1], v[2], v[3]);
  }
  __syncthreads();
  ntt_smem<true, 3, LOGR>(s, tws);
  uint32_t* X = x + (size_t)walk * N;
  // four-step twiddles w^{k1 col}, col = col0 + c0 .. +3: one lookup, then
  // successive products with w^{k1} (tlo[k1], k1 < R <= C)
  for (uint32_t e = threadIdx.x; e < 2 * R; e += blockDim.x) {
    const uint32_t m = e >> 1, c0 = (e & 1) * 4;
    const uint32_t k1 = __brev(m) >> (32 - logR);
    uint32_t t = four_step_tw(k1, col0 + c0, logC, R, tws, tlo);
    const uint32_t step = tlo[k1];
    const uint4 a = *reinterpret_cast<const uint4*>(s + phys<3>(m, c0));
    uint4 o;
    o.x = mmul(a.x, t); t = mmul(t, step);
    o.y = mmul(a.y, t); t = mmul(t, step);
    o.z = mmul(a.z, t); t = mmul(t, step);
    o.w = mmul(a.w, t);
    *reinterpret_cast<uint4*>(X + m * C + col0 + c0) = o;
  }
}

// Row pass over the rows of every walk: C-point forward DIF or inverse DIT
// (the four-step's row transforms need no cross-row twiddles).
template <bool kForward, int LOGC>
__global__ void __launch_bounds__(256) ntt_row_kernel(uint32_t* x, uint32_t R, uint32_t C,
                                                      const uint2* tabC) {
  __shared__ __align__(16) uint32_t s[kMaxRowLen];
  __shared__ uint2 ts[kMaxRowLen];
  const uint32_t N = R * C;
  stage_twiddles(tabC, C, ts);
  __syncthreads();
  for (uint32_t row = blockIdx.x * kRowsPerCta; row < (blockIdx.x + 1) * kRowsPerCta && row < R; ++row) {
    uint32_t* X = x + (size_t)blockIdx.y * N + (size_t)row * C;
    if constexpr (LOGC % 3 != 0) {
      ntt_row_g<kForward, LOGC>(s, ts, X);
    } else {
      for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) s[phys<0>(i, 0)] = X[i];
      __syncthreads();
      ntt_smem<kForward, 0, LOGC>(s, ts);
      for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) X[i] = s[phys<0>(i, 0)];
      __syncthreads();
    }
  }
}

// Spectrum of the correlation at bit-reversed position p (k = brev(p)):
// Z(k) = X(k) X(N-k) w^{(L-1)k}.  With p = m C + c (k = k1 + R k2, k1 =
// brev_R(m), k2 = brev_C(c)) the partner of a row m != 0 is the row
// m' = brev_R(R - k1) read backwards (c -> C-1-c), so one CTA per row pair
// reads and writes both rows coalesced; row 0 pairs within itself.
__global__ void __launch_bounds__(256) ntt_pointwise_kernel(uint32_t* x, uint32_t logN, uint32_t logR,
                                                            uint32_t L, const uint32_t* tw) {
  const uint32_t N = 1u << logN, R = 1u << logR, logC = logN - logR, C = 1u << logC;
  const uint32_t m = blockIdx.x;
  const uint32_t k1 = m ? __brev(m) >> (32 - logR) : 0u;
  const uint32_t m2 = m ? __brev(R - k1) >> (32 - logR) : 0u;
  if (m2 < m) return;                                        // the partner row's CTA
  uint32_t* X = x + (size_t)blockIdx.y * N;
  for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
    const uint32_t k = ((__brev(c) >> (32 - logC)) << logR) + k1;
    const uint32_t kn = (N - k) & (N - 1);
    uint32_t c2;
    if (m) {
      c2 = C - 1 - c;
      if (m2 == m && c2 < c) continue;                       // self-paired row: lower half does it
    } else {
      c2 = __brev(kn >> logR) >> (32 - logC);
      if (c2 < c) continue;
    }
    const uint32_t p = m * C + c, p2 = m2 * C + c2;
    const uint32_t ab = mmul(X[p], X[p2]);
    const uint32_t e1 = (uint32_t)(((uint64_t)(L - 1) * k) & (N - 1));
    const uint32_t e2 = (uint32_t)(((uint64_t)(L - 1) * kn) & (N - 1));
    X[p] = mmul(ab, wpow(tw, e1, N));
    if (p2 != p) X[p2] = mmul(ab, wpow(tw, e2, N));
  }
}

// Inverse column pass: the inverse four-step twiddle w_N^{-k1 col} on the way
// in, R-point DIT, then C_{L-1-i} = z_i N^-1 (signed) into the pivot / local
// tables, PSL and energy.
template <int LOGR>
__global__ void __launch_bounds__(256) ntt_col_inv_kernel(const uint32_t* x, uint32_t R, uint32_t C,
                                                          const uint32_t* twi, const uint2* tabR,
                                                          uint32_t ninv_m,
                                                          uint32_t L, int32_t* Cp, int32_t* Cl,
                                                          size_t c_stride, WalkState* st) {
  __shared__ __align__(16) uint32_t s[kMaxRows * kCols];
  __shared__ uint2 tws[kMaxRows];
  __shared__ uint32_t tlo[kMaxRowLen];
  const uint32_t walk = blockIdx.y, col0 = blockIdx.x * kCols;
  const uint32_t N = R * C, logR = LOGR, logC = 31 - __clz(C);
  const uint32_t* X = x + (size_t)walk * N;
  stage_twiddles(tabR, R, tws);
  for (uint32_t j = threadIdx.x; j < C; j += blockDim.x) tlo[j] = twi[j];
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < 2 * R; e += blockDim.x) {
    const uint32_t m = e >> 1, c0 = (e & 1) * 4;
    const uint32_t k1 = __brev(m) >> (32 - logR);
    uint32_t t = four_step_tw(k1, col0 + c0, logC, R, tws, tlo);
    const uint32_t step = tlo[k1];
    const uint4 a = *reinterpret_cast<const uint4*>(X + m * C + col0 + c0);   // < 4p (DIT rows)
    auto r2 = [](uint32_t v) { return v >= 2 * kP ? v - 2 * kP : v; };
    uint4 o;
    o.x = mmul(r2(a.x), t); t = mmul(t, step);
    o.y = mmul(r2(a.y), t); t = mmul(t, step);
    o.z = mmul(r2(a.z), t); t = mmul(t, step);
    o.w = mmul(r2(a.w), t);
    *reinterpret_cast<uint4*>(s + phys<3>(m, c0)) = o;
  }
  __syncthreads();
  ntt_smem<false, 3, LOGR>(s, tws);
  int32_t* Cw = Cp + (size_t)walk * c_stride;
  int32_t* Cw2 = Cl ? Cl + (size_t)walk * c_stride : nullptr;
  int32_t pm = 0;
  long long en = 0;
  for (uint32_t e = threadIdx.x; e < R * kCols; e += blockDim.x) {
    const uint32_t m = e / kCols, c = e % kCols, i = m * C + col0 + c;
    if (i >= L) continue;
    // z = N c 2^-32 (the pointwise product's Montgomery factor), < 4p;
    // ninv_m = N^-1 2^64 mod p: mmul(z, ninv_m) = c
    const uint32_t z = s[phys<3>(m, c)];
    const uint32_t v = mmul(z >= 2 * kP ? z - 2 * kP : z, ninv_m);
    const int32_t cv = v > kP / 2 ? (int32_t)v - (int32_t)kP : (int32_t)v;
    const uint32_t k = L - 1 - i;
    Cw[k] = cv;
    if (Cw2) Cw2[k] = cv;
    if (k > 0) {
      pm = max(pm, abs(cv));
      en += (long long)cv * cv;
    }
  }
  for (int o = 16; o; o >>= 1) {
    pm = max(pm, __shfl_xor_sync(0xffffffffu, pm, o));
    en += __shfl_xor_sync(0xffffffffu, en, o);
  }
  if (st && (threadIdx.x & 31) == 0) {
    atomicMax(&st[walk].P, pm);
    atomicAdd(reinterpret_cast<unsigned long long*>(&st[walk].energy_best), (unsigned long long)en);
  }
}

// tab[h + j] = (w, floor(w 2^32 / p)) with w = tw[j N / 2h] in normal form,
// for 1 <= h < n, j < h (tab[0] unused)
__global__ void ntt_stage_table_kernel(const uint32_t* tw, uint32_t N, uint32_t n, uint2* tab) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i == 0) { tab[0] = make_uint2(0, 0); continue; }
    const uint32_t h = 1u << (31 - __clz(i)), j = i - h;
    const uint32_t w = mmul(tw[j * (N / (2 * h))], 1u);
    tab[i] = make_uint2(w, (uint32_t)(((uint64_t)w << 32) / kP));
  }
}

__global__ void ntt_twiddle_kernel(uint32_t* tw, uint32_t half, uint32_t root_m) {
  // tw[j] = root^j (Montgomery), each thread by square-and-multiply
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < half; j += gridDim.x * blockDim.x) {
    uint32_t r = kOne, b = root_m, e = j;
    while (e) {
      if (e & 1u) r = mmul(r, b);
      b = mmul(b, b);
      e >>= 1;
    }
    tw[j] = r;
  }
}

uint32_t host_pow(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  b %= kP;
  while (e) {
    if (e & 1) r = r * b % kP;
    b = b * b % kP;
    e >>= 1;
  }
  return (uint32_t)r;
}
uint32_t to_mont(uint32_t x) { return (uint32_t)(((uint64_t)x << 32) % kP); }

}  // namespace

// Builds C for n_walks walks (bits padded as in RunArgs, word i at bits[i+1]).
// Scratch: n_walks * N uint32 + 2 * N/2 twiddles.  Returns launches or -1.
int launch_build_tables_ntt(const RunArgs& a, uint32_t n_walks, cudaStream_t s) {
  const uint32_t L = a.L;
  uint32_t logN = 1;
  while ((1u << logN) < 2 * L) ++logN;
  const uint32_t N = 1u << logN;
  const uint32_t logR = logN / 2, R = 1u << logR, C = N >> logR;   // R <= C <= 2R
  if (R > (uint32_t)kMaxRows || C > (uint32_t)kMaxRowLen || C < (uint32_t)kCols)
    return launch_fail(cudaErrorInvalidValue);
  uint32_t *x = nullptr, *tw = nullptr;
  cudaError_t e = cudaMallocAsync(&x, (size_t)n_walks * N * 4, s);
  if (e != cudaSuccess) return launch_fail(e);
  if ((e = cudaMallocAsync(&tw, (size_t)(N + 4 * R + 4 * C) * 4, s)) != cudaSuccess) {
    cudaFreeAsync(x, s);
    return launch_fail(e);
  }
  uint32_t* twi = tw + N / 2;
  uint2* tabR = reinterpret_cast<uint2*>(tw + N);
  uint2 *tabRi = tabR + R, *tabC = tabRi + R, *tabCi = tabC + C;
  int launches = 0;
  const uint32_t root = host_pow(3, (kP - 1) / N);          // primitive N-th root
  const uint32_t iroot = host_pow(root, kP - 2);
  ntt_twiddle_kernel<<<(N / 2 + 255) / 256, 256, 0, s>>>(tw, N / 2, to_mont(root));
  ntt_twiddle_kernel<<<(N / 2 + 255) / 256, 256, 0, s>>>(twi, N / 2, to_mont(iroot));
  ntt_stage_table_kernel<<<(R + 255) / 256, 256, 0, s>>>(tw, N, R, tabR);
  ntt_stage_table_kernel<<<(R + 255) / 256, 256, 0, s>>>(twi, N, R, tabRi);
  ntt_stage_table_kernel<<<(C + 255) / 256, 256, 0, s>>>(tw, N, C, tabC);
  ntt_stage_table_kernel<<<(C + 255) / 256, 256, 0, s>>>(twi, N, C, tabCi);
  const dim3 gcol(C / kCols, n_walks), grow((R + kRowsPerCta - 1) / kRowsPerCta, n_walks);
  const uint32_t ninv = host_pow(N, kP - 2), ninv_m = to_mont(to_mont(ninv));
  const uint32_t* bits = a.bits_piv + a.w_front + 1;
  switch (logR) {
#define COL_FWD(LR) case LR: ntt_col_fwd_kernel<LR><<<gcol, kNttThreads, 0, s>>>(bits, a.w_stride, L, R, C, tw, tabR, x); break;
    COL_FWD(7) COL_FWD(8) COL_FWD(9) COL_FWD(10)
#undef COL_FWD
    default: cudaFreeAsync(x, s); cudaFreeAsync(tw, s); return launch_fail(cudaErrorInvalidValue);
  }
  const uint32_t logC = logN - logR;
  switch (logC) {
#define ROW(LC, F, T) case LC: ntt_row_kernel<F, LC><<<grow, kNttThreads, 0, s>>>(x, R, C, T); break;
    ROW(7, true, tabC) ROW(8, true, tabC) ROW(9, true, tabC) ROW(10, true, tabC) ROW(11, true, tabC)
    default: cudaFreeAsync(x, s); cudaFreeAsync(tw, s); return launch_fail(cudaErrorInvalidValue);
  }
  ntt_pointwise_kernel<<<dim3(R, n_walks), 256, 0, s>>>(x, logN, logR, L, tw);
  switch (logC) {
    ROW(7, false, tabCi) ROW(8, false, tabCi) ROW(9, false, tabCi) ROW(10, false, tabCi) ROW(11, false, tabCi)
#undef ROW
    default: cudaFreeAsync(x, s); cudaFreeAsync(tw, s); return launch_fail(cudaErrorInvalidValue);
  }
  switch (logR) {
#define COL_INV(LR) case LR: ntt_col_inv_kernel<LR><<<gcol, kNttThreads, 0, s>>>(x, R, C, twi, tabRi, ninv_m, L, a.Cpiv, a.Cloc, a.c_stride, a.st); break;
    COL_INV(7) COL_INV(8) COL_INV(9) COL_INV(10)
#undef COL_INV
    default: cudaFreeAsync(x, s); cudaFreeAsync(tw, s); return launch_fail(cudaErrorInvalidValue);
  }
  launches += 11;
  cudaFreeAsync(x, s);
  cudaFreeAsync(tw, s);
  return launch_status(launches);
}

}  // namespace pslb
