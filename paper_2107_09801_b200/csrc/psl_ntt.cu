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
// Layout: each walk's N values as R rows x C columns (i = m C + col, R C = N).
// Forward DIF (natural -> bit-reversed):  stages with span h >= C pair
// elements of one column (column pass: a CTA holds 8 adjacent columns in
// shared memory, generated straight from the packed bits), stages h < C pair
// elements of one row (row pass: a CTA holds a row).  Pointwise product on the
// bit-reversed spectrum.  Inverse DIT (bit-reversed -> natural): row pass,
// then the column pass, which also scales by N^-1, writes C_k (pivot and local
// tables) and reduces the walk's PSL and energy.  Four passes over HBM instead
// of one per radix-2 stage.
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
// w^e for any e (mod N) from the half table tw[j] = w^j, j < N/2 (w^{N/2} = -1)
__device__ __forceinline__ uint32_t wpow(const uint32_t* tw, uint32_t e, uint32_t N) {
  e &= N - 1;
  const uint32_t h = N >> 1;
  return e < h ? tw[e] : (kP - tw[e - h]) % kP;
}

// Twiddle factors of the column stages for the CTA's 8 columns: stage st
// (hr = R/2 >> st, span h = hr C) needs w^{(jr C + col) N / 2h}
// = w^{jr N / 2hr} * w^{col N / 2h}: rf[hr + jr] and cf[st][c] (Montgomery;
// the product costs one extra mmul per butterfly instead of a scattered load).
__device__ __forceinline__ void col_twiddles(const uint32_t* tw, uint32_t R, uint32_t C, uint32_t col0,
                                             uint32_t* rf, uint32_t* cf) {
  const uint32_t N = R * C;
  for (uint32_t hr = 1; hr < R; hr <<= 1)
    for (uint32_t jr = threadIdx.x; jr < hr; jr += blockDim.x) rf[hr + jr] = tw[jr * (N / (2 * hr))];
  uint32_t st = 0;
  for (uint32_t hr = R >> 1; hr >= 1; hr >>= 1, ++st)
    if (threadIdx.x < (uint32_t)kCols) {
      const uint32_t col = col0 + threadIdx.x;
      // col N / 2h = col R / 2hr * (N / (R C)) ... as an index into tw: col * (N / (2 hr C))
      const uint32_t e = col * (N / (2 * hr * C));
      cf[st * kCols + threadIdx.x] = (N / (2 * hr * C)) ? tw[e] : 0u;
    }
  __syncthreads();
}

// Forward column pass: stages h = N/2 .. C (rows span R/2 .. 1), DIF.  The
// inputs are generated from the packed bits (x_i = +-1 for i < L, 0 past L).
__global__ void __launch_bounds__(256) ntt_col_fwd_kernel(const uint32_t* bits, size_t w_stride,
                                                          uint32_t L, uint32_t R, uint32_t C,
                                                          const uint32_t* tw, uint32_t* x) {
  __shared__ uint32_t s[kMaxRows * kCols];
  __shared__ uint32_t rf[kMaxRows];                          // rf[hr + jr] = w^{jr N / 2hr}
  __shared__ uint32_t cf[11 * kCols];                        // cf[stage][c] = w^{col N / (2 hr C)}
  const uint32_t walk = blockIdx.y, col0 = blockIdx.x * kCols;
  const uint32_t N = R * C;
  const uint32_t* S = bits + (size_t)walk * w_stride;
  col_twiddles(tw, R, C, col0, rf, cf);
  for (uint32_t e = threadIdx.x; e < R * kCols; e += blockDim.x) {
    const uint32_t m = e / kCols, c = e % kCols, i = m * C + col0 + c;
    uint32_t v = 0;
    if (i < L) v = ((S[i >> 5] >> (i & 31)) & 1u) ? kP - kOne : kOne;
    s[e] = v;
  }
  __syncthreads();
  for (uint32_t hr = R >> 1, st = 0; hr >= 1; hr >>= 1, ++st) {
    for (uint32_t b = threadIdx.x; b < (R / 2) * kCols; b += blockDim.x) {
      const uint32_t c = b % kCols, q = b / kCols;          // q-th butterfly row pair
      const uint32_t jr = q & (hr - 1), m1 = ((q - jr) << 1) + jr, m2 = m1 + hr;
      // position j = jr C + col within the 2h block: w^{j N / 2h} = rf * cf
      const uint32_t w = mmul(rf[hr + jr], cf[st * kCols + c]);
      const uint32_t u = s[m1 * kCols + c], v = s[m2 * kCols + c];
      s[m1 * kCols + c] = madd(u, v);
      s[m2 * kCols + c] = mmul(msub(u, v), w);
    }
    __syncthreads();
  }
  uint32_t* X = x + (size_t)walk * N;
  for (uint32_t e = threadIdx.x; e < R * kCols; e += blockDim.x) {
    const uint32_t m = e / kCols, c = e % kCols;
    X[m * C + col0 + c] = s[e];
  }
}

// Row pass over the rows of every walk: forward DIF stages h = C/2 .. 1 or
// inverse DIT stages h = 1 .. C/2.  Twiddles of the row stages (the same for
// every row) staged in shared memory: stage h uses tw[j N / 2h], j < h.
template <bool kForward>
__global__ void __launch_bounds__(256) ntt_row_kernel(uint32_t* x, uint32_t R, uint32_t C,
                                                      const uint32_t* tw) {
  __shared__ uint32_t s[kMaxRowLen];
  __shared__ uint32_t ts[kMaxRowLen];                         // ts[h + j] = stage-h twiddle j
  const uint32_t N = R * C;
  for (uint32_t h = 1; h < C; h <<= 1)
    for (uint32_t j = threadIdx.x; j < h; j += blockDim.x) ts[h + j] = tw[j * (N / (2 * h))];
  uint32_t* X = x + (size_t)blockIdx.y * N + (size_t)blockIdx.x * C;
  for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) s[i] = X[i];
  __syncthreads();
  for (uint32_t it = 0, h = kForward ? C >> 1 : 1; h >= 1 && h < C; ++it, h = kForward ? h >> 1 : h << 1) {
    for (uint32_t b = threadIdx.x; b < C / 2; b += blockDim.x) {
      const uint32_t j = b & (h - 1), i1 = ((b - j) << 1) + j, i2 = i1 + h;
      const uint32_t w = ts[h + j], u = s[i1], v = s[i2];
      if (kForward) {
        s[i1] = madd(u, v);
        s[i2] = mmul(msub(u, v), w);
      } else {
        const uint32_t vw = mmul(v, w);
        s[i1] = madd(u, vw);
        s[i2] = msub(u, vw);
      }
    }
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) X[i] = s[i];
}

// Spectrum of the correlation at bit-reversed position p (k = brev(p)):
// Z(k) = X(k) X(N-k) w^{(L-1)k}.  Pairs (p, p') are updated by the lower of the two.
__global__ void ntt_pointwise_kernel(uint32_t* x, uint32_t logN, uint32_t L, const uint32_t* tw) {
  const uint32_t N = 1u << logN;
  uint32_t* X = x + (size_t)blockIdx.y * N;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    const uint32_t k = __brev(p) >> (32 - logN);
    const uint32_t kn = (N - k) & (N - 1);
    const uint32_t p2 = __brev(kn) >> (32 - logN);
    if (p2 < p) continue;                                    // done by the partner
    const uint32_t a = X[p], b = X[p2];
    const uint32_t ab = mmul(a, b);
    const uint32_t e1 = (uint32_t)(((uint64_t)(L - 1) * k) & (N - 1));
    const uint32_t e2 = (uint32_t)(((uint64_t)(L - 1) * kn) & (N - 1));
    X[p] = mmul(ab, wpow(tw, e1, N));
    if (p2 != p) X[p2] = mmul(ab, wpow(tw, e2, N));
  }
}

// Inverse column pass: DIT stages h = C .. N/2 (rows span 1 .. R/2), then
// C_{L-1-i} = z_i N^-1 (signed) into the pivot / local tables, PSL and energy.
__global__ void __launch_bounds__(256) ntt_col_inv_kernel(const uint32_t* x, uint32_t R, uint32_t C,
                                                          const uint32_t* twi, uint32_t ninv_m,
                                                          uint32_t L, int32_t* Cp, int32_t* Cl,
                                                          size_t c_stride, WalkState* st) {
  __shared__ uint32_t s[kMaxRows * kCols];
  __shared__ uint32_t rf[kMaxRows];
  __shared__ uint32_t cf[11 * kCols];
  const uint32_t walk = blockIdx.y, col0 = blockIdx.x * kCols;
  const uint32_t N = R * C;
  const uint32_t* X = x + (size_t)walk * N;
  col_twiddles(twi, R, C, col0, rf, cf);
  for (uint32_t e = threadIdx.x; e < R * kCols; e += blockDim.x) {
    const uint32_t m = e / kCols, c = e % kCols;
    s[e] = X[m * C + col0 + c];
  }
  __syncthreads();
  uint32_t sg = 0;
  for (uint32_t hr = R >> 1; hr >= 1; hr >>= 1) ++sg;       // stage index of hr = 1 in col_twiddles order
  for (uint32_t hr = 1; hr < R; hr <<= 1) {
    --sg;
    for (uint32_t b = threadIdx.x; b < (R / 2) * kCols; b += blockDim.x) {
      const uint32_t c = b % kCols, q = b / kCols;
      const uint32_t jr = q & (hr - 1), m1 = ((q - jr) << 1) + jr, m2 = m1 + hr;
      const uint32_t w = mmul(rf[hr + jr], cf[sg * kCols + c]);
      const uint32_t u = s[m1 * kCols + c], vw = mmul(s[m2 * kCols + c], w);
      s[m1 * kCols + c] = madd(u, vw);
      s[m2 * kCols + c] = msub(u, vw);
    }
    __syncthreads();
  }
  int32_t* Cw = Cp + (size_t)walk * c_stride;
  int32_t* Cw2 = Cl ? Cl + (size_t)walk * c_stride : nullptr;
  int32_t pm = 0;
  long long en = 0;
  for (uint32_t e = threadIdx.x; e < R * kCols; e += blockDim.x) {
    const uint32_t m = e / kCols, c = e % kCols, i = m * C + col0 + c;
    if (i >= L) continue;
    // z holds N c R (Montgomery); mmul(., N^-1 R) = c R; mmul(., 1) = c
    const uint32_t v = mmul(mmul(s[e], ninv_m), 1u);
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
  if (R > (uint32_t)kMaxRows || C > (uint32_t)kMaxRowLen || C < (uint32_t)kCols) return -1;
  uint32_t *x = nullptr, *tw = nullptr;
  if (cudaMallocAsync(&x, (size_t)n_walks * N * 4, s) != cudaSuccess) return -1;
  if (cudaMallocAsync(&tw, (size_t)N * 4, s) != cudaSuccess) return -1;
  uint32_t* twi = tw + N / 2;
  int launches = 0;
  const uint32_t root = host_pow(3, (kP - 1) / N);          // primitive N-th root
  const uint32_t iroot = host_pow(root, kP - 2);
  ntt_twiddle_kernel<<<(N / 2 + 255) / 256, 256, 0, s>>>(tw, N / 2, to_mont(root));
  ntt_twiddle_kernel<<<(N / 2 + 255) / 256, 256, 0, s>>>(twi, N / 2, to_mont(iroot));
  const dim3 gcol(C / kCols, n_walks), grow(R, n_walks);
  ntt_col_fwd_kernel<<<gcol, 256, 0, s>>>(a.bits_piv + a.w_front + 1, a.w_stride, L, R, C, tw, x);
  ntt_row_kernel<true><<<grow, 256, 0, s>>>(x, R, C, tw);
  ntt_pointwise_kernel<<<dim3(std::min<uint32_t>(N / 256, 1024), n_walks), 256, 0, s>>>(x, logN, L, tw);
  ntt_row_kernel<false><<<grow, 256, 0, s>>>(x, R, C, twi);
  const uint32_t ninv = host_pow(N, kP - 2);
  ntt_col_inv_kernel<<<gcol, 256, 0, s>>>(x, R, C, twi, to_mont(ninv), L, a.Cpiv, a.Cloc, a.c_stride,
                                           a.st);
  launches += 7;
  cudaFreeAsync(x, s);
  cudaFreeAsync(tw, s);
  return cudaGetLastError() == cudaSuccess ? launches : -1;
}

}  // namespace pslb
