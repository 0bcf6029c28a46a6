// psl_ntt.cu -- SidelobeTable::build (sequence.cpp:46-60) for many walks by an
// exact number-theoretic transform.
//
// C_k = sum_i s_i s_{i+k} is the correlation of the +-1 sequence with itself:
// C_k = (s * rev(s))[L-1-k].  Over Z_p with p = 998244353 = 119 * 2^23 + 1
// (3 is a primitive root) the cyclic convolution of length N = 2^ceil(log2(2L))
// is exact, and |C_k| <= L < p/2 recovers the signed value.  O(L log L) per
// walk instead of the O(L^2) popcount kernel (which stays for small L and the
// single-table C-ABI call).  Forward DIF (natural -> bit-reversed), pointwise
// product, inverse DIT (bit-reversed -> natural): no permutation pass.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "psl_internal.h"

namespace pslb {
namespace {

constexpr uint32_t kP = 998244353u;
constexpr uint32_t kPinv = 998244351u;   // -p^{-1} mod 2^32 (Montgomery)

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

// +-1 -> Montgomery form of +1 / -1; x natural order, y reversed.
__global__ void ntt_load_kernel(const uint32_t* bits, size_t w_stride, uint32_t L, uint32_t N,
                                uint32_t* x, uint32_t* y) {
  const uint32_t walk = blockIdx.y;
  const uint32_t* S = bits + (size_t)walk * w_stride;
  uint32_t* X = x + (size_t)walk * N;
  uint32_t* Y = y + (size_t)walk * N;
  const uint32_t one = 301989884u;            // 2^32 mod p  (Montgomery 1)
  const uint32_t mone = kP - one;             // Montgomery -1
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    uint32_t vx = 0, vy = 0;
    if (i < L) {
      vx = ((S[i >> 5] >> (i & 31)) & 1u) ? mone : one;
      const uint32_t r = L - 1 - i;
      vy = ((S[r >> 5] >> (r & 31)) & 1u) ? mone : one;
    }
    X[i] = vx;
    Y[i] = vy;
  }
}

// One radix-2 stage over all walks.  tw[j] = w_N^j (Montgomery), j < N/2.
template <bool kForward>
__global__ void ntt_stage_kernel(uint32_t* a, uint32_t N, uint32_t h, const uint32_t* tw,
                                 uint32_t walks_per_arr) {
  const uint32_t arr = blockIdx.y;
  uint32_t* A = a + (size_t)arr * N;
  const uint32_t stride = N / (2 * h);
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < N / 2; t += gridDim.x * blockDim.x) {
    const uint32_t j = t & (h - 1);
    const uint32_t i1 = ((t - j) << 1) + j;
    const uint32_t i2 = i1 + h;
    const uint32_t w = tw[j * stride];
    const uint32_t u = A[i1], v = A[i2];
    if (kForward) {            // DIF: (u+v, (u-v) w)
      A[i1] = madd(u, v);
      A[i2] = mmul(msub(u, v), w);
    } else {                   // DIT: (u + v w, u - v w)
      const uint32_t vw = mmul(v, w);
      A[i1] = madd(u, vw);
      A[i2] = msub(u, vw);
    }
  }
  (void)walks_per_arr;
}

__global__ void ntt_pointwise_kernel(uint32_t* x, const uint32_t* y, size_t total) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x)
    x[i] = mmul(x[i], y[i]);
}

// z = INTT output (times N, Montgomery): C_k = z[L-1-k] * N^-1, signed.
__global__ void ntt_extract_kernel(const uint32_t* z, uint32_t N, uint32_t ninv_m, uint32_t L,
                                   int32_t* C, int32_t* Cloc, size_t c_stride, WalkState* st) {
  const uint32_t walk = blockIdx.y;
  const uint32_t* Z = z + (size_t)walk * N;
  int32_t* Cw = C + (size_t)walk * c_stride;
  int32_t* Cl = Cloc ? Cloc + (size_t)walk * c_stride : nullptr;
  int32_t pm = 0;
  long long en = 0;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < L; k += gridDim.x * blockDim.x) {
    // mmul(v, ninv_m) with ninv_m = N^-1 * 2^64 mod p... see host: result in normal form
    uint32_t v = mmul(mmul(Z[L - 1 - k], ninv_m), 1u);
    const int32_t cv = v > kP / 2 ? (int32_t)v - (int32_t)kP : (int32_t)v;
    Cw[k] = cv;
    if (Cl) Cl[k] = cv;
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
  // tw[j] = root^j, computed per block by powering (each thread: square-and-multiply)
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < half; j += gridDim.x * blockDim.x) {
    const uint32_t one = 301989884u;
    uint32_t r = one, b = root_m, e = j;
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
// Scratch: 2 * n_walks * N uint32 + N/2 twiddles.  Returns launches or -1.
int launch_build_tables_ntt(const RunArgs& a, uint32_t n_walks, cudaStream_t s) {
  const uint32_t L = a.L;
  uint32_t N = 1;
  while (N < 2 * L) N <<= 1;
  uint32_t *x = nullptr, *y = nullptr, *tw = nullptr, *twi = nullptr;
  const size_t total = (size_t)n_walks * N;
  if (cudaMallocAsync(&x, 2 * total * 4, s) != cudaSuccess) return -1;
  y = x + total;                              // [x arrays | y arrays]
  if (cudaMallocAsync(&tw, (size_t)N / 2 * 4, s) != cudaSuccess) return -1;
  if (cudaMallocAsync(&twi, (size_t)N / 2 * 4, s) != cudaSuccess) return -1;
  int launches = 0;
  const uint32_t root = host_pow(3, (kP - 1) / N);          // primitive N-th root
  const uint32_t iroot = host_pow(root, kP - 2);
  ntt_twiddle_kernel<<<(N / 2 + 255) / 256, 256, 0, s>>>(tw, N / 2, to_mont(root));
  ntt_twiddle_kernel<<<(N / 2 + 255) / 256, 256, 0, s>>>(twi, N / 2, to_mont(iroot));
  launches += 2;
  const dim3 gl(std::min<uint32_t>((N + 255) / 256, 256), n_walks);
  ntt_load_kernel<<<gl, 256, 0, s>>>(a.bits_piv + a.w_front + 1, a.w_stride, L, N, x, y);
  launches += 1;
  const uint32_t bx = std::min<uint32_t>((N / 2 + 255) / 256, 1024);
  for (uint32_t h = N / 2; h >= 1; h >>= 1) {
    ntt_stage_kernel<true><<<dim3(bx, 2 * n_walks), 256, 0, s>>>(x, N, h, tw, n_walks);
    launches += 1;
    if (h == 1) break;
  }
  ntt_pointwise_kernel<<<4096, 256, 0, s>>>(x, y, total);
  launches += 1;
  for (uint32_t h = 1; h <= N / 2; h <<= 1) {
    ntt_stage_kernel<false><<<dim3(bx, n_walks), 256, 0, s>>>(x, N, h, twi, n_walks);
    launches += 1;
  }
  // N^-1 in Montgomery-domain factor: z holds N*c (Montgomery form, i.e. N*c*R).
  // mmul(zM, ninvM) = N*c*R * Ninv*R / R = c*R ; mmul(., 1) = c.
  const uint32_t ninv = host_pow(N, kP - 2);
  ntt_extract_kernel<<<dim3(std::min<uint32_t>((L + 255) / 256, 256), n_walks), 256, 0, s>>>(
      x, N, to_mont(ninv), L, a.Cpiv, a.Cloc, a.c_stride, a.st);
  launches += 1;
  cudaFreeAsync(x, s);
  cudaFreeAsync(tw, s);
  cudaFreeAsync(twi, s);
  return cudaGetLastError() == cudaSuccess ? launches : -1;
}

}  // namespace pslb
