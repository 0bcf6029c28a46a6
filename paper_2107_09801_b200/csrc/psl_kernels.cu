// psl_kernels.cu -- sm_100a kernels for the two-phase low-PSL search hot path.
//
// Reference path (/root/reference/proj): detail::eval_flip (sequence.hpp:126-162)
// called n_lmt times per step by scan_chunk/ScanPool (search.cpp:156-260),
// reduce_scan (search.cpp:271-292), apply_flip (sequence.cpp:198-224) and the
// run_search step loop (search.cpp:327-430).
//
// B200 design (DESIGN.md has the full derivation):
//  * one persistent CTA per walk (the exact sweep: 256 threads, two CTAs per
//    SM; the certified scan, psl_cert.cuh: 512 threads, one per SM).  The whole
//    step loop -- scan, argmin/PSL reduction, move, snapshots, restarts, RNG,
//    events -- stays on device.
//  * C_k lives in HBM/L2 and is streamed through shared memory in chunks of
//    512 shifts.  While streaming, the builder threads fold the previous
//    step's accepted flip(s) into C (the O(L) apply_flip is fused into the
//    next sweep); the exact sweep expands every C_k into a 64-byte record of
//    the five possible terms |C_k + d|^alpha, d in {-4,-2,0,+2,+4}.
//  * exact sweep: every neighbour's fitness is the reference's serial
//    ascending-k double chain (one DADD per cell, RN, no reassociation), so
//    values are bit-identical; each thread owns 4 adjacent neighbours and per
//    32-shift block turns two sequence-bit windows into term selections.
//  * certified scan (the default): per-row intervals from tcgen05 / mma.sync
//    correlations that provably hold the serial doubles; undecided steps go
//    to the exact sweep (decision-exact records).
//  * the pivot is bit-packed in global memory (L1-resident; bit = 1 <-> -1)
//    with zero pads so sliding windows run off either end unclamped.
//  * neighbour PSL is exact but not computed per cell: only shifts with
//    |C_k| >= PSL(pivot) - 8 can hold a neighbour's peak, and those are
//    collected while streaming.
#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#include "psl_internal.h"

namespace pslb {

namespace {

constexpr uint32_t FULL = 0xffffffffu;

// Device bounds checks (-DPSL_DEBUG_BOUNDS; tools/ablate.sh bounds=PSL_DEBUG_BOUNDS):
// every shared-memory buffer write of the certified pipeline, every C / high-
// sidelobe / scratch index and every padded bit-array word index is tested;
// a violation prints its site and traps.  The stand-in for compute-sanitizer
// memcheck, which this GPU pool does not allow (profiles/r02_bounds_check.md).
#ifdef PSL_DEBUG_BOUNDS
}  // namespace
}  // namespace pslb
#include <cstdio>
namespace pslb {
namespace {
#define PSL_CHK(cond, site)                                                                  \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("PSL bounds violation: site %d block %d thread %d\n", (int)(site), (int)blockIdx.x, \
             (int)threadIdx.x);                                                              \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define PSL_CHK(cond, site) do {} while (0)
#endif
// valid word indices of a walk's padded bit array around sb (sb[0] = the last
// front pad word; nw + 47 pad words before it, nw + 48 + kBitsPad after the
// sequence): [-(nw + 47), 2 nw + 57)
__device__ __forceinline__ bool sb_ok(long long idx, uint32_t L) {
  const long long nw = ((long long)L + 31) / 32;
  return idx >= -(nw + 47) && idx < 2 * nw + 49 + kBitsPad;
}
__device__ __forceinline__ bool in_buf(const void* p, const void* base, size_t bytes, size_t len = 1) {
  const char* q = static_cast<const char*>(p);
  const char* b = static_cast<const char*>(base);
  return q >= b && q + len <= b + bytes;
}

// ------------------------------------------------------------ primitives

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// rng.hpp:20-30
__device__ __forceinline__ void rng_seed(uint64_t* s, uint64_t seed) {
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) {
    z += 0x9e3779b97f4a7c15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    s[i] = x ^ (x >> 31);
  }
}

// rng.hpp:32-42
__device__ __forceinline__ uint64_t rng_next(uint64_t* s) {
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

// The state transition of rng_next alone: linear over GF(2) (xors, shifts, a rotation).
__device__ __forceinline__ void rng_step(uint64_t* s) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
}

// rng.hpp:46-52
__device__ __forceinline__ uint64_t rng_bounded(uint64_t* s, uint64_t n) {
  const uint64_t mask = (n <= 1) ? 0ull : (~0ull >> __clzll((long long)(n - 1)));
  for (;;) {
    const uint64_t v = rng_next(s) & mask;
    if (v < n) return v;
  }
}

// sequence.cpp:95-105 -- same factor order, IEEE round-to-nearest multiplies.
__device__ __forceinline__ double pow_int_dev(double base, uint32_t e) {
  double result = 1.0, factor = base;
  while (e != 0) {
    if (e & 1u) result = __dmul_rn(result, factor);
    e >>= 1;
    if (e != 0) factor = __dmul_rn(factor, factor);
  }
  return result;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// bits 0..15 / 16..31 of x to the even bit positions of a 32-bit word
__device__ __forceinline__ uint32_t spread_lo(uint32_t x) {
  x = __byte_perm(x, 0u, 0x4140);
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}
__device__ __forceinline__ uint32_t spread_hi(uint32_t x) {
  x = __byte_perm(x, 0u, 0x4342);
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// sequence value at position x (0 <= x < L) from the padded smem bit array
__device__ __forceinline__ int sval(const uint32_t* sb, uint32_t x) {
  return 1 - 2 * (int)((sb[(x >> 5) + 1] >> (x & 31)) & 1u);
}

// padded word fetch; word index w may run past either end (reads a zero pad)
__device__ __forceinline__ uint32_t sword(const uint32_t* sb, int w, int nwords) {
  w = max(-1, min(w, nwords));
  return sb[w + 1];
}
// (v & mask) | base as one LOP3 (the compiler would turn a disjoint OR into
// an extra add)
__device__ __forceinline__ uint32_t and_or(uint32_t v, uint32_t mask, uint32_t base) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(v), "r"(mask), "r"(base));
  return r;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// ------------------------------------------------------------ shared layout

struct Ctl {
  WalkState st;
  double rv[32];
  uint32_t ri[32];
  int32_t rp[32];
  uint32_t rpi[32];
  int32_t rbad[32];
  int32_t rmax[32];
  long long re[32];
  double best_v, fit, cv;
  uint32_t best_i, best_pi, ci, cpi;
  int32_t best_psl, bad, cp, cbad;
  uint32_t start, jstar, ppos;
  int32_t do_scan, need_pass, imp, improve, restart;
  uint32_t hcount, hf_count, steps_this_launch;
  int32_t P_new;
  long long energy;
  // certified scan (psl_cert.cuh)
  int32_t cert, need_exact, need_vl, cmp, cv_exact, c_qH, c_qR, c_ovf;
  double cv_lo, cv_hi, gv_lo, gv_hi;
  double c_scaleH, c_unitH, c_scaleR, c_unitR, c_sconst, c_errconst;
  uint32_t m_lo, m_hi, M_lo, M_hi;
  double rs5[5][16];
  uint32_t cfw[72], crv[72]; // per-chunk tcgen05 flags of the pass segment (bit c: fwd / rev MMAs)
  uint64_t mbar[2];          // tcgen05 commit barriers (iteration parity)
  uint64_t cbar[3];          // bulk-copy barriers of the certified C ring (one per slot)
  uint32_t tmem;             // TMEM base of this CTA's accumulators (kTmemCols columns)
  // certificate check mode (RunArgs::cert_check)
  int32_t chk_on, chk_dec, chk_cmp;
  uint32_t chk_ci, chk_rows, chk_viol;
  unsigned long long chk_tight, chk_relw;   // non-negative doubles as bit patterns (atomicMax)
};

constexpr size_t kTabBytes = 2ull * kChunk * kRecDoubles * sizeof(double);
constexpr size_t kTailBytes = 2ull * kChunk * sizeof(double);
constexpr size_t kHfBytes = (size_t)kHCap * sizeof(int2);
constexpr size_t kCtlBytes = (sizeof(Ctl) + 15) & ~size_t(15);
// the exact sweep's records and the certified scan's buffers share one region
// (psl_cert.cuh: 4 digit rows + 4 window copies + 2 record buffers)
constexpr size_t kCertRegion = 2ull * 256 * 128 + 2ull * (2 * 82 * 128) + 2ull * 8 * (512 + 16) + 48 +
                                 4ull * 4 * 1568 + 2ull * 512 * 4 + 3ull * 512 * 4;
constexpr size_t kExactMain = kTabBytes + kTailBytes;

struct Smem {
  double* tab;     // [2][kChunk][8]
  double* tail;    // [2][kChunk]
  int2* hf;        // [kHCap]
  Ctl* ctl;
  const uint32_t* sb;  // the walk's bit-packed pivot in global memory (L1-cached):
                       // sb[0] zero pad, word i at sb[i+1], zero pads after
};

template <bool kCert = false>
__device__ __forceinline__ Smem carve(unsigned char* base) {
  // the exact sweep's records and (certified kernel) the certified scan's
  // buffers share the first region
  constexpr size_t main_bytes = kCert ? (kExactMain > kCertRegion ? kExactMain : kCertRegion) : kExactMain;
  Smem m;
  m.tab = reinterpret_cast<double*>(base);
  m.tail = reinterpret_cast<double*>(base + kTabBytes);
  m.hf = reinterpret_cast<int2*>(base + main_bytes);
  m.ctl = reinterpret_cast<Ctl*>(base + main_bytes + kHfBytes);
  m.sb = nullptr;
  return m;
}

// ------------------------------------------------------------ the sweep

struct SweepIO {
  uint32_t L, nwords, nchunks;
  const int32_t* Csrc;
  int32_t* Cdst;             // nullptr: do not write C back
  int32_t* Cloc;             // nullptr: no local-snapshot copy
  const uint32_t* flips;     // pending flips folded into C while streaming
  uint32_t F;
  uint32_t alpha;            // terms = pow_int(a, alpha) ...
  const double* lut;         // ... or lut[a] when non-null (ScanJob mode)
  uint32_t lut_size;
  int2* hlist;               // nullptr: no high-sidelobe collection
  uint32_t* hcount;          // smem counter
  int32_t hthr;
  bool scan;                 // score neighbours
  bool chain;                // thread 0 runs the pivot fitness chain
};

// apply_flip (sequence.cpp:198-224) folded into one C_k, for F pending flips
// applied in order.  sb holds the sequence AFTER all of them.
__device__ __forceinline__ int32_t fold_flips(int32_t cv, uint32_t k, const SweepIO& io,
                                              const uint32_t* sb) {
  for (uint32_t i = 0; i < io.F; ++i) {
    const uint32_t f = io.flips[i];
    int acc = 0;
    if (k <= f) {
      const uint32_t x = f - k;
      int s = sval(sb, x);
      for (uint32_t m = i + 1; m < io.F; ++m) s = (io.flips[m] == x) ? -s : s;
      acc += s;
    }
    if (f + k < io.L) {
      const uint32_t x = f + k;
      int s = sval(sb, x);
      for (uint32_t m = i + 1; m < io.F; ++m) s = (io.flips[m] == x) ? -s : s;
      acc += s;
    }
    const int sf = -sval(sb, f);  // value of s_f before flip i
    cv += -2 * sf * acc;
  }
  return cv;
}

__device__ __forceinline__ double term(const SweepIO& io, int32_t a) {
  if (io.lut) return (uint32_t)a < io.lut_size ? io.lut[a] : 0.0;
  return pow_int_dev((double)a, io.alpha);
}

// Expand chunk c of C into the per-k term records (kChunk records, the CTA's
// threads take kChunk / kThreads each).
__device__ __forceinline__ void build_chunk(const SweepIO& io, uint32_t c, double* tab,
                                            double* tail, const uint32_t* sb, int32_t& pmax) {
#pragma unroll 1
  for (uint32_t r = threadIdx.x; r < (uint32_t)kChunk; r += blockDim.x) {
    const uint32_t k = 1 + c * kChunk + r;
    double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0, e4 = 0.0;
    bool want = false;
    int32_t cv = 0;
    if (k < io.L) {
      cv = io.Csrc[k];
      if (io.Cloc) io.Cloc[k] = cv;   // lazy local snapshot: the pre-fold table
      if (io.F) cv = fold_flips(cv, k, io, sb);
      if (io.Cdst) io.Cdst[k] = cv;
      const int32_t av = abs(cv);
      pmax = max(pmax, av);
      want = io.hlist != nullptr && av >= io.hthr;
      e2 = term(io, av);
      e4 = term(io, abs(cv - 4));
      e3 = term(io, abs(cv - 2));
      e1 = term(io, abs(cv + 2));
      e0 = term(io, abs(cv + 4));
    }
    if (io.hlist) {
      const uint32_t m = __ballot_sync(FULL, want);
      if (m) {
        const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(io.hcount, (uint32_t)__popc(m));
        base = __shfl_sync(FULL, base, leader);
        PSL_CHK(!want || base + __popc(m & ((1u << lane) - 1)) < io.L, 33);
        if (want) io.hlist[base + __popc(m & ((1u << lane) - 1))] = make_int2((int)k, cv);
      }
    }
    double2* rec = reinterpret_cast<double2*>(tab + (size_t)r * kRecDoubles);
    rec[0] = make_double2(e4, e2);   // BOTH slot = 2*bA' + bB'
    rec[1] = make_double2(e2, e0);
    rec[2] = make_double2(e3, e1);   // ONE  slot = one valid bit
    rec[3] = make_double2(e1, e2);   // (slot 3: e2, unused)
    tail[r] = e2;
  }
}

enum : int { CLS_BOTH = 0, CLS_ONE = 1, CLS_TAIL = 2, CLS_MIXED = 3 };

__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void lds_f64x2(uint32_t a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// bits of word x for cell q, moved so the field lands at bit `to`
template <int FIELD_BITS, int TO>
__device__ __forceinline__ uint32_t field_at(uint32_t x, int q) {
  const int sh = FIELD_BITS * q - TO;
  return sh < 0 ? (x << (-sh)) : (x >> sh);
}

// One full sweep over k = 1..L-1 for the kJ adjacent neighbours j[m] of this
// lane (sum[m] = their fitness, the reference's serial ascending-k chain).
//
// Per 32-shift block the warp picks one code path from warp-uniform
// thresholds over its 128 neighbours (no per-lane branching):
//   BOTH  every neighbour has both s_{j-k} and s_{j+k}: 2-bit cell code
//         (bA', bB') -> record slot {e4, e2, e2, e0} via a divergent LDS.64
//   ONE   every neighbour past its both-range, before its one-range end:
//         1-bit code b' selects e3 / e1, loaded once per k (uniform LDS.128)
//         and chosen per neighbour on the ALU (FSEL) or the FMA pipe
//         (IMAD on the two 32-bit halves: e3 + b'(e1 - e3) mod 2^32)
//   TAIL  every neighbour past its one-range end: |C_k|^alpha, loaded once
//         per two shifts (uniform LDS.128) for all kJ chains
//   MIXED some range boundary inside the block: per-cell region, LDS path
// with bA' = [s_{j-k} == -s_j], bB' = [s_{j+k} == -s_j]; the term is
// |C_k - 2 s_j (s_{j-k} + s_{j+k})|^alpha = e_{2 + s_j(s_{j-k}+s_{j+k})}.
__device__ __forceinline__ void sweep(const SweepIO& io, const Smem& sm, const bool (&active)[kJ],
                                      const uint32_t (&jin)[kJ], double (&sum)[kJ],
                                      int32_t& pmax, double& chain) {
  const uint32_t L = io.L;
  const int nwords = (int)io.nwords;
  const uint32_t* sb = sm.sb;
  // inactive neighbours shadow the warp's first active one (results discarded)
  const uint32_t src = __ffs(__ballot_sync(FULL, active[0])) - 1;
  const uint32_t jsrc = __shfl_sync(FULL, jin[0], src < 32 ? src : 0);
  uint32_t mbj[kJ], jm[kJ];
  uint32_t sideA_bits = 0;           // bit m: neighbour m's one-side range uses s[j-k]
  uint32_t lminBE = FULL, lmaxBE = 0, lminOE = FULL, lmaxOE = 0;
#pragma unroll
  for (int m = 0; m < kJ; ++m) {
    const uint32_t j = active[m] ? jin[m] : jsrc;
    jm[m] = j;
    const uint32_t left = j, right = L - 1 - j;       // sequence.hpp:131-135
    const uint32_t be = left < right ? left : right;
    const uint32_t oe = left < right ? right : left;
    sideA_bits |= (left >= right ? 1u : 0u) << m;
    mbj[m] = ((sb[(j >> 5) + 1] >> (j & 31)) & 1u) ? FULL : 0u;
    lminBE = min(lminBE, be); lmaxBE = max(lmaxBE, be);
    lminOE = min(lminOE, oe); lmaxOE = max(lmaxOE, oe);
  }
  // The kJ neighbours of a lane are consecutive positions except when the
  // neighbourhood wraps past L-1 inside the lane (or lanes shadow inactive
  // neighbours): such lanes rebuild their planes from memory each block.
  bool adj = true;
#pragma unroll
  for (int m = 1; m < kJ; ++m) adj = adj && jm[m] == jm[0] + m;
  // shared sliding windows (3 words each) of an adjacent lane:
  //   B: positions j0 + k0 .. j0 + k0 + 34      (s_{j+k})
  //   A: positions j0 - k0 - 31 .. j0 - k0 + 3  (s_{j-k}, reversed by BREV)
  // (the walk's bit array carries >= nwords+48 zero words on both sides, so
  // these pointers slide past either end without clamps)
  const uint32_t shB = (jm[0] + 1) & 31;
  const uint32_t shA = jm[0] & 31;
  const uint32_t* pB = sb + (int)((jm[0] + 1) >> 5) + 1;          // word of j0 + k0
  const uint32_t* pA = sb + ((int)(jm[0] >> 5) - 1) + 1;          // word of j0 - k0 - 31
  const uint32_t minBE = __reduce_min_sync(FULL, lminBE), maxBE = __reduce_max_sync(FULL, lmaxBE);
  const uint32_t minOE = __reduce_min_sync(FULL, lminOE), maxOE = __reduce_max_sync(FULL, lmaxOE);
#pragma unroll
  for (int m = 0; m < kJ; ++m) sum[m] = 0.0;
  const bool warp_scans = io.scan && __any_sync(FULL, active[0]);
  const uint32_t tab0 = smem_u32(sm.tab), tail0 = smem_u32(sm.tail);

  build_chunk(io, 0, sm.tab, sm.tail, sb, pmax);
  __syncthreads();
  for (uint32_t c = 0; c < io.nchunks; ++c) {
    const uint32_t buf = c & 1;
    if (c + 1 < io.nchunks)
      build_chunk(io, c + 1, sm.tab + (size_t)(buf ^ 1) * kChunk * kRecDoubles,
                  sm.tail + (size_t)(buf ^ 1) * kChunk, sb, pmax);
    const uint32_t tab = tab0 + buf * (kChunk * kRecDoubles * 8);
    const uint32_t tail = tail0 + buf * (kChunk * 8);
    if (warp_scans) {
#pragma unroll 1
      for (uint32_t blk = 0; blk < kChunk / 32; ++blk) {
        const uint32_t k0 = 1 + c * kChunk + blk * 32;
        const uint32_t kend = k0 + 31;
        const uint32_t rb = tab + blk * 32 * (kRecDoubles * 8);   // 64-byte aligned
        const bool ub = maxBE < k0 || minBE >= kend;
        const bool uo = maxOE < k0 || minOE >= kend;
        const int cls = !(ub && uo) ? CLS_MIXED
                        : minBE >= kend ? CLS_BOTH : (maxOE < k0 ? CLS_TAIL : CLS_ONE);
        // bit planes of the block: Bp[m] bit q = bB'(k0+q), Ap[m] bit q = bA'(k0+q)
        // (shared 64-bit windows XB:YB / XA:YA for a lane of adjacent neighbours)
        uint32_t XB = 0, YB = 0, XA = 0, YA = 0;
        uint32_t Bp[kJ], Ap[kJ];
        if (cls != CLS_TAIL) {
          if (adj) {
            PSL_CHK(sb_ok(pB + 2 - sb, L) && sb_ok(pA - sb, L), 30);
            const uint32_t b0 = pB[0], b1 = pB[1], b2 = pB[2];
            const uint32_t a0 = pA[0], a1 = pA[1], a2 = pA[2];
            XB = __funnelshift_r(b0, b1, shB); YB = __funnelshift_r(b1, b2, shB);
            XA = __funnelshift_r(a0, a1, shA); YA = __funnelshift_r(a1, a2, shA);
            if (cls != CLS_BOTH) {
#pragma unroll
              for (int m = 0; m < kJ; ++m) {
                Bp[m] = __funnelshift_r(XB, YB, m) ^ mbj[m];
                Ap[m] = __brev(__funnelshift_r(XA, YA, m)) ^ mbj[m];
              }
            }
          } else {
#pragma unroll
            for (int m = 0; m < kJ; ++m) {
              const int pbB = (int)(jm[m] + k0), pbA = (int)jm[m] - (int)k0 - 31;
              const int wB = pbB >> 5, wA = pbA >> 5;       // arithmetic shift = floor
              Bp[m] = __funnelshift_r(sword(sb, wB, nwords), sword(sb, wB + 1, nwords), pbB & 31) ^ mbj[m];
              Ap[m] = __brev(__funnelshift_r(sword(sb, wA, nwords), sword(sb, wA + 1, nwords),
                                             pbA & 31)) ^ mbj[m];
            }
          }
        }
        if (cls == CLS_BOTH) {
          // BOTH: 2-bit code, slot = 2 bA' + bB'; W[m] interleaves (bB', bA')
          uint32_t Wlo[kJ], Whi[kJ];
          if (adj) {
            // spread the shared windows once; neighbour m is a 2m-bit funnel
            const uint32_t SB0 = spread_lo(XB), SB1 = spread_hi(XB), SB2 = spread_lo(YB);
            const uint32_t RL = __brev(YA), RH = __brev(XA);   // bit-reversed A window
            const uint32_t SA1 = spread_hi(RL) << 1, SA2 = spread_lo(RH) << 1,
                           SA3 = spread_hi(RH) << 1;
#pragma unroll
            for (int m = 0; m < kJ; ++m) {
              const uint32_t blo = m ? __funnelshift_r(SB0, SB1, 2 * m) : SB0;
              const uint32_t bhi = m ? __funnelshift_r(SB1, SB2, 2 * m) : SB1;
              const uint32_t alo = m ? __funnelshift_r(SA1, SA2, 32 - 2 * m) : SA2;
              const uint32_t ahi = m ? __funnelshift_r(SA2, SA3, 32 - 2 * m) : SA3;
              Wlo[m] = (blo | alo) ^ mbj[m];
              Whi[m] = (bhi | ahi) ^ mbj[m];
            }
          } else {
#pragma unroll
            for (int m = 0; m < kJ; ++m) {
              Wlo[m] = spread_lo(Bp[m]) | (spread_lo(Ap[m]) << 1);
              Whi[m] = spread_hi(Bp[m]) | (spread_hi(Ap[m]) << 1);
            }
          }
#pragma unroll
          for (int q = 0; q < 32; ++q) {
#pragma unroll
            for (int m = 0; m < kJ; ++m) {
              const uint32_t v = field_at<2, 3>(q < 16 ? Wlo[m] : Whi[m], q & 15);
              sum[m] = __dadd_rn(sum[m], lds_f64(and_or(v, 0x18u, rb) + q * 64));
            }
          }
        } else if (cls == CLS_ONE) {
          // ONE: 1-bit code from the neighbour's valid side selects e3 / e1,
          // loaded once per k for all kJ neighbours.  Cells go in groups of
          // kG so the per-cell predicates come from one R2P per neighbour.
          constexpr int kG = 4;
          uint32_t P[kJ];
#pragma unroll
          for (int m = 0; m < kJ; ++m) P[m] = ((sideA_bits >> m) & 1u) ? Ap[m] : Bp[m];
#pragma unroll
          for (int g = 0; g < 32 / kG; ++g) {
            double e3[kG], e1[kG];
#pragma unroll
            for (int qq = 0; qq < kG; ++qq) lds_f64x2(rb + (g * kG + qq) * 64 + 32, e3[qq], e1[qq]);
#pragma unroll
            for (int m = 0; m < kJ; ++m) {
              // predicates of kG cells of one neighbour from one R2P; the kJ
              // chains are independent, each still adds in ascending k
              const uint32_t x = P[m] >> (g * kG);
#pragma unroll
              for (int qq = 0; qq < kG; ++qq)
                sum[m] = __dadd_rn(sum[m], ((x >> qq) & 1u) ? e1[qq] : e3[qq]);
            }
          }
        } else if (cls == CLS_TAIL) {
          // TAIL: the term is |C_k|^alpha for every neighbour
          const uint32_t t2 = tail + blk * 32 * 8;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            double x, y;
            lds_f64x2(t2 + q * 16, x, y);
#pragma unroll
            for (int m = 0; m < kJ; ++m) {
              sum[m] = __dadd_rn(sum[m], x);
              sum[m] = __dadd_rn(sum[m], y);
            }
          }
        } else {
          // MIXED: a region boundary inside the block for some neighbour
#pragma unroll
          for (int m = 0; m < kJ; ++m) {
            const uint32_t Wlo = spread_lo(Bp[m]) | (spread_lo(Ap[m]) << 1);
            const uint32_t Whi = spread_hi(Bp[m]) | (spread_hi(Ap[m]) << 1);
            double s = sum[m];
#pragma unroll 4
            for (int q = 0; q < 32; ++q) {
              const uint32_t k = k0 + q;
              const uint32_t x = q < 16 ? Wlo : Whi;
              const int sh = 2 * (q & 15) - 3;
              const uint32_t v = sh < 0 ? (x << (-sh)) : (x >> sh);
              const uint32_t jl = jm[m], jr = L - 1 - jm[m];
              const bool inb = k <= min(jl, jr);
              const bool ino = k <= max(jl, jr);
              const uint32_t mask = inb ? 0x18u : (ino ? (((sideA_bits >> m) & 1u) ? 0x10u : 0x08u) : 0u);
              const uint32_t base = inb ? 0u : (ino ? 32u : 8u);
              s = __dadd_rn(s, lds_f64(and_or(v, mask, base | rb) + q * 64));
            }
            sum[m] = s;
          }
        }
        ++pB;
        --pA;
      }
    }
    if (io.chain && threadIdx.x == 0) {
      // fitness(table, pow) (sequence.cpp:131-141): serial ascending k
      for (int r = 0; r < kChunk / 2; ++r) {
        double x, y;
        lds_f64x2(tail + r * 16, x, y);
        chain = __dadd_rn(chain, x);
        chain = __dadd_rn(chain, y);
      }
    }
    __syncthreads();
  }
}

// Exact neighbour PSL from the high-sidelobe list (entries (k, C_k)).
__device__ __forceinline__ int32_t neighbour_psl(const int2* h, uint32_t nh, int32_t thr,
                                                 bool filtered, uint32_t j, uint32_t L,
                                                 const uint32_t* sb) {
  const int sj = sval(sb, j);
  int32_t peak = 0;
#pragma unroll 4
  for (uint32_t e = 0; e < nh; ++e) {          // unrolled: the entries' bit loads overlap
    const int2 kc = h[e];
    if (!filtered && abs(kc.y) < thr) continue;
    const uint32_t k = (uint32_t)kc.x;
    const int sa = (k <= j) ? sval(sb, j - k) : 0;
    const int sbv = (j + k < L) ? sval(sb, j + k) : 0;
    const int32_t a = abs(kc.y - 2 * sj * (sa + sbv));
    peak = max(peak, a);
  }
  return peak;
}

// Block-wide lexicographic (value, i) and (psl, i) minima + non-finite flag.
// Result in ctl->best_* (valid after the trailing __syncthreads).
__device__ __forceinline__ void block_reduce_scan(Ctl* ctl, double v, uint32_t i, int32_t p,
                                                  uint32_t pi, int bad) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(FULL, v, o);
    const uint32_t i2 = __shfl_xor_sync(FULL, i, o);
    const int32_t p2 = __shfl_xor_sync(FULL, p, o);
    const uint32_t pi2 = __shfl_xor_sync(FULL, pi, o);
    bad |= __shfl_xor_sync(FULL, bad, o);
    if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
    if (p2 < p || (p2 == p && pi2 < pi)) { p = p2; pi = pi2; }
  }
  if (lane == 0) { ctl->rv[warp] = v; ctl->ri[warp] = i; ctl->rp[warp] = p; ctl->rpi[warp] = pi; ctl->rbad[warp] = bad; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    v = lane < nw ? ctl->rv[lane] : __longlong_as_double(0x7ff0000000000000ll);
    i = lane < nw ? ctl->ri[lane] : 0xffffffffu;
    p = lane < nw ? ctl->rp[lane] : 0x7fffffff;
    pi = lane < nw ? ctl->rpi[lane] : 0xffffffffu;
    bad = lane < nw ? ctl->rbad[lane] : 0;
    for (int o = 16; o; o >>= 1) {
      const double v2 = __shfl_xor_sync(FULL, v, o);
      const uint32_t i2 = __shfl_xor_sync(FULL, i, o);
      const int32_t p2 = __shfl_xor_sync(FULL, p, o);
      const uint32_t pi2 = __shfl_xor_sync(FULL, pi, o);
      bad |= __shfl_xor_sync(FULL, bad, o);
      if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
      if (p2 < p || (p2 == p && pi2 < pi)) { p = p2; pi = pi2; }
    }
    if (lane == 0) { ctl->best_v = v; ctl->best_i = i; ctl->best_psl = p; ctl->best_pi = pi; ctl->bad = bad; }
  }
  __syncthreads();
}

__device__ __forceinline__ int32_t block_max(Ctl* ctl, int32_t v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) ctl->rmax[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? ctl->rmax[lane] : 0;
    v = warp_max(v);
    if (lane == 0) ctl->rmax[0] = v;
  }
  __syncthreads();
  const int32_t r = ctl->rmax[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ long long block_sum64(Ctl* ctl, long long v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  if (lane == 0) ctl->re[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? ctl->re[lane] : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (lane == 0) ctl->re[0] = v;
  }
  __syncthreads();
  const long long r = ctl->re[0];
  __syncthreads();
  return r;
}

// merit_factor energy (sequence.cpp:143-152) of the pivot with position f
// flipped (f < 0: unflipped).  sb holds the pivot.
__device__ long long energy_sweep(Ctl* ctl, const int32_t* C, uint32_t L, const uint32_t* sb,
                                  int64_t f) {
  long long e = 0;
  const int sf = f >= 0 ? sval(sb, (uint32_t)f) : 0;
  // four shifts per thread and load (C is 16-byte aligned per walk; slots
  // k = 0 and k >= L of the padded row are skipped)
  for (uint32_t q = threadIdx.x; 4 * q < L; q += blockDim.x) {
    const int4 c4 = reinterpret_cast<const int4*>(C)[q];
    const int32_t cs[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t k = 4 * q + i;
      if (k == 0 || k >= L) continue;
      long long cv = cs[i];
      if (f >= 0) {
        const uint32_t fu = (uint32_t)f;
        int acc = 0;
        if (k <= fu) acc += sval(sb, fu - k);
        if (fu + k < L) acc += sval(sb, fu + k);
        cv += -2 * sf * acc;
      }
      e += cv * cv;
    }
  }
  return block_sum64(ctl, e);
}

// ------------------------------------------------------------ kernels

// random_sequence's L spin draws split into chunks of kSpinChunk draws: the
// state at the start of chunk j+1 is J s_j with J = T^kSpinChunk, T the
// xoshiro256 transition as a 256x256 GF(2) matrix; column c of J (= J e_c)
// is g_rng_jump[c].  One warp walks the chunk starts, then one thread per
// chunk draws its spins: the same bits and end state as L serial draws.
constexpr uint32_t kSpinChunk = 4096;
constexpr uint32_t kMaxSpinChunks = (1u << 20) / kSpinChunk;   // L <= 2^20
__device__ uint64_t g_rng_jump[256][4];

__global__ void __launch_bounds__(256) rng_jump_kernel() {
  const uint32_t c = threadIdx.x;
  uint64_t st[4] = {0, 0, 0, 0};
  st[c >> 6] = 1ull << (c & 63);
  for (uint32_t i = 0; i < kSpinChunk; ++i) rng_step(st);
#pragma unroll
  for (int q = 0; q < 4; ++q) g_rng_jump[c][q] = st[q];
}

// Walk setup: RNG, pivot (random_sequence, search.cpp:120-129, or warm start),
// snapshot copies.  One CTA per walk.
__global__ void __launch_bounds__(256) init_walks_kernel(RunArgs a, const uint64_t* seeds,
                                                         const uint32_t* packed, size_t packed_stride) {
  const uint32_t w = blockIdx.x;
  WalkState* S = a.st + w;
  uint32_t* bp = a.bits_piv + (size_t)w * a.w_stride + a.w_front;
  uint32_t* bl = a.bits_loc + (size_t)w * a.w_stride + a.w_front;
  uint32_t* bb = a.bits_best + (size_t)w * a.w_stride + a.w_front;
  uint32_t* us = a.used + (size_t)w * a.w_stride + a.w_front;
  const uint32_t nw = a.nwords;
  if (threadIdx.x == 0) {
    WalkState z = {};
    rng_seed(z.rng, seeds[w]);
    z.seed = seeds[w];
    z.nse = 1;                 // the initial fitness evaluation (search.cpp:349)
    z.phase = 1;
    z.fitness_pending = 1;
    z.loc_at_pivot = 1;        // local best = the start pivot (search.cpp:354-355)
    z.psl_best = -1;           // set from P on the first pass
    *S = z;
  }
  if (!packed) {
    // L spin() draws in position order; bit = top bit of next() (1 <-> -1)
    __shared__ uint64_t cs[kMaxSpinChunks][4];
    __shared__ uint64_t jm[256][4];
    const uint32_t nch = (a.L + kSpinChunk - 1) / kSpinChunk;
    if (nch > 1)
      for (uint32_t i = threadIdx.x; i < 256 * 4; i += blockDim.x) jm[i >> 2][i & 3] = g_rng_jump[i >> 2][i & 3];
    __syncthreads();
    if (threadIdx.x < 32) {
      const uint32_t l = threadIdx.x;
      uint64_t st[4];
      rng_seed(st, seeds[w]);
      for (uint32_t j = 0; j < nch; ++j) {
        if (l == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) cs[j][q] = st[q];
        }
        if (j + 1 == nch) break;
        // st = J st: lane l folds the columns of state bits 8l .. 8l+7
        uint64_t acc[4] = {0, 0, 0, 0};
        const uint64_t byte = (st[l >> 3] >> (8 * (l & 7))) & 0xffull;
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if ((byte >> b) & 1ull) {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] ^= jm[8 * l + b][q];
          }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int o = 16; o; o >>= 1) acc[q] ^= __shfl_xor_sync(0xffffffffu, acc[q], o);
          st[q] = acc[q];
        }
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < nch; j += blockDim.x) {
      uint64_t st[4] = {cs[j][0], cs[j][1], cs[j][2], cs[j][3]};
      const uint32_t p0 = j * kSpinChunk, p1 = min(a.L, p0 + kSpinChunk);
      for (uint32_t wd = p0 >> 5; wd < (p1 + 31) >> 5; ++wd) {
        uint32_t word = 0;
        const uint32_t nb = min(32u, a.L - wd * 32);
        for (uint32_t b = 0; b < nb; ++b) word |= (uint32_t)(rng_next(st) >> 63) << b;
        bp[wd + 1] = word;
      }
      if (j + 1 == nch) {
#pragma unroll
        for (int q = 0; q < 4; ++q) S->rng[q] = st[q];     // the state after all L draws
      }
    }
  }
  if (packed) {
    // warm starts, validated and bit-packed on the host (psl_api.cu pack_walk):
    // nw words per walk (stride 0: one start shared by every walk)
    const uint32_t* src = packed + (size_t)w * packed_stride;
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) bp[i + 1] = src[i];
  }
  __syncthreads();
  // padded layout: zero pads around words 1..nw (relative to the walk base);
  // the pads let the scan's sliding windows run off either end unclamped
  const long long lo = -(long long)a.w_front, hi = (long long)(a.w_stride - a.w_front);
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const bool in = i >= 1 && i <= (long long)nw;
    const uint32_t v = in ? bp[i] : 0u;
    if (!in) bp[i] = 0u;
    bl[i] = v;
    bb[i] = v;
    us[i] = 0u;
  }
}

// SidelobeTable::build (sequence.cpp:46-60) in bit-parallel form:
// C_k = (L-k) - 2 * popc(s[0..L-k) XOR s[k..L)).  Each warp owns 128
// consecutive shifts (lane: k, k+32, k+64, k+96) and slides over the words.
// Optionally reduces PSL and energy into the walk state and copies C to Cloc.
constexpr int kTabR = 4;
__global__ void __launch_bounds__(256) build_tables_kernel(const uint32_t* bits, size_t w_stride,
                                                          int32_t* C, int32_t* Cloc,
                                                          size_t c_stride, uint32_t L,
                                                          WalkState* st) {
  const uint32_t walk = blockIdx.y;
  const uint32_t* S = bits + (size_t)walk * w_stride;
  int32_t* Cw = C + (size_t)walk * c_stride;
  int32_t* Cl = Cloc ? Cloc + (size_t)walk * c_stride : nullptr;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint32_t kb = 1 + gw * 32 * kTabR;
  if (gw == 0 && lane == 0) { Cw[0] = (int32_t)L; if (Cl) Cl[0] = (int32_t)L; }
  if (kb >= L) return;
  const uint32_t k0 = kb + lane;               // this lane's smallest shift
  const uint32_t sh = k0 & 31;
  const uint32_t base = k0 >> 5;
  uint32_t win[kTabR + 1];
#pragma unroll
  for (int r = 0; r <= kTabR; ++r) win[r] = S[base + r];
  uint32_t diff[kTabR] = {0, 0, 0, 0};
  // pairs (p, p+k) exist for p < L-k; full words while 32(i+1) <= L - kmax_warp
  const uint32_t kmax_warp = kb + 32 * kTabR - 1;
  const uint32_t full = kmax_warp < L ? (L - kmax_warp) / 32 : 0;
  uint32_t i = 0;
  for (; i < full; ++i) {
    const uint32_t s0 = S[i];
#pragma unroll
    for (int r = 0; r < kTabR; ++r) diff[r] += __popc(s0 ^ __funnelshift_r(win[r], win[r + 1], sh));
#pragma unroll
    for (int r = 0; r < kTabR; ++r) win[r] = win[r + 1];
    win[kTabR] = S[i + 1 + base + kTabR];
  }
  // ragged end: mask by the per-shift pair count
  const uint32_t kmin = k0;
  const uint32_t last = kmin < L ? (L - kmin + 31) / 32 : 0;
  for (; i < last; ++i) {
    const uint32_t s0 = S[i];
#pragma unroll
    for (int r = 0; r < kTabR; ++r) {
      const uint32_t k = k0 + 32 * r;
      if (k < L) {
        const int rem = (int)(L - k) - (int)(32 * i);
        if (rem > 0) {
          const uint32_t m = rem >= 32 ? FULL : ((1u << rem) - 1u);
          diff[r] += __popc((s0 ^ __funnelshift_r(win[r], win[r + 1], sh)) & m);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kTabR; ++r) win[r] = win[r + 1];
    win[kTabR] = S[i + 1 + base + kTabR];
  }
  int32_t pm = 0;
  long long en = 0;
#pragma unroll
  for (int r = 0; r < kTabR; ++r) {
    const uint32_t k = k0 + 32 * r;
    if (k < L) {
      const int32_t cv = (int32_t)(L - k) - 2 * (int32_t)diff[r];
      Cw[k] = cv;
      if (Cl) Cl[k] = cv;
      pm = max(pm, abs(cv));
      en += (long long)cv * cv;
    }
  }
  if (st) {
    pm = warp_max(pm);
    for (int o = 16; o; o >>= 1) en += __shfl_xor_sync(FULL, en, o);
    if (lane == 0) {
      atomicMax(&st[walk].P, pm);
      atomicAdd(reinterpret_cast<unsigned long long*>(&st[walk].energy_best),
                (unsigned long long)en);
    }
  }
}

#include "psl_cert.cuh"
static_assert(kCertBytes <= kCertRegion, "certified buffers exceed the shared region");
static_assert(((1u << 20) - 1 + kCC - 1) / kCC + kLag <= 72 * 32, "per-chunk flag words");

// Neighbour PSL + thread-local reduce_scan over this thread's kJ neighbours
// (ascending offset) + the block-wide lexicographic minima (ctl->best_*).
__device__ __forceinline__ void reduce_group(Ctl* ctl, const Smem& sm, const int2* hlist,
                                             const bool (&active)[kJ], const uint32_t (&jj)[kJ],
                                             const double (&val)[kJ], uint32_t ibase, uint32_t L) {
  const uint32_t nf = ctl->hf_count;
  double bv = __longlong_as_double(0x7ff0000000000000ll);
  uint32_t bi = 0xffffffffu, bpi = 0xffffffffu;
  int32_t bp = 0x7fffffff;
  int bad = 0;
#pragma unroll
  for (int m = 0; m < kJ; ++m) {
    if (!active[m]) continue;
    const uint32_t i = ibase + m + 1;
    const int32_t psl = nf <= (uint32_t)kHCap
        ? neighbour_psl(sm.hf, nf, 0, true, jj[m], L, sm.sb)
        : neighbour_psl(hlist, ctl->hcount, ctl->P_new - 8, false, jj[m], L, sm.sb);
    bad |= !isfinite(val[m]);
    if (bi == 0xffffffffu || val[m] < bv) { bv = val[m]; bi = i; }
    if (psl < bp) { bp = psl; bpi = i; }
  }
  block_reduce_scan(ctl, bv, bi, bp, bpi, bad);
}

// First-pass bookkeeping shared by the exact and certified passes: the new
// pivot PSL, consumed pending flips, the restart fitness chain.
__device__ __forceinline__ void first_pass_state(Ctl* ctl, const RunArgs& a, uint32_t w,
                                                 int32_t Pn, double chain, uint32_t alpha) {
  WalkState& S = ctl->st;
  // the lazily materialised snapshot is the PRE-fold table: its PSL is the
  // previous pass's
  if (S.local_pending) { S.P_local = S.P; S.local_pending = 0; }
  ctl->P_new = Pn;
  S.P = Pn;
  S.n_pending = 0;
  S.src_local = 0;
  if (S.fitness_pending) {
    S.fitness_pending = 0;
    if (!isfinite(chain)) {
      // fitness() throws OverflowError (sequence.cpp:139); a provisional
      // phase-switch event / trace from the restart step is withdrawn.
      S.status = PSL_ERR_OVERFLOW; S.err_kind = 1; S.err_alpha = alpha;
      if (S.switch_pending && S.n_events) --S.n_events;
      if (S.trace_patch && S.n_traces) --S.n_traces;
    } else {
      S.value_local = chain;
      S.vl_exact = 1; S.vl_lo = chain; S.vl_hi = chain;
      if (S.trace_patch) {
        a.traces[(size_t)w * a.traces_cap + S.n_traces - 1].value_local = chain;
      }
    }
    S.trace_patch = 0;
    S.switch_pending = 0;
  }
  ctl->hf_count = 0;
}

// Filter the pass's high-sidelobe list into smem (entries that can still
// carry a neighbour's peak: |C_k| >= P - 8).
__device__ __forceinline__ void filter_hlist(Ctl* ctl, const Smem& sm, const int2* hlist) {
  const int32_t thr = ctl->P_new - 8;
  const uint32_t hc = ctl->hcount;
  for (uint32_t e = threadIdx.x; e < hc; e += blockDim.x) {
    const int2 kc = hlist[e];
    if (abs(kc.y) >= thr) {
      const uint32_t slot = atomicAdd(&ctl->hf_count, 1u);
      if (slot < (uint32_t)kHCap) sm.hf[slot] = kc;
    }
  }
}

// value_step vs value_local: -1 less, 0 equal, +1 greater, 2 undecided
__device__ __forceinline__ int compare_local(const WalkState& S, double lo, double hi, bool exact,
                                             double v) {
  if (exact && S.vl_exact) return v < S.value_local ? -1 : (v > S.value_local ? 1 : 0);
  const double vlo = S.vl_exact ? S.value_local : S.vl_lo;
  const double vhi = S.vl_exact ? S.value_local : S.vl_hi;
  if (hi < vlo) return -1;
  if (lo > vhi) return 1;
  return 2;
}

// The device-resident run_search loop (search.cpp:327-430), one CTA per walk.
// kCert: steps may be decided by the certified scan (psl_cert.cuh); any step
// it cannot decide is re-scored by the exact sweep, so every decision (and
// the RunRecord) is the reference's.
// kCert: 512 threads, one walk per SM (the certified scan's digit ring and
// chunk buffers need the shared memory); the exact kernel: 256 threads, two per
// SM.  The exact sweep in the 512-thread kernel leaves threads >= 256 inactive.
#ifndef PSL_FWD_WARP
#define PSL_FWD_WARP 15
#endif
#ifndef PSL_REV_WARP
#define PSL_REV_WARP 14
#endif
#ifndef PSL_STAGGER
#define PSL_STAGGER 0              // 1: half the warps cross-then-build, half build-then-cross (measured +0.4-1.6 %)
#endif
#ifndef PSL_ISSUE_SPLIT
#define PSL_ISSUE_SPLIT 1          // 2: issue a direction in two halves around other work (measured: +-1 %)
#endif

// Timing-only instrumentation (-DPSL_PHASE_TIMING, tools/ablate.sh): per-warp
// cycles per phase of the certified chunk loop, printed by CTA 0 at exit.
#ifdef PSL_PHASE_TIMING
}  // namespace
}  // namespace pslb
#include <cstdio>
namespace pslb {
namespace {
constexpr int kPT = 19;  // loop top, build, cores, barrier, issue, cross, band, pass prologue, mbar wait, fence,
                         // tail, row intervals, reduce, exact/vl, control, step top
#define PT_MARK(i)                                                   \
  do {                                                               \
    const long long _n = clock64();                                  \
    if ((t & 31) == 0) pt_acc[t >> 5][i] += _n - pt_last;            \
    pt_last = _n;                                                    \
  } while (0)
#else
#define PT_MARK(i) do {} while (0)
#endif

template <bool kCert>
__global__ void __launch_bounds__(kCert ? 2 * kThreads : kThreads, kCert ? 1 : 2) run_kernel(RunArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem sm = carve<kCert>(smem_raw);
  Ctl* ctl = sm.ctl;
  const uint32_t w = blockIdx.x, t = threadIdx.x;
#ifdef PSL_PHASE_TIMING
  __shared__ long long pt_acc[16][kPT];
  if (t < 16 * kPT) pt_acc[t / kPT][t % kPT] = 0;
  __syncthreads();
  long long pt_last = clock64();
  const long long pt_t0 = pt_last;
#endif
  const uint32_t L = a.L, nw = a.nwords;
  WalkState* gst = a.st + w;
  uint32_t* bits_piv = a.bits_piv + (size_t)w * a.w_stride + a.w_front;
  uint32_t* bits_loc = a.bits_loc + (size_t)w * a.w_stride + a.w_front;
  uint32_t* bits_best = a.bits_best + (size_t)w * a.w_stride + a.w_front;
  uint32_t* used = a.used + (size_t)w * a.w_stride + a.w_front;
  int32_t* Cpiv = a.Cpiv + (size_t)w * a.c_stride;
  int32_t* Cloc = a.Cloc + (size_t)w * a.c_stride;
  int2* hlist = a.hlist + (size_t)w * a.h_stride;
  uint32_t* flips = a.flips + (size_t)w * a.f_stride;

  if (t == 0) {
    ctl->st = *gst;
    ctl->steps_this_launch = 0;
    if (ctl->st.t0_ns == 0) ctl->st.t0_ns = globaltimer();
    if (ctl->st.psl_best < 0) { ctl->st.psl_best = ctl->st.P; ctl->st.P_local = ctl->st.P; }
  }
  sm.sb = bits_piv;   // padded: word i at bits_piv[i + 1]
  __syncthreads();
  if (ctl->st.done || ctl->st.status != PSL_OK) return;
  uint32_t mb_par = 0u;            // bit b: next phase parity to wait for on ctl->mbar[b]
                                   // (a bit mask: an indexed 2-array lived in local memory)
  uint32_t cphase = 0u;             // ... on ctl->cbar[0..2] (bit per slot)
  if (kCert) {
    if (t < 32) {   // the certified scan's tcgen05 accumulators live in TMEM
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&ctl->tmem)), "r"(kTmemCols) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) {
      // two committing warps per iteration (forward: warp 15, reversed: warp 14)
      for (int i = 0; i < 2; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&ctl->mbar[i])) : "memory");
      for (int i = 0; i < 3; ++i)   // C ring: thread 0's arrive.expect_tx + the copy's bytes
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ctl->cbar[i])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }

  const uint32_t ngroups = (a.n + kGroup - 1) / kGroup;
  for (;;) {
    // ---- top of step: stop checks, max-nse first (search.cpp:371-374)
    if (t == 0) {
      WalkState& S = ctl->st;
      const double elapsed = (double)(globaltimer() - S.t0_ns) * 1e-9;
      const bool stop = (a.has_max_nse && S.nse >= a.max_nse) ||
                        (a.has_max_seconds && elapsed >= a.max_seconds);
      const bool room = ctl->steps_this_launch < a.step_budget &&
                        (!a.record_events || S.n_events + 2 <= a.events_cap) &&
                        (!a.record_traces || S.n_traces + 1 <= a.traces_cap);
      ctl->do_scan = !stop && room;
      if (stop) { S.done = 1; S.end_ns = globaltimer(); }
      ctl->need_pass = ctl->do_scan || S.fitness_pending;
      if (ctl->do_scan) ctl->start = (uint32_t)rng_bounded(S.rng, L);  // search.cpp:375
      ctl->hcount = 0;
      ctl->fit = 0.0;
      ctl->cert = 0;
      ctl->need_exact = 0;
      ctl->need_vl = 0;
      ctl->chk_on = 0; ctl->chk_rows = 0; ctl->chk_viol = 0;
      ctl->chk_tight = 0ull; ctl->chk_relw = 0ull;
      if (kCert && a.cert && ctl->do_scan &&
          L >= kCertMinL) {
        // fixed-point scale: every |H4|, |R4| <= 2 pow(Amax, alpha) < 2^(62+q)
        const uint32_t alpha = S.phase == 1 ? a.alpha1 : a.alpha2;
        const int32_t Psrc = S.src_local ? S.P_local : S.P;
        const double amax = (double)Psrc + 4.0 * S.n_pending + 4.0;
        const double fa = pow_int_dev(amax, alpha);
        if (isfinite(fa) && fa * 8.0 * (double)L < 1e300) {
          // digit units: |H4| <= 8 alpha Amax^(alpha-1), |R4| <= 16 alpha (alpha-1)
          // Amax^(alpha-2) (mean-value bounds; x4 margin for rounding; a digit
          // overflow is detected in the builder and sends the step to the exact sweep)
          const double bh = 4.0 * fmin(2.0 * fa, 8.0 * alpha * pow(amax, (double)alpha - 1.0));
          const double br = 4.0 * (alpha >= 2 ? fmin(2.0 * fa, 16.0 * alpha * (alpha - 1.0) *
                                                             pow(amax, (double)alpha - 2.0))
                                              : 2.0 * amax);
          const int qh = bh > 0.0 ? max(0, ilogb(bh) + 1 - 62) : 0;
          const int qr = br > 0.0 ? max(0, ilogb(br) + 1 - 62) : 0;
          ctl->c_scaleH = ldexp(1.0, -qh); ctl->c_unitH = ldexp(1.0, qh); ctl->c_qH = qh;
          ctl->c_scaleR = ldexp(1.0, -qr); ctl->c_unitR = ldexp(1.0, qr); ctl->c_qR = qr;
          ctl->c_ovf = 0;
          ctl->cert = 1;
        }
      }
    }
    __syncthreads();
    PT_MARK(15);
    if (!ctl->need_pass) break;
    const bool do_scan = ctl->do_scan;
    const uint32_t start = ctl->start;
    // the few walk-state fields the pass needs (not the whole struct: registers)
    const uint32_t alpha = ctl->st.phase == 1 ? a.alpha1 : a.alpha2;
    const double* lut = ctl->st.phase == 1 ? a.lut1 : a.lut2;
    const uint32_t s_src_local = ctl->st.src_local, s_local_pending = ctl->st.local_pending;
    const uint32_t s_n_pending = ctl->st.n_pending, s_fitness_pending = ctl->st.fitness_pending;
    const int32_t s_Psrc = s_src_local ? ctl->st.P_local : ctl->st.P;

    if (kCert && ctl->cert) {
      // ================= certified pass(es) (psl_cert.cuh).  Rows rho = i - 1
      // (offset i) are neighbours j = start + i mod L; a window that wraps past
      // L - 1 is scored in two passes, one per contiguous row segment.
      const CertSmem cs = cert_carve(smem_raw);
#if PSL_XTMEM
      const CertLane ln = cert_lane8(cs);
#else
      const CertLane ln = cert_lane(cs);
#endif
      // row intervals [lo, hi] and midpoints of the current group, through global
      // scratch (not registers across the chunk loop)
      double* ivm = a.iv_buf + (size_t)w * 3 * kGroup;
      double* ivl = ivm + kGroup;
      double* ivh = ivl + kGroup;
      // the phase's PowerTable head (indices <= Psrc + 4F + 4 cover every lookup
      // of the pass) in shared memory when it fits
      const double* lut_c = lut;
      {
        const uint32_t nlut = (uint32_t)s_Psrc + 4u * s_n_pending + 5u;
        if (nlut <= kLutS) {
          double* lut_s = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ctl) + kCtlBytes);
          for (uint32_t i = t; i < nlut; i += blockDim.x) lut_s[i] = __ldg(lut + i);
          lut_c = lut_s;
        }
      }
      // n_lmt > 1024: groups of 1024 rows, one certified pass each (the first one
      // folds the move into C, collects the high sidelobes and the fitness chain);
      // group results combine in ascending offset order like the exact sweep's
      const uint32_t ngrp = (a.n + kGroup - 1) / kGroup;
      double* lo_all = a.lo_buf + (size_t)w * a.n;           // per-row lower bounds (ngrp > 1)
      for (uint32_t g = 0; g < ngrp; ++g) {
      const bool first = g == 0;
      const uint32_t gn = min((uint32_t)kGroup, a.n - g * kGroup);
      const uint32_t gs = (uint32_t)(((uint64_t)start + (uint64_t)g * kGroup) % L);   // rows j = gs + 1 + rho
      const uint32_t nA = min(gn, L - 1 - gs);               // rows before the wrap
      const int nseg = (nA > 0 && nA < gn) ? 2 : 1;
      for (int seg = 0; seg < nseg; ++seg) {
        const bool wrapped = seg == 1 || nA == 0;            // rows past L - 1: j = rho - nA
        const uint32_t r_lo = seg ? nA : 0, r_hi = (nseg == 2 && seg == 0) ? nA : gn;
        const int32_t j0 = wrapped ? (int32_t)gs + 1 - (int32_t)L : (int32_t)gs + 1;
        if (t == 0) {
          // zones over the segment's neighbours [jlo, jhi] (m_j = min(j, L-1-j))
          const uint32_t jlo = (uint32_t)(j0 + (int32_t)r_lo), jhi = (uint32_t)(j0 + (int32_t)r_hi - 1);
          const uint32_t h = (L - 1) / 2;
          const uint32_t m0 = min(jlo, L - 1 - jlo), m1 = min(jhi, L - 1 - jhi);
          ctl->m_lo = min(m0, m1);
          ctl->m_hi = (jlo <= L - 1 - h && jhi >= h) ? h : max(m0, m1);
          ctl->M_lo = L - 1 - ctl->m_hi;
          ctl->M_hi = L - 1 - ctl->m_lo;
        }
        __syncthreads();
        CertIO io;
        io.L = L; io.n = gn; io.nchunks = (L - 1 + kCC - 1) / kCC;
        io.j0 = j0; io.r_lo = r_lo; io.r_hi = r_hi; io.JT = j0 + (int32_t)r_lo;
        if (first && seg == 0) {
          io.Csrc = s_src_local ? Cloc : Cpiv;
          io.Cdst = Cpiv;
          io.Cloc = s_local_pending ? Cloc : nullptr;
          io.F = s_n_pending;
          io.hlist = hlist;
        } else {   // C already folded and written by the first pass
          io.Csrc = Cpiv; io.Cdst = nullptr; io.Cloc = nullptr; io.F = 0; io.hlist = nullptr;
        }
        io.flips = flips;
        io.f1 = io.F == 1 ? flips[0] : 0u;
        io.sf1 = io.F == 1 ? sval(sm.sb, io.f1) : 0;
        io.alpha = alpha; io.lut = lut_c;
        io.hcount = &ctl->hcount;
        io.hthr = s_Psrc - 4 * (int32_t)s_n_pending - 8;
        io.scaleH = ctl->c_scaleH; io.scaleR = ctl->c_scaleR;
        io.m_lo = ctl->m_lo; io.m_hi = ctl->m_hi; io.M_lo = ctl->M_lo; io.M_hi = ctl->M_hi;
        io.b2M = a.b2 + (size_t)w * 2 * kGroup;
        io.b2E = io.b2M + kGroup;
        io.c_stride = a.c_stride;
        io.cbar = ctl->cbar;
        // first step / restart: fitness() of the folded table, serially, by one
        // thread of warp 14 behind the builder (search.cpp:348, :409)
        // the first step's value_local (search.cpp:348) as an interval from a
        // parallel sum: it is only compared with (and, if undecided, recomputed
        // exactly as fitness() of) the local snapshot = the initial table.  After a
        // restart (:409) value_local belongs to the kicked pivot, not to the
        // snapshot, so there the exact serial chain runs (one thread behind the builder).
        const bool initial = ctl->st.nse == 1;
        io.fsum = first && seg == 0 && s_fitness_pending != 0 && initial;
        io.chain = first && seg == 0 && s_fitness_pending != 0 && !initial;
        double chain = 0.0;
#if !PSL_XTMEM
        int acc[kCertTiles][4];
#pragma unroll
        for (int r = 0; r < kCertTiles; ++r)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[r][e] = 0;
#endif
        bool ovf = false;
        double part[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        double Bs[kBandRows] = {0.0, 0.0};   // band-1 sums of rows kBandRows t + m
        int32_t pmax = 0;
        uint32_t nmma = 0, numma = 0, started = 0;
        const uint32_t tmem = ctl->tmem;
#if PSL_XTMEM
#define XACC tmem
#else
#define XACC acc
#endif
        // digit cores of shifts <= 0 (read by the first chunks' shifted N-groups) are zero
        for (int32_t cz = -(int32_t)kLag; cz < 0; ++cz) cert_zero_digits(cs, cz);
        // C_k streams into shared memory by cp.async two chunks ahead
        const uint32_t nch = io.nchunks;
        const bool builder = t < kCC;   // every thread builds one shift per chunk
        // which iterations issue forward (kappa-chunk c) / reversed (c - kLag) MMAs
        for (uint32_t c = t; c < (nch + kLag + 31) / 32 * 32; c += blockDim.x) {
          bool fw = false, rv = false;
          if (c < nch + kLag) {
            const long long kb = (long long)cert_kb(c);
            fw = io.JT + kb < (long long)L && cert_lin_in(io, kb - 896, kb + kCC - 1);
            const long long kbr = (long long)(int32_t)cert_kb((int32_t)c - (int32_t)kLag);
            rv = (long long)io.JT + 127 - kbr >= 0 && cert_lin_in(io, kbr, kbr + kCC - 1 + 896);
          }
          const uint32_t mf = __ballot_sync(FULL, fw), mr = __ballot_sync(FULL, rv);
          if ((t & 31) == 0) { ctl->cfw[c >> 5] = mf; ctl->crv[c >> 5] = mr; }
        }
        __syncthreads();
        // Chunks from c_end on are pure tail (zone 5: H4 = R4 = 0, every row's term
        // is |C_k|^alpha, no MMA reads their digit cores, no band constants): they
        // skip the chunk pipeline and are streamed by cert_tail after it.  The
        // serial fitness chain (restart passes) needs every chunk's record in
        // order, so chain passes keep the pipeline to the end.
        uint32_t c_end = nch;
        if (!io.chain) {
          uint32_t cl = io.M_hi >= 1 ? (io.M_hi - 1) / kCC : 0u;   // last chunk with kb <= M_hi
          while (cl + 1 < nch && ((ctl->cfw[(cl + 1) >> 5] >> ((cl + 1) & 31)) & 1u)) ++cl;
          c_end = min(nch, cl + 1);
        }
        if (builder) {
          cert_prefetch(io, cs, 0);
          if (c_end > 1) cert_prefetch(io, cs, 1);
        }
        uint2 fwords = (builder && io.F == 1) ? cert_fold_words(io, 0, sm.sb) : make_uint2(0u, 0u);
#ifndef PSL_LATE_WAIT
#define PSL_LATE_WAIT 1
#endif
        uint32_t issued = 0;        // bit (c & 1): iteration c committed MMAs not yet waited for
        // iteration c: build chunk c, stage the sequence cores of forward kappa-chunk c and
        // reversed kappa'-chunk c - kLag, issue their tcgen05 MMAs (one thread, async),
        // then the zone-1 cross MMAs (mma.sync) and band-1 cells of chunk c
        PT_MARK(7);
        {
        // warp 15 issues the forward MMAs of chunk c: half right after the chunk
        // barrier, half after its cross / band work; warp 14 the reversed ones
        // in the next iteration: half at the loop top, half after its build.  So
        // the tensor-pipe waits are split over two warps and two points each.
        constexpr int kHalf = PSL_ISSUE_SPLIT > 1 ? kCCols / 2 : kCCols;
#ifndef PSL_FWD_AFTER_CROSS
#define PSL_FWD_AFTER_CROSS 1      // warp 15 runs its cross rows before issuing the forward MMAs
                                   // (the tensor queue has drained by then; -1.7 % ms/step at m20)
#endif
        constexpr int kHalfF = PSL_FWD_AFTER_CROSS ? 0 : kHalf;
#ifndef PSL_REV_ISSUE
#define PSL_REV_ISSUE 2            // reversed MMAs of chunk c: 0 top of c + 1, 1 after warp 14's
                                   // build in c + 1 (+0.6 %), 2 after warp 14's cross rows in c (-0.7 %)
#endif
        constexpr int kHalfR = PSL_REV_ISSUE == 1 ? 0 : kHalf;
        const bool early = t < (uint32_t)kThreads;   // warps 0-7 (PSL_STAGGER)
        int32_t pend_c = -1;
        bool pend_rv = false;
        uint32_t pend_started = 0;
        for (uint32_t c = 0; c < c_end + kLag; ++c) {
          int32_t rv_c = -1;         // this iteration finishes the reversed MMAs of rv_c
          if (pend_c >= 0) {
            if (PSL_REV_ISSUE != 2 && kHalfR > 0 && (t >> 5) == PSL_REV_WARP)
              cert_issue_dir(cs, tmem, pend_c, 1, pend_rv, pend_started, &ctl->mbar[pend_c & 1], 0, kHalfR,
                             kHalfR == kCCols);
            rv_c = pend_c;
            pend_c = -1;
          }
#if !PSL_LATE_WAIT
          if (issued & (1u << (c & 1))) {      // MMAs of iteration c - 2 read this buffer
            PT_MARK(0);
            mbar_wait(&ctl->mbar[c & 1], (mb_par >> (c & 1)) & 1u);
            PT_MARK(8);
            mb_par ^= 1u << (c & 1);
            issued &= ~(1u << (c & 1));
          }
#endif
          PT_MARK(0);
          const bool fw = (ctl->cfw[c >> 5] >> (c & 31)) & 1u, rv = (ctl->crv[c >> 5] >> (c & 31)) & 1u;
          if (c < c_end) {
            if (builder) {
              if (c + 2 < c_end) cert_prefetch(io, cs, c + 2);
              const uint2 fnext = (io.F == 1 && c + 1 < c_end) ? cert_fold_words(io, c + 1, sm.sb) : fwords;
              const int pending = (int)min(2u, c_end - 1 - c);
              cert_build(io, cs, c, sm.sb, pmax, part, cert_take(io, cs, c, pending, cphase), fwords, ovf);
              fwords = fnext;
            }
          } else {
            cert_zero_digits(cs, c);
          }
          if (PSL_REV_ISSUE != 2 && kHalfR < kCCols && rv_c >= 0 && (t >> 5) == PSL_REV_WARP)
            cert_issue_dir(cs, tmem, rv_c, 1, pend_rv, pend_started, &ctl->mbar[rv_c & 1], kHalfR, kCCols, true);
          PT_MARK(1);
          // PSL_STAGGER: warps 0-7 run the cross MMAs / band cells of chunk c - 1
          // after building chunk c, warps 8-15 before (end of the previous
          // iteration), so one half's builder overlaps the other half's IMMA work
          // inside every barrier interval (buffers of c - 1 live until iteration c + 1)
          if (PSL_STAGGER && early && c >= 1 && c - 1 < c_end) {
            cert_cross_chunk(io, cs, ln, c - 1, XACC, nmma);
          }
#if PSL_LATE_WAIT
          // the MMAs of iteration c - 2 read A-core buffer c & 1 (and nothing the
          // builder writes: its digit-ring slots are 8 chunks apart), so their
          // completion is awaited only before this iteration's cores
          if (issued & (1u << (c & 1))) {
            PT_MARK(2);
            mbar_wait(&ctl->mbar[c & 1], (mb_par >> (c & 1)) & 1u);
            PT_MARK(8);
            mb_par ^= 1u << (c & 1);
            issued &= ~(1u << (c & 1));
          }
#endif
          cert_cores(io, cs, (int32_t)c, sm.sb, fw, rv);
          PT_MARK(2);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          PT_MARK(9);
          __syncthreads();
          PT_MARK(3);
#ifdef PSL_ABLATE_ISSUE
          if (false) {
#else
          if ((fw || rv)) {
#endif
            // warp 15 (stages no cores) issues, one lane elected per MMA
            if (kHalfF > 0 && (t >> 5) == PSL_FWD_WARP)
              cert_issue_dir(cs, tmem, (int32_t)c, 0, fw, started, &ctl->mbar[c & 1], 0, kHalfF, kHalfF == kCCols);
            pend_c = (int32_t)c; pend_rv = rv; pend_started = started;
            started |= (fw ? 1u : 0u) | (rv ? 2u : 0u);   // uniform copy of the issuer's flags
            numma += (fw ? kCCols : 0) + (rv ? kCCols : 0);
            issued |= 1u << (c & 1);
          }
          PT_MARK(4);
          if (c < c_end && !(PSL_STAGGER && early)) {   // zone-1 cross MMAs
            cert_cross_chunk(io, cs, ln, c, XACC, nmma);
            PT_MARK(5);
            if (io.chain && t == kCertThreads - 64) cert_chain_chunk(io, cs, c, chain);
            PT_MARK(6);
          }
          if (kHalfF < kCCols && pend_c == (int32_t)c && (t >> 5) == PSL_FWD_WARP)
            cert_issue_dir(cs, tmem, (int32_t)c, 0, fw, pend_started, &ctl->mbar[c & 1], kHalfF, kCCols, true);
          if (PSL_REV_ISSUE == 2 && pend_c == (int32_t)c && (t >> 5) == PSL_REV_WARP)
            cert_issue_dir(cs, tmem, (int32_t)c, 1, rv, pend_started, &ctl->mbar[c & 1], 0, kCCols, true);
        }
        if (PSL_REV_ISSUE != 2 && pend_c >= 0 && (t >> 5) == PSL_REV_WARP)
          cert_issue_dir(cs, tmem, pend_c, 1, pend_rv, pend_started, &ctl->mbar[pend_c & 1], 0, kCCols, true);
        }
        PT_MARK(0);
        // the tail chunks, streamed while the last MMAs drain
        cert_tail(io, c_end, nch, sm.sb, pmax, part);
        PT_MARK(10);
        for (uint32_t bb = 0; bb < 2; ++bb)
          if (issued & (1u << bb)) { mbar_wait(&ctl->mbar[bb], (mb_par >> bb) & 1u); mb_par ^= 1u << bb; }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        PT_MARK(16);
        // band-1 cells (the digit ring is free now; C of the band is folded and
        // written once every thread passed the barrier)
        if (io.m_hi > io.m_lo) {
          __syncthreads();
          PT_MARK(17);
          cert_band_records(io, cs, io.Cdst ? io.Cdst : io.Csrc, sm.sb);
          __syncthreads();
          PT_MARK(18);
          cert_band_rows(io, cs, Bs);
        }
        PT_MARK(6);
        // band-1 row sums to the row-interval scratch (read back by the row owners)
#pragma unroll
        for (int m = 0; m < kBandRows; ++m) {
          const uint32_t rho = kBandRows * t + m;
          if (rho >= r_lo && rho < r_hi) ivm[rho] = Bs[m];
        }
        if ((t & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->st.n_mma),
                                     (unsigned long long)nmma);
        if (t == 0) ctl->st.n_umma += numma;
        if (ovf) atomicOr(&ctl->c_ovf, 1);
        if (first && seg == 0) {
          if (io.chain && t == kCertThreads - 64) ctl->fit = chain;
          if (io.fsum) {
            double v = part[3];
            for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
            if ((t & 31) == 0) ctl->rs5[3][t >> 5] = v;
          }
          const int32_t Pn = block_max(ctl, pmax);   // (its barriers publish ctl->fit, rs5)
          if (t == 0) {
            if (io.fsum) {
              double S = 0.0;
              for (int x = 0; x < (int)(blockDim.x >> 5); ++x) S = __dadd_rn(S, ctl->rs5[3][x]);
              if (isfinite(S) && S < 0x1p1020) {
                // serial fitness in [S_exact (1 -+ g_L)], S_exact in S / (1 +- g_p): the
                // parallel sum's depth is L/kCC per thread + 5 + 16
                const double gL = gamma_n((double)L), gp = gamma_n((double)L / kCC + 24.0);
                const double u = 0x1p-53;
                first_pass_state(ctl, a, w, Pn, S, alpha);
                WalkState& St = ctl->st;
                St.vl_exact = 0;
                St.vl_lo = S * (1.0 - gL) / (1.0 + gp) * (1.0 - 8.0 * u);
                St.vl_hi = S * (1.0 + gL) / (1.0 - gp) * (1.0 + 8.0 * u);
              } else {
                // near or past DBL_MAX: the exact serial chain decides OverflowError
                double ch = 0.0;
                for (uint32_t k = 1; k < L; ++k) ch = __dadd_rn(ch, io.lut[abs(Cpiv[k])]);
                first_pass_state(ctl, a, w, Pn, ch, alpha);
              }
            } else {
              first_pass_state(ctl, a, w, Pn, ctl->fit, alpha);
            }
          }
        }
        // window constants: warp sums, then a fixed-order sum over warps
        {
          const int lane = t & 31, warp = t >> 5;
#pragma unroll
          for (int i = 0; i < 5; ++i) {
            double v = part[i];
            for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
            if (lane == 0) ctl->rs5[i][warp] = v;
          }
        }
#if PSL_XTMEM
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");   // cross accumulators in TMEM
#endif
        __syncthreads();                       // windows / cores are free: row arrays alias them
        double* linrow = cs.linrow;
        const double* xrow = cs.xrow;
#if PSL_XTMEM
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        cert_cross_rows(tmem, ctl->m_lo, ctl->c_unitR, cs.xrow);
#else
        cert_cross_rows(acc, ctl->c_unitR, cs.xrow);
#endif
#undef XACC
        double* linrev = reinterpret_cast<double*>(cs.dring);   // free: band 1 is done
        cert_lin_rows(tmem, started, ctl->c_unitH, io, linrow, linrev);
        double v5 = 0.0;                       // window constant i = t: its warp sums in fixed order
        if (t < 5)
          for (int x = 0; x < (int)(blockDim.x >> 5); ++x) v5 = __dadd_rn(v5, ctl->rs5[t][x]);
        __syncthreads();
        if (t < 5) ctl->rs5[t][0] = v5;
        __syncthreads();
        if (t == 0) {
          double sm5[5];
          for (int i = 0; i < 5; ++i) sm5[i] = ctl->rs5[i][0];
          const double u = 0x1p-53;
          const double Sc = __dadd_rn(__dadd_rn(sm5[0], sm5[1]), sm5[2]);
          ctl->c_sconst = Sc;
          ctl->c_errconst = 2.0 * gamma_n((double)L / 256.0 + 80.0) * Sc + 8.0 * u * sm5[0] +
                            64.0 * u * (2.0 * sm5[0] + sm5[1]) +   // sum|H4| <= S_P + S_M, sum|R4| <= S_P
                            (ctl->c_qH > 0 ? (double)L * ctl->c_unitH : 0.0) +
                            (ctl->c_qR > 0 ? (double)ctl->m_lo * ctl->c_unitR : 0.0) +
                            1024.0 * u * (double)L * (ctl->c_unitH + ctl->c_unitR);
        }
        __syncthreads();
        if (ctl->M_hi > ctl->M_lo) cert_band2_scan(io, ctl->M_hi - ctl->M_lo, reinterpret_cast<double*>(cs.rec));
        __syncthreads();
        if (t == 0 && ctl->M_hi > ctl->M_lo) {
          // scan rounding, absolute: relative to the band-2 totals
          const uint32_t nb2 = ctl->M_hi - ctl->M_lo;
          ctl->c_errconst += 4.0 * gamma_n(128.0) * (io.b2M[nb2 - 1] + io.b2E[0]);
        }
        __syncthreads();
        // per-row intervals [lo, hi] that provably hold the serial double V(j)
        {
          const double u = 0x1p-53;
          const double gL = gamma_n((double)L), gB = gamma_n(2100.0), g8 = gamma_n(8.0);
          const double Sc = ctl->c_sconst, E0 = ctl->c_errconst;
#pragma unroll
          for (int m = 0; m < kJ; ++m) {
            if (t < (uint32_t)kThreads) break;              // row owners: threads 256..511
            const uint32_t rho = kJ * (t - kThreads) + m;
            if (rho < r_lo || rho >= r_hi) continue;
            const uint32_t j = (uint32_t)(j0 + (int32_t)rho);
            const double lin = __dadd_rn(linrow[rho], linrev[rho]), xv = xrow[rho];
            const uint32_t Mj = max(j, L - 1 - j);
            const double B4 = __dadd_rn(__dmul_rn(4.0, ivm[rho]),   // band-1 sum, stored above
                                        cert_band2_const(io, ctl->M_hi - ctl->M_lo, Mj - ctl->M_lo));
            const int sj = sval(sm.sb, j);
            const double T4 = __dadd_rn(__dadd_rn(__dadd_rn(Sc, B4), sj > 0 ? lin : -lin), xv);
            const double Abs = Sc + B4 + fabs(lin) + fabs(xv);
            const double Err = E0 + 2.0 * gB * B4 + 2.0 * g8 * Abs + u * (fabs(lin) + fabs(xv)) +
                               a.cert_slack * Abs;
            const double hv = 0.25 * (T4 + Err) * (1.0 + gL) * (1.0 + 8.0 * u);
            PSL_CHK(rho < (uint32_t)kGroup, 31);
            ivm[rho] = isfinite(hv) ? 0.25 * T4 : __longlong_as_double(0x7ff8000000000000ll);   // -> bad
            ivl[rho] = fmax(0.0, 0.25 * (T4 - Err)) * (1.0 - gL) * (1.0 - 8.0 * u);
            ivh[rho] = hv;
          }
        }
        __syncthreads();
        PT_MARK(11);
      }
      if (first) {
        filter_hlist(ctl, sm, hlist);
        __syncthreads();
      }
      {
        bool active[kJ];
        uint32_t jj[kJ];
        const uint32_t owner = t >= (uint32_t)kThreads ? t - kThreads : 0u;
        const uint32_t ibase = g * kGroup + kJ * owner;
#pragma unroll
        for (int m = 0; m < kJ; ++m) {
          const uint32_t rho = kJ * owner + m;
          active[m] = t >= (uint32_t)kThreads && rho < gn;
          uint32_t j = gs + 1 + rho;
          if (j >= L) j -= L;
          jj[m] = j;
        }
        double mid[kJ], lo[kJ], hi[kJ];
#pragma unroll
        for (int m = 0; m < kJ; ++m) {
          const uint32_t rho = kJ * owner + m;
          mid[m] = active[m] ? ivm[rho] : 0.0;
          lo[m] = active[m] ? ivl[rho] : 0.0;
          hi[m] = active[m] ? ivh[rho] : 0.0;
        }
        reduce_group(ctl, sm, hlist, active, jj, mid, ibase, L);
        const uint32_t bi = ctl->best_i;
#pragma unroll
        for (int m = 0; m < kJ; ++m) {
          if (active[m] && ibase + m + 1 == bi) { ctl->gv_lo = lo[m]; ctl->gv_hi = hi[m]; }
          PSL_CHK(!(active[m] && ngrp > 1) || ibase + m < a.n, 32);
          if (active[m] && ngrp > 1) lo_all[ibase + m] = lo[m];
        }
        __syncthreads();
        if (t == 0) {   // combine groups in ascending offset order (strict <: smallest offset wins)
          if (first || ctl->best_v < ctl->cv) {
            ctl->cv = ctl->best_v; ctl->ci = ctl->best_i; ctl->cv_lo = ctl->gv_lo; ctl->cv_hi = ctl->gv_hi;
          }
          if (first || ctl->best_psl < ctl->cp) { ctl->cp = ctl->best_psl; ctl->cpi = ctl->best_pi; }
          ctl->cbad = first ? ctl->bad : (ctl->cbad | ctl->bad);
        }
        __syncthreads();
        if (g + 1 == ngrp) {
          // certified argmin: no other row's interval reaches below the best's upper bound
          const double hs = ctl->cv_hi;
          const uint32_t ci = ctl->ci;
          int amb = 0;
          if (ngrp == 1) {
#pragma unroll
            for (int m = 0; m < kJ; ++m) amb |= active[m] && ibase + m + 1 != ci && lo[m] <= hs;
          } else {
            for (uint32_t i = t; i < a.n; i += blockDim.x) amb |= i + 1 != ci && lo_all[i] <= hs;
          }
          amb = __syncthreads_or(amb);
          if (t == 0) {
            ctl->cv_exact = 0;
            const WalkState& S = ctl->st;
            int need = amb || ctl->cbad || ctl->c_ovf;
            if (!need) {
              ctl->cmp = compare_local(S, ctl->cv_lo, ctl->cv_hi, false, ctl->cv);
              need = ctl->cmp == 2;
            }
            ctl->st.n_cert += need ? 0 : 1;
            ctl->st.n_refine += need ? 1 : 0;
            if (a.cert_check && ngrp == 1) {
              // check mode: remember the certified decision, re-score exactly anyway
              ctl->chk_on = 1; ctl->chk_dec = !need; ctl->chk_ci = ctl->ci;
              ctl->chk_cmp = need ? 2 : ctl->cmp;
              need = 1;
            }
            ctl->need_exact = need;
          }
          __syncthreads();
        }
      }
      }   // groups
      PT_MARK(12);
      if (ctl->need_exact) {
        // exact re-score of the same pivot (flips already folded into Cpiv), in
        // groups of kJ * blockDim.x rows combined in ascending offset order
        const uint32_t rows_per = kJ * blockDim.x;
        const uint32_t ng2 = (a.n + rows_per - 1) / rows_per;
        for (uint32_t g2 = 0; g2 < ng2; ++g2) {
          const uint32_t ibase = g2 * rows_per + (t >> 5) * (32 * kJ) + (t & 31) * kJ;
          bool active[kJ];
          uint32_t jj[kJ];
#pragma unroll
          for (int m = 0; m < kJ; ++m) {
            const uint32_t i = ibase + m + 1;
            active[m] = i <= a.n;
            uint32_t j = 0;
            if (active[m]) { j = (uint32_t)(((uint64_t)start + i) % L); }
            jj[m] = j;
          }
          SweepIO sio;
          sio.L = L; sio.nwords = nw; sio.nchunks = a.nchunks;
          sio.alpha = alpha; sio.lut = lut; sio.lut_size = a.lut_n;
          sio.scan = true; sio.hcount = &ctl->hcount;
          sio.Csrc = Cpiv; sio.Cdst = nullptr; sio.Cloc = nullptr;
          sio.flips = flips; sio.F = 0; sio.hlist = nullptr; sio.hthr = 0; sio.chain = false;
          int32_t pm = 0;
          double chain = 0.0;
          double val[kJ];
          sweep(sio, sm, active, jj, val, pm, chain);
          if (ctl->chk_on) {
            // every row's serial double against its certified interval (one group:
            // row rho = offset - 1 = ibase + m, intervals still in iv_buf)
            const double* ivm = a.iv_buf + (size_t)w * 3 * kGroup;
            const double* ivl = ivm + kGroup;
            const double* ivh = ivl + kGroup;
            uint32_t rows = 0, viol = 0;
            double tight = 0.0, relw = 0.0;
#pragma unroll
            for (int m = 0; m < kJ; ++m) {
              if (!active[m]) continue;
              const uint32_t rho = ibase + m;
              const double md = ivm[rho], lo = ivl[rho], hi = ivh[rho], v = val[m];
              if (!isfinite(md) || !isfinite(v)) continue;   // non-finite rows go exact by design
              ++rows;
              if (!(v >= lo && v <= hi)) ++viol;
              const double half = v >= md ? hi - md : md - lo;
              if (half > 0.0) tight = fmax(tight, fabs(v - md) / half);
              if (md > 0.0) relw = fmax(relw, (hi - lo) / md);
            }
            if (rows) {
              atomicAdd(&ctl->chk_rows, rows);
              if (viol) atomicAdd(&ctl->chk_viol, viol);
              atomicMax(&ctl->chk_tight, (unsigned long long)__double_as_longlong(tight));
              atomicMax(&ctl->chk_relw, (unsigned long long)__double_as_longlong(relw));
            }
          }
          reduce_group(ctl, sm, hlist, active, jj, val, ibase, L);
          if (t == 0) {
            if (g2 == 0 || ctl->best_v < ctl->cv) { ctl->cv = ctl->best_v; ctl->ci = ctl->best_i; }
            if (g2 == 0 || ctl->best_psl < ctl->cp) { ctl->cp = ctl->best_psl; ctl->cpi = ctl->best_pi; }
            ctl->cbad = g2 == 0 ? ctl->bad : (ctl->cbad | ctl->bad);
          }
          __syncthreads();
        }
        if (t == 0) {
          ctl->cv_exact = 1; ctl->cv_lo = ctl->cv; ctl->cv_hi = ctl->cv;
          ctl->cmp = compare_local(ctl->st, ctl->cv, ctl->cv, true, ctl->cv);
          ctl->need_vl = !ctl->cbad && ctl->cmp == 2;
        }
        __syncthreads();
      }
    } else {
      // ================= exact pass(es)
      for (uint32_t g = 0; g < ngroups; ++g) {
        // this thread's kJ adjacent neighbours: offsets i = base + 1 .. base + kJ
        const uint32_t ibase = g * kGroup + (t >> 5) * (32 * kJ) + (t & 31) * kJ;
        bool active[kJ];
        uint32_t jj[kJ];
#pragma unroll
        for (int m = 0; m < kJ; ++m) {
          const uint32_t i = ibase + m + 1;
          active[m] = do_scan && i <= a.n;
          uint32_t j = 0;
          if (active[m]) { j = start + i; if (j >= L) j -= L; }
          jj[m] = j;
        }
        SweepIO io;
        io.L = L; io.nwords = nw; io.nchunks = a.nchunks;
        io.alpha = alpha; io.lut = lut; io.lut_size = a.lut_n;
        io.scan = do_scan;
        io.hcount = &ctl->hcount;
        if (g == 0) {
          io.Csrc = s_src_local ? Cloc : Cpiv;
          io.Cdst = Cpiv;
          io.Cloc = s_local_pending ? Cloc : nullptr;
          io.flips = flips; io.F = s_n_pending;
          io.hlist = hlist;
          io.hthr = s_Psrc - 4 * (int32_t)s_n_pending - 8;
          io.chain = s_fitness_pending != 0;
        } else {
          io.Csrc = Cpiv; io.Cdst = nullptr; io.Cloc = nullptr;
          io.flips = flips; io.F = 0; io.hlist = nullptr; io.hthr = 0; io.chain = false;
        }
        int32_t pmax = 0;
        double chain = 0.0;
        double val[kJ];
        sweep(io, sm, active, jj, val, pmax, chain);
        if (g == 0) {
          const int32_t Pn = block_max(ctl, pmax);
          if (t == 0) first_pass_state(ctl, a, w, Pn, chain, alpha);
          __syncthreads();
          if (ctl->st.status != PSL_OK) break;
          filter_hlist(ctl, sm, hlist);
          __syncthreads();
        }
        if (!do_scan) break;
        reduce_group(ctl, sm, hlist, active, jj, val, ibase, L);
        if (t == 0) {
          // combine groups in ascending offset order (strict <: smallest offset wins)
          if (g == 0) {
            ctl->cv = ctl->best_v; ctl->ci = ctl->best_i;
            ctl->cp = ctl->best_psl; ctl->cpi = ctl->best_pi; ctl->cbad = ctl->bad;
          } else {
            if (ctl->best_v < ctl->cv) { ctl->cv = ctl->best_v; ctl->ci = ctl->best_i; }
            if (ctl->best_psl < ctl->cp) { ctl->cp = ctl->best_psl; ctl->cpi = ctl->best_pi; }
            ctl->cbad |= ctl->bad;
          }
        }
        __syncthreads();
      }
      if (t == 0 && do_scan && ctl->st.status == PSL_OK) {
        ctl->cv_exact = 1; ctl->cv_lo = ctl->cv; ctl->cv_hi = ctl->cv;
        ctl->cmp = compare_local(ctl->st, ctl->cv, ctl->cv, true, ctl->cv);
        ctl->need_vl = !ctl->cbad && ctl->cmp == 2;
      }
      __syncthreads();
    }
    if (ctl->st.status != PSL_OK || !do_scan) break;

    if (ctl->need_vl) {
      // value_local is only known as an interval: its exact value is the serial
      // fitness of the local snapshot table (the argmin neighbour's chain is
      // fitness() of the moved table, term for term)
      const bool none[kJ] = {false, false, false, false};
      const uint32_t zj[kJ] = {0, 0, 0, 0};
      SweepIO sio;
      sio.L = L; sio.nwords = nw; sio.nchunks = a.nchunks;
      sio.alpha = alpha; sio.lut = lut; sio.lut_size = a.lut_n;
      sio.scan = false; sio.hcount = &ctl->hcount;
      // (not yet materialised: the local best is the pivot, whose table this
      // step's pass just wrote to Cpiv)
      sio.Csrc = ctl->st.loc_at_pivot ? Cpiv : Cloc; sio.Cdst = nullptr; sio.Cloc = nullptr;
      sio.flips = flips; sio.F = 0; sio.hlist = nullptr; sio.hthr = 0; sio.chain = true;
      int32_t pm = 0;
      double chain = 0.0;
      double val[kJ];
      sweep(sio, sm, none, zj, val, pm, chain);
      if (t == 0) {
        WalkState& S = ctl->st;
        S.value_local = chain; S.vl_exact = 1; S.vl_lo = chain; S.vl_hi = chain;
        S.n_vlchain += 1;
        ctl->cmp = compare_local(S, ctl->cv, ctl->cv, true, ctl->cv);
      }
      __syncthreads();
    }

    if (kCert && t == 0 && ctl->chk_on) {
      WalkState& S = ctl->st;
      S.chk_steps += 1;
      S.chk_rows += ctl->chk_rows;
      S.chk_viol += ctl->chk_viol;
      if (ctl->chk_dec) {
        S.chk_dec += 1;
        S.chk_dec_bad += (ctl->chk_ci != ctl->ci || ctl->chk_cmp != ctl->cmp) ? 1 : 0;
      }
      S.chk_tight = fmax(S.chk_tight, __longlong_as_double((long long)ctl->chk_tight));
      S.chk_relw = fmax(S.chk_relw, __longlong_as_double((long long)ctl->chk_relw));
    }

    // ---- reduce_scan result + Algorithm 1 control (search.cpp:379-419)
    PT_MARK(13);
    if (t == 0) {
      WalkState& S = ctl->st;
      S.nse += a.n;                                            // :379
      const double value_step = ctl->cv;
      const uint32_t best_i = ctl->ci;
      const int32_t psl_min = ctl->cp;
      const uint32_t psl_i = ctl->cpi;
      const double elapsed = (double)(globaltimer() - S.t0_ns) * 1e-9;
      ctl->imp = ctl->improve = ctl->restart = 0;
      if (ctl->cbad) {                                      // :275-281
        S.status = PSL_ERR_OVERFLOW; S.err_kind = 2; S.err_alpha = alpha;
      } else {
        auto emit = [&](uint32_t kind) {
          if (a.record_events) {
            psl_event& ev = a.events[(size_t)w * a.events_cap + S.n_events];
            ev.nse = S.nse; ev.elapsed_seconds = elapsed; ev.psl_best = S.psl_best;
            ev.phase_index = S.phase; ev.kind = kind;
          }
          ++S.n_events;
        };
        const uint32_t jstar = (uint32_t)(((uint64_t)start + best_i) % L);
        const uint32_t ppos = (uint32_t)(((uint64_t)start + psl_i) % L);
        ctl->jstar = jstar; ctl->ppos = ppos;
        if (psl_min < S.psl_best) {                            // :383-389
          S.psl_best = psl_min;
          ctl->imp = 1;
          emit(PSL_EVENT_IMPROVED_PSL);
        }
        if (ctl->cmp < 0) {                                    // :394-399
          S.value_local = value_step;
          S.vl_exact = ctl->cv_exact; S.vl_lo = ctl->cv_lo; S.vl_hi = ctl->cv_hi;
          S.unimproved = 0;
          ctl->improve = 1;
          emit(PSL_EVENT_LOCAL_BEST_IMPROVED);
        } else if (ctl->cmp > 0) {                             // :400-413
          if (++S.unimproved > a.ls_lmt) {
            ctl->restart = 1;
            S.phase = (S.phase == 1) ? 2u : 1u;
            S.nse += 1;
            S.unimproved = 0;
            S.switches += 1;
            S.fitness_pending = 1;
            S.switch_pending = 1;
            emit(PSL_EVENT_PHASE_SWITCH);
          }
        }
        if (a.record_traces) {                                 // :417-419
          psl_trace& tr = a.traces[(size_t)w * a.traces_cap + S.n_traces];
          tr.nse = S.nse; tr.value_step = value_step; tr.value_local = S.value_local;
          tr.psl_best = S.psl_best; tr.phase_index = S.phase;
          ++S.n_traces;
          S.trace_patch = ctl->restart ? 1u : 0u;
        }
        S.steps += 1;
        ctl->steps_this_launch += 1;
      }
    }
    __syncthreads();
    if (ctl->st.status != PSL_OK) break;

    if (ctl->imp) {
      // best_seq = pivot with the best-PSL neighbour's flip (:385-387)
      const uint32_t pp = ctl->ppos;
      for (uint32_t i = t; i < nw; i += blockDim.x) {
        uint32_t v = bits_piv[i + 1];
        if (i == (pp >> 5)) v ^= 1u << (pp & 31);
        bits_best[i + 1] = v;
      }
      const long long e = energy_sweep(ctl, Cpiv, L, sm.sb, (int64_t)pp);
      if (t == 0) ctl->st.energy_best = e;
    }
    __syncthreads();
    // Local-best snapshot (search.cpp:394-399), materialised lazily: while the
    // walk keeps improving the local best IS the pivot and nothing is copied.
    // The first non-improving move leaves it behind: its bits are the pivot's
    // before this move, its table the next pass's pre-fold C (no 4 MB copy per
    // improving step).  A restart needs >= 2 worsening steps after the last
    // improvement (ls_lmt >= 1), so the snapshot is materialised before any
    // restart reads it.
    const bool materialise = !ctl->restart && !ctl->improve && ctl->st.loc_at_pivot;
    if (materialise)
      for (uint32_t i = t; i < nw; i += blockDim.x) bits_loc[i + 1] = bits_piv[i + 1];
    __syncthreads();
    if (ctl->restart) {
      // back to the phase-local best (:405-406): bits from the snapshot, C via
      // the next pass (src_local); then flip_random_distinct (:407, :131-148)
      for (uint32_t i = t; i < nw; i += blockDim.x) bits_piv[i + 1] = bits_loc[i + 1];
      __syncthreads();
      if (t == 0) {
        WalkState& S = ctl->st;
        uint32_t done = 0;
        while (done < a.flip_lmt) {
          const uint32_t pos = (uint32_t)rng_bounded(S.rng, L);
          const uint32_t bit = 1u << (pos & 31);
          if (used[pos >> 5] & bit) continue;
          used[pos >> 5] |= bit;
          flips[done++] = pos;
          bits_piv[(pos >> 5) + 1] ^= bit;
        }
        for (uint32_t m = 0; m < done; ++m) used[flips[m] >> 5] = 0u;
        S.n_pending = done;
        S.src_local = 1;
      }
    } else if (t == 0) {
      // the pivot always moves to the argmin neighbour (:392)
      const uint32_t js = ctl->jstar;
      bits_piv[(js >> 5) + 1] ^= 1u << (js & 31);
      flips[0] = js;
      ctl->st.n_pending = 1;
      ctl->st.src_local = 0;
      if (ctl->improve) {
        ctl->st.loc_at_pivot = 1;
      } else if (materialise) {
        ctl->st.loc_at_pivot = 0;
        ctl->st.local_pending = 1;
      }
    }
    if (ctl->restart && t == 0) ctl->st.loc_at_pivot = 0;
    __syncthreads();
    PT_MARK(14);
  }

  // ---- persist
  PT_MARK(7);
  __syncthreads();
#ifdef PSL_PHASE_TIMING
  if (kCert && t == 0) printf("PTCTA %u %lld\n", w, clock64() - pt_t0);
  if (kCert && w == 0 && t < 16) {
    const long long* q = pt_acc[t];
    printf("PT warp %2u top %lld build %lld cores %lld bar %lld issue %lld cross %lld band %lld prologue %lld mbarwait %lld fence %lld "
           "tail %lld rows %lld reduce %lld exact %lld control %lld steptop %lld epimbar %lld episync %lld epirec %lld\n", t,
           q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7], q[8], q[9], q[10], q[11], q[12], q[13], q[14], q[15],
           q[16], q[17], q[18]);
  }
#endif
  if (t == 0) {
    if (ctl->st.status != PSL_OK) ctl->st.end_ns = globaltimer();
    *gst = ctl->st;
  }
  if (a.sol_out && ctl->st.done && ctl->st.status == PSL_OK) {
    // the walk's best sequence as int8 +-1 straight into the caller's pinned
    // host buffer (unpack_kernel's encoding), 16-byte stores over PCIe
    int8_t* o = a.sol_out + (size_t)w * L;
    const uint32_t* bb = bits_best + 1;
    const uint32_t head = min(L, (uint32_t)((16u - ((uintptr_t)o & 15u)) & 15u));
    const uint32_t nvec = (L - head) >> 4;
    for (uint32_t i = t; i < head; i += blockDim.x) o[i] = ((bb[i >> 5] >> (i & 31)) & 1u) ? (int8_t)-1 : (int8_t)1;
    for (uint32_t v = t; v < nvec; v += blockDim.x) {
      const uint32_t j = head + 16 * v;
      const uint32_t b16 = __funnelshift_r(bb[j >> 5], bb[(j >> 5) + 1], j & 31) & 0xffffu;
      uint32_t q[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) q[k] = 0x01010101u + (((b16 >> (4 * k)) & 0xfu) * 0x00204081u & 0x01010101u) * 0xfeu;
      *reinterpret_cast<uint4*>(o + j) = make_uint4(q[0], q[1], q[2], q[3]);
    }
    for (uint32_t i = head + 16 * nvec + t; i < L; i += blockDim.x)
      o[i] = ((bb[i >> 5] >> (i & 31)) & 1u) ? (int8_t)-1 : (int8_t)1;
  }
  if (kCert && t < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(ctl->tmem), "r"(kTmemCols) : "memory");
  }
}

// tcgen05.mma kind::i8 M128 N64 K32 issue rate (the certified scan's MMA shape):
// one CTA per SM, one thread issues `per` MMAs back to back per commit.
__global__ void __launch_bounds__(128) probe_umma_kernel(int reps, int per, int* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  for (int i = threadIdx.x; i < 8192 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem_raw)[i] = make_uint4(0x01010101u * (i & 3), 0u, 0x02020202u, 0u);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(64) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = smem_u32(smem_raw);
  uint32_t par = 0;
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      // the certified scan's descriptors and K-step walk (16 steps of 512 B of A, 256 B of B)
      const uint64_t da = umma_desc(base, 256, 128), db = umma_desc(base + 4096, 128, 1024);
      for (int i = 0; i < per; ++i)
        umma_i8(tmem_base, da + (uint64_t)((i & 15) * (512 >> 4)), db + (uint64_t)((i & 15) * (256 >> 4)),
                i > 0 ? 1u : 0u);
      umma_commit(&mbar);
    }
    mbar_wait(&mbar, par);
    par ^= 1u;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(64) : "memory");
  if (threadIdx.x == 0 && reps < 0) out[0] = 1;
}

// ScanJob / neighborhood_scan: neighbours of one given pivot, kGroup per CTA,
// terms from the caller's PowerTable.
__global__ void __launch_bounds__(kThreads, 2) scan_kernel(ScanArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem sm = carve<false>(smem_raw);
  const uint32_t t = threadIdx.x;
  const uint32_t nw = a.nwords;
  sm.sb = a.bits;     // padded: word i at a.bits[i + 1]
  const uint32_t hcount = *a.hcount;
  const bool in_smem = hcount <= (uint32_t)kHCap;
  if (in_smem)
    for (uint32_t e = t; e < hcount; e += kThreads) sm.hf[e] = a.hlist[e];
  __syncthreads();
  const uint32_t ibase = blockIdx.x * kGroup + (t >> 5) * (32 * kJ) + (t & 31) * kJ;
  bool active[kJ];
  uint32_t jj[kJ];
#pragma unroll
  for (int m = 0; m < kJ; ++m) {
    const uint32_t i = ibase + m + 1;
    active[m] = i <= a.n;
    uint32_t j = 0;
    if (active[m]) { j = a.start + i; if (j >= a.L) j -= a.L; }
    jj[m] = j;
  }
  SweepIO io;
  io.L = a.L; io.nwords = nw; io.nchunks = a.nchunks;
  io.Csrc = a.C; io.Cdst = nullptr; io.Cloc = nullptr; io.flips = nullptr; io.F = 0;
  io.alpha = 0; io.lut = a.lut; io.lut_size = a.lut_size;
  io.hlist = nullptr; io.hcount = nullptr; io.hthr = 0;
  io.scan = true; io.chain = false;
  int32_t pmax = 0;
  double chain = 0.0;
  double v[kJ];
  sweep(io, sm, active, jj, v, pmax, chain);
#pragma unroll
  for (int m = 0; m < kJ; ++m) {
    if (!active[m]) continue;
    const uint32_t i = ibase + m + 1;
    const int32_t p = in_smem ? neighbour_psl(sm.hf, hcount, 0, true, jj[m], a.L, sm.sb)
                              : neighbour_psl(a.hlist, hcount, 0, true, jj[m], a.L, sm.sb);
    a.values[i] = v[m];
    a.psls[i] = p;
  }
}

// The ScanJob seam's pivot PSL (max |C_k|, sequence.cpp:84-93) and the list of
// shifts that can carry a neighbour's peak (|C_k| >= PSL - 8), on the device.
__global__ void scan_psl_kernel(const int32_t* C, uint32_t L, int32_t* P) {
  int32_t pm = 0;
  for (uint32_t k = 1 + blockIdx.x * blockDim.x + threadIdx.x; k < L; k += gridDim.x * blockDim.x)
    pm = max(pm, abs(C[k]));
  pm = warp_max(pm);
  if ((threadIdx.x & 31) == 0 && pm > 0) atomicMax(P, pm);
}
__global__ void scan_hlist_kernel(const int32_t* C, uint32_t L, const int32_t* P, int2* h,
                                  uint32_t* count) {
  const int32_t thr = *P - 8;
  for (uint32_t k = 1 + blockIdx.x * blockDim.x + threadIdx.x; k < L; k += gridDim.x * blockDim.x) {
    const int32_t c = C[k];
    if (abs(c) >= thr) h[atomicAdd(count, 1u)] = make_int2((int)k, c);
  }
}

// apply_flip (sequence.cpp:198-224) for the C-ABI: C_k += delta_k, then s_j flips.
__global__ void apply_flip_kernel(uint32_t* bits, int32_t* C, uint32_t L, uint32_t j) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x + 1;
  auto sv = [&](uint32_t x) { return 1 - 2 * (int)((bits[x >> 5] >> (x & 31)) & 1u); };
  if (k < L) {
    int acc = 0;
    if (k <= j) acc += sv(j - k);
    if (j + k < L) acc += sv(j + k);
    C[k] += -2 * sv(j) * acc;
  }
}
__global__ void flip_bit_kernel(uint32_t* bits, uint32_t j) { bits[j >> 5] ^= 1u << (j & 31); }

// flip_deltas (sequence.cpp:154-172): out[0] = 0, out[k] = -2 s_j (s_{j-k} [k <= j]
// + s_{j+k} [j + k < L]) on the sequence before the flip; one shift per thread.
__global__ void flip_deltas_kernel(const uint32_t* bits, uint32_t L, uint32_t j, int32_t* out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  auto sv = [&](uint32_t x) { return 1 - 2 * (int)((bits[x >> 5] >> (x & 31)) & 1u); };
  if (k >= L) return;
  if (k == 0) { out[0] = 0; return; }
  int acc = 0;
  if (k <= j) acc += sv(j - k);
  if (j + k < L) acc += sv(j + k);
  out[k] = -2 * sv(j) * acc;
}

// fitness(table, PowerTable) (sequence.cpp:131-141): the reference's serial
// ascending-k double chain, one thread (the order is the result); C_k and the
// table entries are loaded 8 shifts ahead of the dependent adds.
__global__ void fitness_chain_kernel(const int32_t* C, uint32_t L, const double* lut, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double sum = 0.0;
  uint32_t k = 1;
  for (; k + 8 <= L; k += 8) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(lut + abs(__ldg(C + k + i)));
#pragma unroll
    for (int i = 0; i < 8; ++i) sum = __dadd_rn(sum, v[i]);
  }
  for (; k < L; ++k) sum = __dadd_rn(sum, __ldg(lut + abs(__ldg(C + k))));
  *out = sum;
}

// PowerTable(L, alpha) for both phases (sequence.hpp:72-84): lut[a] = pow_int(a, alpha)
__global__ void power_tables_kernel(double* lut, uint32_t n, uint32_t alpha1, uint32_t alpha2) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    lut[i] = pow_int_dev((double)i, alpha1);
    lut[n + i] = pow_int_dev((double)i, alpha2);
  }
}

}  // namespace

size_t run_smem_bytes(bool cert) {
  const size_t main_bytes = cert ? (kExactMain > kCertRegion ? kExactMain : kCertRegion) : kExactMain;
  return main_bytes + kHfBytes + kCtlBytes + (cert ? (size_t)kLutS * sizeof(double) : 0);
}

RunArgs walk_offset(const RunArgs& a, uint32_t w0) {
  RunArgs b = a;
  b.st += w0;
  b.Cpiv += (size_t)w0 * a.c_stride;
  b.Cloc += (size_t)w0 * a.c_stride;
  b.bits_piv += (size_t)w0 * a.w_stride;
  b.bits_loc += (size_t)w0 * a.w_stride;
  b.bits_best += (size_t)w0 * a.w_stride;
  b.used += (size_t)w0 * a.w_stride;
  b.hlist += (size_t)w0 * a.h_stride;
  b.flips += (size_t)w0 * a.f_stride;
  return b;
}

int launch_init_walks(const RunArgs& a, uint32_t n_walks, const uint64_t* d_seeds,
                      const uint32_t* d_packed, size_t packed_stride, cudaStream_t s) {
  const bool jump = !d_packed && a.L > kSpinChunk;
  if (jump) rng_jump_kernel<<<1, 256, 0, s>>>();
  init_walks_kernel<<<n_walks, 256, 0, s>>>(a, d_seeds, d_packed, packed_stride);
  return launch_status(jump ? 2 : 1);
}

int launch_build_tables(const RunArgs& a, uint32_t n_walks, cudaStream_t s) {
  const uint32_t per_block = 8 * 32 * kTabR;
  dim3 grid((a.L + per_block - 1) / per_block, n_walks);
  build_tables_kernel<<<grid, 256, 0, s>>>(a.bits_piv + a.w_front + 1, a.w_stride, a.Cpiv, a.Cloc,
                                           a.c_stride, a.L, a.st);
  return launch_status(1);
}

int launch_table_only(const uint32_t* d_bits, int32_t* d_C, uint32_t L, uint32_t nwords,
                      cudaStream_t s) {
  const uint32_t per_block = 8 * 32 * kTabR;
  dim3 grid((L + per_block - 1) / per_block, 1);
  build_tables_kernel<<<grid, 256, 0, s>>>(d_bits, nwords + kBitsPad, d_C, nullptr, L, L, nullptr);
  return launch_status(1);
}

// The dynamic shared-memory opt-in is a per-device function attribute: set it
// once per device (a context may live on any GPU; several host threads may make
// their first launch together).
constexpr int kMaxDevices = 64;
static bool smem_opt_in(const void* fn, size_t bytes, std::atomic<uint32_t> (&done)[kMaxDevices]) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return false;
  if (done[dev].load(std::memory_order_acquire) == bytes) return true;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) { launch_fail(e); return false; }
  done[dev].store((uint32_t)bytes, std::memory_order_release);
  return true;
}
static std::atomic<uint32_t> g_attr_run_cert[kMaxDevices], g_attr_run_exact[kMaxDevices], g_attr_scan[kMaxDevices];

int launch_run(const RunArgs& a, uint32_t n_walks, cudaStream_t s) {
  if (a.cert) {
    if (!smem_opt_in((const void*)run_kernel<true>, run_smem_bytes(true), g_attr_run_cert)) return -1;
    run_kernel<true><<<n_walks, 2 * kThreads, run_smem_bytes(true), s>>>(a);
  } else {
    if (!smem_opt_in((const void*)run_kernel<false>, run_smem_bytes(false), g_attr_run_exact)) return -1;
    run_kernel<false><<<n_walks, kThreads, run_smem_bytes(false), s>>>(a);
  }
  return launch_status(1);
}

int launch_scan(const ScanArgs& a, cudaStream_t s) {
  const size_t smem = run_smem_bytes(false);
  if (!smem_opt_in((const void*)scan_kernel, smem, g_attr_scan)) return -1;
  const uint32_t pg = std::min<uint32_t>((a.L + 255) / 256, 1184);
  cudaError_t e = cudaMemsetAsync(a.P, 0, 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(a.hcount, 0, 4, s);
  if (e != cudaSuccess) return launch_fail(e);
  scan_psl_kernel<<<pg, 256, 0, s>>>(a.C, a.L, a.P);
  scan_hlist_kernel<<<pg, 256, 0, s>>>(a.C, a.L, a.P, a.hlist, a.hcount);
  const uint32_t groups = (a.n + kGroup - 1) / kGroup;
  scan_kernel<<<groups, kThreads, smem, s>>>(a);
  return launch_status(3);
}

int launch_power_tables(double* lut, uint32_t lut_n, uint32_t alpha1, uint32_t alpha2,
                        cudaStream_t s) {
  power_tables_kernel<<<(lut_n + 255) / 256, 256, 0, s>>>(lut, lut_n, alpha1, alpha2);
  return launch_status(1);
}

int launch_apply_flip(uint32_t* d_bits, int32_t* d_C, uint32_t L, uint32_t j, cudaStream_t s) {
  apply_flip_kernel<<<(L + 255) / 256, 256, 0, s>>>(d_bits, d_C, L, j);
  flip_bit_kernel<<<1, 1, 0, s>>>(d_bits, j);
  return launch_status(2);
}

int launch_flip_deltas(const uint32_t* d_bits, uint32_t L, uint32_t j, int32_t* d_out, cudaStream_t s) {
  flip_deltas_kernel<<<(L + 255) / 256, 256, 0, s>>>(d_bits, L, j, d_out);
  return launch_status(1);
}

int launch_fitness_chain(const int32_t* d_C, uint32_t L, const double* d_lut, double* d_out,
                         cudaStream_t s) {
  fitness_chain_kernel<<<1, 32, 0, s>>>(d_C, L, d_lut, d_out);
  return launch_status(1);
}

}  // namespace pslb

// ---------------------------------------------------------------- probes
// Roofline denominators measured live (bench.py): the FP64 add pipe (the
// serial fitness chain needs exactly one dependent DADD per cell) and the
// divergent-LDS.64 + DADD rate of a per-cell table-lookup loop.
namespace pslb {
namespace {
__global__ void __launch_bounds__(1024, 1) probe_dadd_kernel(int reps, double* out, long long* cyc) {
  double s1 = threadIdx.x * 1e-3, s2 = 0.5, s3 = 0.25, s4 = 1.0;
  const double x = 1.0000001 + threadIdx.x * 1e-9;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      s1 = __dadd_rn(s1, x); s2 = __dadd_rn(s2, x); s3 = __dadd_rn(s3, x); s4 = __dadd_rn(s4, x);
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s1 + s2 + s3 + s4;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void __launch_bounds__(1024, 1) probe_lds_kernel(int reps, double* out, long long* cyc) {
  __shared__ __align__(16) double tab[512 * 8];
  for (int i = threadIdx.x; i < 512 * 8; i += blockDim.x) tab[i] = 1.0 + (i & 7) * 0.25;
  __syncthreads();
  uint32_t w = 0x9E3779B9u * (threadIdx.x + 1);
  double sum = 0.0;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll 1
    for (int kb = 0; kb < 512; kb += 16) {
      const char* rb = reinterpret_cast<const char*>(tab + kb * 8);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const uint32_t v = q < 2 ? (w << (3 - 2 * q)) : (w >> (2 * q - 3));
        sum = __dadd_rn(sum, *reinterpret_cast<const double*>(rb + q * 64 + (v & 0x18u)));
      }
      w = w * 1664525u + 1013904223u;
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
}  // namespace

// legacy tensor pipe: mma.sync m16n8k32 s8 throughput (8 independent accumulators per warp)
__global__ void __launch_bounds__(256) probe_imma_kernel(int reps, int* out) {
  uint32_t a0 = 0x01010101u * (threadIdx.x + 1), a1 = a0 ^ 0x5a5a5a5au, a2 = ~a0, a3 = a0 + 7;
  const uint32_t b0 = 0x03030303u * threadIdx.x, b1 = ~b0;
  int d[8][4] = {};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(d[q][0]), "+r"(d[q][1]), "+r"(d[q][2]), "+r"(d[q][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    a0 += 1;
  }
  int s = 0;
  for (int q = 0; q < 8; ++q) s += d[q][0] + d[q][1] + d[q][2] + d[q][3];
  if (s == 0x7fffffff) out[0] = s;
}

int probe_umma(int nsm, cudaStream_t s, double* mma_per_s) {
  int* out = nullptr;
  cudaError_t e = cudaMalloc(&out, 64);
  if (e != cudaSuccess) return launch_fail(e);
  if ((e = cudaFuncSetAttribute(probe_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384)) != cudaSuccess) {
    cudaFree(out);
    return launch_fail(e);
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 400, per = 256;
  probe_umma_kernel<<<nsm, 128, 16384, s>>>(4, per, out);
  cudaEventRecord(a, s);
  probe_umma_kernel<<<nsm, 128, 16384, s>>>(reps, per, out);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *mma_per_s = (double)nsm * reps * per / (ms * 1e-3);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  return launch_status(2);
}

int probe_imma(int nsm, cudaStream_t s, double* mma_per_s) {
  int* out = nullptr;
  if (const cudaError_t e = cudaMalloc(&out, 64); e != cudaSuccess) return launch_fail(e);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 2048, blocks = nsm * 4;
  probe_imma_kernel<<<blocks, 256, 0, s>>>(8, out);
  cudaEventRecord(a, s);
  probe_imma_kernel<<<blocks, 256, 0, s>>>(reps, out);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *mma_per_s = (double)blocks * 8 * reps * 8 / (ms * 1e-3);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  return launch_status(2);
}

int probe_peaks(int nsm, cudaStream_t s, double* dadd_cps, double* lds_cps, double* mhz) {
  double* out = nullptr;
  long long* cyc = nullptr;
  if (const cudaError_t e = cudaMalloc(&out, sizeof(double) * nsm * 1024); e != cudaSuccess) return launch_fail(e);
  if (const cudaError_t e = cudaMalloc(&cyc, sizeof(long long) * nsm); e != cudaSuccess) { cudaFree(out); return launch_fail(e); }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 2000;
  float ms = 0.f;
  long long c0 = 0;
  probe_dadd_kernel<<<nsm, 1024, 0, s>>>(10, out, cyc);
  cudaEventRecord(a, s);
  probe_dadd_kernel<<<nsm, 1024, 0, s>>>(reps, out, cyc);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  *dadd_cps = (double)nsm * 1024 * reps * 64 / (ms * 1e-3);
  *mhz = (double)c0 / (ms * 1e-3) / 1e6;
  probe_lds_kernel<<<nsm, 1024, 0, s>>>(10, out, cyc);
  cudaEventRecord(a, s);
  probe_lds_kernel<<<nsm, 1024, 0, s>>>(reps / 10, out, cyc);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  *lds_cps = (double)nsm * 1024 * (reps / 10) * 512 / (ms * 1e-3);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  cudaFree(cyc);
  return launch_status(4);
}
}  // namespace pslb

namespace pslb {
namespace {
// bit-packed best sequences -> int8 +-1 (one walk per blockIdx.y)
__global__ void unpack_kernel(const uint32_t* bits, size_t w_stride, uint32_t L, int8_t* out) {
  const uint32_t w = blockIdx.y;
  const uint32_t* b = bits + (size_t)w * w_stride;   // caller passes word 0 of walk 0
  int8_t* o = out + (size_t)w * L;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x)
    o[i] = ((b[i >> 5] >> (i & 31)) & 1u) ? (int8_t)-1 : (int8_t)1;
}
}  // namespace
int launch_unpack(const uint32_t* bits, size_t w_stride, uint32_t L, uint32_t n_walks, int8_t* out,
                  cudaStream_t s) {
  unpack_kernel<<<dim3(std::min<uint32_t>((L + 255) / 256, 512), n_walks), 256, 0, s>>>(bits, w_stride, L, out);
  return launch_status(1);
}
}  // namespace pslb

namespace pslb {
namespace {
// oracle::verify_sequence (oracle.cpp:172-197) reductions over a device table:
// PSL, exact energy, |C_k| histogram (k = 1..L-1).
__global__ void verify_kernel(const int32_t* C, uint32_t L, int32_t* psl, unsigned long long* energy,
                              unsigned long long* hist) {
  int32_t pm = 0;
  unsigned long long en = 0;
  for (uint32_t k = 1 + blockIdx.x * blockDim.x + threadIdx.x; k < L; k += gridDim.x * blockDim.x) {
    const int32_t a = abs(C[k]);
    pm = max(pm, a);
    en += (unsigned long long)((long long)C[k] * C[k]);
    atomicAdd(&hist[a], 1ull);
  }
  for (int o = 16; o; o >>= 1) {
    pm = max(pm, __shfl_xor_sync(0xffffffffu, pm, o));
    en += __shfl_xor_sync(0xffffffffu, en, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(psl, pm);
    atomicAdd(energy, en);
  }
}
}  // namespace
int launch_verify(const int32_t* C, uint32_t L, int32_t* psl, unsigned long long* energy,
                  unsigned long long* hist, cudaStream_t s) {
  verify_kernel<<<std::min<uint32_t>((L + 255) / 256, 1184), 256, 0, s>>>(C, L, psl, energy, hist);
  return launch_status(1);
}
}  // namespace pslb
