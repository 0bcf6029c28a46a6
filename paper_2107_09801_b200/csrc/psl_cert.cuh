// psl_cert.cuh -- the certified (decision-exact) neighbourhood scan.
// Included by psl_kernels.cu inside its anonymous namespace (after the exact
// sweep helpers).
//
// The reference scores neighbour j by the serial double chain
//   V(j) = fl( sum_{k=1}^{L-1} E_k(2 + s_j (s_{j-k} + s_{j+k})) )       (sequence.hpp:126-162)
// with E_k(x) = pow_int(|C_k - 2(x-2)|, alpha) and out-of-range s = 0.  The
// serial chain only matters through the DECISIONS run_search takes from it
// (argmin with smallest-offset ties, value_step vs value_local; search.cpp:
// 383-413), so this scan computes an approximation of the exact real sum T(j)
// with a rigorous error bound, turns it into an interval that provably holds
// V(j) (|V - T| <= gamma_{L} T for a serial sum of L-1 nonnegative terms), and
// hands the step to the exact sweep whenever the intervals cannot decide.
//
// Per shift k the term is affine in u = s_j s_{j+k}, v = s_j s_{j-k} and uv:
//   both sides in range: 4E = 4P + 4Q (u + v) + 4R uv,  4P = e4+e0+2e2,
//                        4Q = e4-e0, 4R = e4+e0-2e2        (e_x = E_k(x))
//   one side in range:   4E = 4M + 4N (u or v),          4M = 2(e3+e1), 4N = 2(e3-e1)
//   none:                4E = 4 e2
// so with zones over the row window (m_j = min(j, L-1-j), M_j = L-1-m_j):
//   4T(j) = S_P + S_M + S_E                       (window-wide constants, k in Z1/Z3/Z5)
//         + s_j sum_k H4_k (s_{j+k} + s_{j-k})    (H4 = 4Q in Z1, 4N past m_hi: a correlation)
//         + sum_{k in Z1} 4R_k s_{j+k} s_{j-k}    (the both-sides cross term)
//         + band-1 exact terms + band-2 constants (the <= n-wide bands)
//
// Tensor cores.  The correlation runs on tcgen05 (kind::i8, accumulators in
// TMEM): rows j = JT + u, u = rho + 128 sigma (rho = TMEM lane, sigma = one of 8
// row blocks, an N-group), so one M128 x N64 x K32 MMA scores 1024 rows:
//   forward  D_f[rho][(7-sigma, d)] += s_{JT+rho+kappa} * digit_d(H4(kappa - 128 sigma))
//   reversed D_r[r][(sigma, d)]     += s_{JT+127-r-kappa'} * digit_d(H4(kappa' + 128 sigma))
// A = "Hankel cores" of the staged sequence (core m: 8 rows x 16 bytes of
// s[base + 8m + i ..]; the descriptor's row-group / k-half strides overlap them,
// so no per-row copies), B = a ring of digit cores (8 digits x 16 shifts) that
// the N-group stride (1 KB = 128 shifts) walks through.  The cross term is not
// separable (s_{j+k} s_{j-k}) and stays on mma.sync (zone 1 only).
#pragma once

// The certified kernel's CTA (one walk per SM) is 16 warps: every thread
// builds one shift per chunk (kCC = 512); warps 15 and 14 also issue the
// chunk's forward / reversed tcgen05 MMAs; all 16 warps run the cross MMAs.
constexpr uint32_t kCertThreads = 2 * kThreads;
#ifndef PSL_STAGE_PRE
#define PSL_STAGE_PRE 1            // zone-1 window staging: pivot words loaded at the top of the build
#endif
#ifndef PSL_REV_WARP_C
#define PSL_REV_WARP_C 14u         // the warp that issues the reversed MMAs (PSL_REV_WARP)
#endif
constexpr uint32_t kCC = kCertThreads;        // shifts per certified chunk (one per builder thread)
constexpr int kCCols = kCC / 32;              // 32-shift columns per chunk
constexpr int kCertTiles = 4;                 // mma.sync m16 row tiles per warp (64 rows, 16 warps)
constexpr uint32_t kLag = 2;                  // reversed MMAs trail the builder by 2 chunks (>= 896 shifts)
static_assert(kLag * kCC >= 896 && kCC % 32 == 0, "chunk geometry");
constexpr uint32_t kRing = 256;               // digit-core ring (x2 mapped), cores of 16 shifts
constexpr uint32_t kACores = (128 + kCC) / 8 + 2;   // sequence cores per direction per chunk
constexpr int kLimbStride = kCC + 16;         // bytes per R digit row (bank spread)
constexpr int kWinBytes = 1568;               // staged bytes per copy (392 words, = 8 mod 32)
constexpr int kY0 = 1031;                     // origin of the reversed window
constexpr size_t kLimbBuf = 8ull * kLimbStride;
constexpr size_t kWinBuf = 4ull * kWinBytes;
constexpr size_t kCertRecBuf = (size_t)kCC * sizeof(int32_t);
#ifndef PSL_BULK_C
#define PSL_BULK_C 1               // C chunks by one bulk async copy (TMA engine); 0: per-thread cp.async
#endif
constexpr uint32_t kCSlot = kCC + 4;          // C ring slot: the 16-byte aligned span C[kb-1, kb+515)
constexpr size_t kCertCBuf = (size_t)kCSlot * sizeof(int32_t);
constexpr size_t kDRing = 2ull * kRing * 128;            // digit cores, double mapped
constexpr size_t kABuf = 2ull * kACores * 128;           // fwd + rev cores, one buffer
// [digit ring][A cores 2][R digit rows 2][win_f 2][win_r 2][rec 2][C ring 3]
constexpr size_t kCertBytes = kDRing + 2 * kABuf + 2 * kLimbBuf + 4 * kWinBuf +
                              2 * kCertRecBuf + 3 * kCertCBuf;
constexpr long long kMaxD = 0x7F7F7F7F7F7F7F7Fll;      // 8 balanced base-256 digits
constexpr uint32_t kCertMinL = 2048;
#ifndef PSL_XTMEM
#define PSL_XTMEM 0                // 1: cross term on 8 row tiles x half the columns per warp, accumulators
                                   // parked in TMEM between zone-1 chunks (half the LDS per MMA).  Correct, but
                                   // measured 21.6 vs 16.4 ms/step at m20 (its -DPSL_PHASE_TIMING build: -2 %);
                                   // 0: 4 tiles x all columns, accumulators in registers
#endif
constexpr uint32_t kTmemCols = PSL_XTMEM ? 256 : 128;   // fwd 0-63, rev 64-127, cross 128-255
constexpr uint32_t kLutS = 6144;             // PowerTable entries staged in shared memory           // fwd accumulator cols 0-63, rev 64-127

struct CertIO {
  uint32_t L, n, nchunks;
  int32_t j0;                                 // rows j = j0 + rho (may be < 0 for inactive rows)
  uint32_t r_lo, r_hi;                        // active rows of this pass: r_lo <= rho < r_hi
  int32_t JT;                                 // j0 + r_lo: tensor-core row u = rho - r_lo
  const int32_t* Csrc;
  int32_t* Cdst;
  int32_t* Cloc;
  const uint32_t* flips;
  uint32_t F;
  uint32_t f1;                                // flips[0] and s_{f1} (after) when F == 1
  int sf1;
  uint32_t alpha;
  const double* lut;                          // PowerTable of the phase (covers |C_k| + 4): its
                                              // head staged in shared memory when it fits (generic loads)
  int2* hlist;
  uint32_t* hcount;
  int32_t hthr;
  double scaleH, scaleR;                      // 2^-qH, 2^-qR
  uint32_t m_lo, m_hi, M_lo, M_hi;            // zone bounds (see above)
  double* b2M;                                // [1024] global scratch: band-2 4M_k, 4 e2_k
  double* b2E;
  bool chain;                                 // also the serial fitness() of the folded table
  bool fsum;                                  // the initial fitness() as a certified interval:
                                              // builders add lut[|C_k|] into part[3]
  size_t c_stride;                            // C entries per walk (a multiple of 32)
  uint64_t* cbar;                             // [3] mbarriers of the C ring's bulk copies
};

struct CertSmem {
  unsigned char* dring;   // [2 kRing][8 x 16] H4 digit cores, core q at q % kRing and + kRing
  unsigned char* acore;   // [2][fwd kACores | rev kACores][128] sequence cores
  unsigned char* limbR;   // [2][8][kLimbStride] R4 digit rows (zone-1 chunks, mma.sync)
  unsigned char* winF;    // [2][4][kWinBytes]  F[x] = s_{j0+kb+x}
  unsigned char* winV;    // [2][4][kWinBytes]  V[y] = s_{j0-kb+kY0-y}
  int32_t* rec;           // [2][kCC]           C_k (band-1 chunks only)
  int32_t* cring;         // [3][kCC]           C_k of chunks c+1, c+2 in flight (cp.async)
  double* linrow;         // [1024] (aliases the windows after the pass)
  double* xrow;           // [1024] (aliases the sequence cores after the pass)
};

__device__ __forceinline__ CertSmem cert_carve(unsigned char* base) {
  CertSmem m;
  m.dring = base;
  m.acore = base + kDRing;
  m.limbR = m.acore + 2 * kABuf;
  m.winF = m.limbR + 2 * kLimbBuf;
  m.winV = m.winF + 2 * kWinBuf;
  m.rec = reinterpret_cast<int32_t*>(m.winV + 2 * kWinBuf);
  m.cring = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(m.rec) + 2 * kCertRecBuf);
  m.linrow = reinterpret_cast<double*>(m.winF);
  m.xrow = reinterpret_cast<double*>(m.acore);
  return m;
}
static_assert(2 * kWinBuf >= kGroup * sizeof(double) && 2 * kABuf >= kGroup * sizeof(double),
              "row arrays alias the windows / cores");

__device__ __forceinline__ uint32_t cert_kb(int32_t c) { return (uint32_t)(1 + c * (int32_t)kCC); }

// shifts with nonzero H4 (zone 1, past band 1 up to M_hi) intersect [lo, hi]?
__device__ __forceinline__ bool cert_lin_in(const CertIO& io, long long lo, long long hi) {
  if (hi < 1 || lo > (long long)io.L - 1) return false;
  return lo <= (long long)io.m_lo || (hi > (long long)io.m_hi && lo <= (long long)io.M_hi);
}

// +-1 / 0 bytes of staged sequence data
__device__ __forceinline__ uint32_t nib_bytes(uint32_t nib) {
  return ((nib * 0x00204081u) & 0x01010101u) * 0xFEu + 0x01010101u;
}
__device__ __forceinline__ uint32_t sbyte(const uint32_t* sb, long long p, uint32_t L) {
  if (p < 0 || p >= (long long)L) return 0u;
  return ((sb[(p >> 5) + 1] >> (p & 31)) & 1u) ? 0xFFu : 0x01u;
}
// 16 bytes for positions p0 + dir * x, x = 0..15 (dir = +1 / -1), as 4 words
__device__ __forceinline__ uint4 seq16(const uint32_t* sb, long long p0, int dir, uint32_t L) {
  const long long lo = dir > 0 ? p0 : p0 - 15, hi = lo + 15;
  uint4 r = make_uint4(0u, 0u, 0u, 0u);
  if (hi < 0 || lo >= (long long)L) return r;
  if (lo >= 0 && hi < (long long)L) {
    uint32_t x = __funnelshift_r(sb[(lo >> 5) + 1], sb[(lo >> 5) + 2], (uint32_t)(lo & 31)) & 0xFFFFu;
    if (dir < 0) x = __brev(x) >> 16;
    r.x = nib_bytes(x & 0xF); r.y = nib_bytes((x >> 4) & 0xF);
    r.z = nib_bytes((x >> 8) & 0xF); r.w = nib_bytes(x >> 12);
    return r;
  }
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  for (int i = 0; i < 16; ++i) w[i >> 2] |= sbyte(sb, p0 + dir * i, L) << (8 * (i & 3));
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(mbar)), "r"(parity) : "memory");
  }
}

// C_k of chunk c -> ring slot c % 3, asynchronously.  PSL_BULK_C: thread 0
// issues ONE bulk copy (cp.async.bulk, the TMA engine) of the 16-byte aligned
// span C[kb-1, kb+515) (clamped to the walk's c_stride entries; shifts >= L are
// never used) that completes on the slot's mbarrier; otherwise every thread
// copies its own 4 bytes with cp.async (zero-filled past L).
__device__ __forceinline__ void cert_prefetch(const CertIO& io, const CertSmem& cs, uint32_t c) {
#if PSL_BULK_C
  if (threadIdx.x != 0) return;
  const uint32_t slot = c % 3;
  const size_t base = (size_t)cert_kb((int32_t)c) - 1;                 // = kCC * c, 16-byte aligned
  const uint32_t n = (uint32_t)min((size_t)kCSlot, io.c_stride - base);
  const uint32_t bytes = n * 4u;                                         // a multiple of 128
  int32_t* dst = cs.cring + (size_t)slot * kCSlot;
  PSL_CHK(in_buf(dst, cs.cring, 3 * kCertCBuf, bytes) && n > 0 && (base & 3) == 0, 1);
  const uint32_t bar = smem_u32(io.cbar + slot);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(io.Csrc + base), "r"(bytes), "r"(bar) : "memory");
#else
  const uint32_t k = cert_kb(c) + threadIdx.x;
  int32_t* dst = cs.cring + (size_t)(c % 3) * kCSlot + 1 + threadIdx.x;
  const bool in = k < io.L;
  PSL_CHK(in_buf(dst, cs.cring, 3 * kCertCBuf, 4), 1);
  const int32_t* src = io.Csrc + (in ? k : 0);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(in ? 4 : 0) : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
#endif
}
// This thread's C_k of chunk c (after the slot's copy landed).  cphase: bit s =
// the parity of slot s's next completion (kept by every thread across passes).
__device__ __forceinline__ int32_t cert_take(const CertIO& io, const CertSmem& cs, uint32_t c,
                                             int pending, uint32_t& cphase) {
  const uint32_t slot = c % 3;
#if PSL_BULK_C
  (void)pending;
  mbar_wait(io.cbar + slot, (cphase >> slot) & 1u);
  cphase ^= 1u << slot;
#else
  (void)io; (void)cphase;
  if (pending >= 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
  else if (pending == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
  else asm volatile("cp.async.wait_group 0;" ::: "memory");
#endif
  return cs.cring[(size_t)slot * kCSlot + 1 + threadIdx.x];
}

__device__ __forceinline__ unsigned char* dcore(const CertSmem& cs, long long q) {
  return cs.dring + (size_t)(((q % kRing) + kRing) % kRing) * 128;
}

// Builder for chunk c: fold pending flips into C, write C back, collect high
// sidelobes, window constants, band records, the H4 digit cores (ring) and,
// in zone-1 chunks, the R4 digit rows + sequence windows of the cross MMAs.
// One shift per thread.
// The single move's fold words of chunk c (s_{f-k}, s_{f+k} for this thread's
// k), loaded one iteration ahead so the global latency overlaps a chunk.
// Positions past either end index the zero pads (the fold masks them out).
__device__ __forceinline__ uint2 cert_fold_words(const CertIO& io, uint32_t c, const uint32_t* sb) {
  const int32_t k = (int32_t)cert_kb(c) + (int32_t)threadIdx.x;
  const int32_t f = (int32_t)io.f1;
  PSL_CHK(sb_ok(((f - k) >> 5) + 1, io.L) && sb_ok(((f + k) >> 5) + 1, io.L), 2);
  return make_uint2(sb[((f - k) >> 5) + 1], sb[((f + k) >> 5) + 1]);
}

__device__ __forceinline__ void cert_build(const CertIO& io, const CertSmem& cs, uint32_t c,
                                           const uint32_t* sb, int32_t& pmax, double (&part)[5],
                                           int32_t cpre, uint2 fw, bool& ovf) {
  const uint32_t t = threadIdx.x;
  const uint32_t kb = cert_kb(c), k = kb + t;
  const uint32_t b = c & 1;
  const int L = (int)io.L, j0 = io.j0;
  constexpr int kW = kWinBytes / 4;
  // window-staging word q of direction dir: bytes 4q..4q+7 (fwd: positions p0 + i, rev: p0 - i)
  auto stage_p0 = [&](int idx, int& dir) {
    dir = idx >= kW ? 1 : 0;
    const int q = dir ? idx - kW : idx;
    return dir == 0 ? j0 + (int)kb + 4 * q : j0 - (int)kb + kY0 - 4 * q;
  };
#if PSL_STAGE_PRE
  // zone-1 chunks: the staging's pivot words, loaded before the build (L2 latency off the barrier path)
  uint2 pw0 = make_uint2(0u, 0u), pw1 = make_uint2(0u, 0u);
  if (kb <= io.m_lo) {
    auto pre = [&](int idx) {
      int dir;
      const int p0 = stage_p0(idx, dir);
      const int lo = dir == 0 ? p0 : p0 - 7;
      return (lo >= 0 && lo + 7 < L) ? make_uint2(sb[(lo >> 5) + 1], sb[(lo >> 5) + 2]) : make_uint2(0u, 0u);
    };
    pw0 = pre((int)t);
    if ((int)(t + kCC) < 2 * kW) pw1 = pre((int)(t + kCC));
  }
#endif
  bool want = false;
  int32_t cv = 0;
  if (k < io.L) {
    cv = cpre;
    PSL_CHK(k >= 1, 3);
    if (io.Cloc) io.Cloc[k] = cpre;   // lazy local snapshot: the pre-fold table
#ifndef PSL_ABLATE_FOLD
    if (io.F == 1) {
      // the common single move: C_k += 2 s_f (s_{f-k} + s_{f+k}), s_f after the flip
      const uint32_t f = io.f1;
      const int bA = (int)((fw.x >> ((f - k) & 31)) & 1u), bB = (int)((fw.y >> ((f + k) & 31)) & 1u);
      const int acc = (k <= f ? 1 - 2 * bA : 0) + (f + k < io.L ? 1 - 2 * bB : 0);
      cv += 2 * io.sf1 * acc;
    } else if (io.F) {
      SweepIO fio;
      fio.L = io.L; fio.flips = io.flips; fio.F = io.F;
      cv = fold_flips(cv, k, fio, sb);
    }
#endif
    if (io.fsum) part[3] = __dadd_rn(part[3], io.lut[abs(cv)]);
    if (io.Cdst) io.Cdst[k] = cv;
    const int32_t a = abs(cv);
    pmax = max(pmax, a);
    want = io.hlist != nullptr && a >= io.hthr;
  }
  if (io.hlist) {
    const uint32_t m = __ballot_sync(FULL, want);
    if (m) {
      const int lane = t & 31, leader = __ffs(m) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(io.hcount, (uint32_t)__popc(m));
      base = __shfl_sync(FULL, base, leader);
      PSL_CHK(!want || base + __popc(m & ((1u << lane) - 1)) < io.L, 4);
      if (want) io.hlist[base + __popc(m & ((1u << lane) - 1))] = make_int2((int)k, cv);
    }
  }
  // per zone only the terms it needs (PowerTable lookups, e_x = E_k(x))
  double H = 0.0, R = 0.0;
  if (k < io.L) {
    if (k <= io.m_lo) {                               // Z1: both sides for every row
      const double e4 = io.lut[abs(cv - 4)], e0 = io.lut[abs(cv + 4)];
      const double e2 = io.lut[abs(cv)];
      H = __dsub_rn(e4, e0);
      R = __dsub_rn(__dadd_rn(e4, e0), __dmul_rn(2.0, e2));
      part[0] = __dadd_rn(part[0], __dadd_rn(__dadd_rn(e4, e0), __dmul_rn(2.0, e2)));
    } else if (k <= io.m_hi) {                        // band 1: exact terms per row
    } else if (k <= io.M_hi) {                        // Z3 / band 2: one side or none
      const double e3 = io.lut[abs(cv - 2)], e1 = io.lut[abs(cv + 2)];
      H = __dmul_rn(2.0, __dsub_rn(e3, e1));
      const double m4 = __dmul_rn(2.0, __dadd_rn(e3, e1));
      if (k <= io.M_lo) {
        part[1] = __dadd_rn(part[1], m4);
      } else {                                        // band 2: per-row prefix sums
        PSL_CHK(k - io.M_lo - 1 < (uint32_t)kGroup, 5);
        io.b2M[k - io.M_lo - 1] = m4;
        io.b2E[k - io.M_lo - 1] = __dmul_rn(4.0, io.lut[abs(cv)]);
      }
    } else {                                          // Z5: no side for any row
      part[2] = __dadd_rn(part[2], __dmul_rn(4.0, io.lut[abs(cv)]));
    }
  }
  // fixed point -> 8 balanced base-256 digits
  const double hs = __dmul_rn(H, io.scaleH);
  // |v| < 2^61 (the units leave a 4x margin under 2^62 < kMaxD), tested on the
  // double (doubles near 2^61 are 512 apart, so the rounded value is below it too;
  // NaN fails the test)
  ovf |= !(fabs(hs) < 0x1p61);
  const long long hv = __double2ll_rn(hs);
  const unsigned long long dh = ((unsigned long long)hv + 0x8080808080808080ull) ^ 0x8080808080808080ull;
  // H4 digit core: core q = 16 c + t / 16 holds rows d (16 shifts each).  Lane
  // x of a 4-lane group assembles row (x & 3) / row 4 + (x & 3) of the group's
  // 4 shifts from the group's digit words (shuffles + byte permutes): two word
  // stores per mapping instead of eight byte stores.
#ifndef PSL_ABLATE_DIGITS
  {
    const uint32_t lane = t & 31, x = lane & 3, gbase = lane & ~3u;
    const uint32_t lo = (uint32_t)dh, hi = (uint32_t)(dh >> 32);
    uint32_t L4[4], H4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      L4[i] = __shfl_sync(FULL, lo, gbase + i);
      H4[i] = __shfl_sync(FULL, hi, gbase + i);
    }
    // byte x of each of the 4 words -> one word (shift i's byte at position i)
    const uint32_t sel = x | ((4 + x) << 4);
    const uint32_t wl = __byte_perm(__byte_perm(L4[0], L4[1], sel), __byte_perm(L4[2], L4[3], sel), 0x5410);
    const uint32_t wh = __byte_perm(__byte_perm(H4[0], H4[1], sel), __byte_perm(H4[2], H4[3], sel), 0x5410);
    const uint32_t col = (t & 15) & ~3u;                 // first of the group's 4 shifts in the core
    unsigned char* p0 = dcore(cs, (long long)(kCC / 16) * c + (t >> 4)) + col;
    unsigned char* p1 = p0 + kRing * 128;
    PSL_CHK(in_buf(p0 + 16 * x, cs.dring, kDRing, 4) && in_buf(p1 + 16 * (4 + x), cs.dring, kDRing, 4), 6);
    *reinterpret_cast<uint32_t*>(p0 + 16 * x) = wl;
    *reinterpret_cast<uint32_t*>(p0 + 16 * (4 + x)) = wh;
    *reinterpret_cast<uint32_t*>(p1 + 16 * x) = wl;
    *reinterpret_cast<uint32_t*>(p1 + 16 * (4 + x)) = wh;
  }
#endif
  PSL_CHK(b * kCC + t < 2 * kCC, 7);
  if (io.chain) cs.rec[b * kCC + t] = cv;
  if (kb > io.m_lo) return;
  // zone-1 chunk: R4 digit rows and the sequence windows of the cross MMAs
  {
    const double rs = __dmul_rn(R, io.scaleR);
    ovf |= !(fabs(rs) < 0x1p61);
    const long long rv = __double2ll_rn(rs);
    const unsigned long long dr = ((unsigned long long)rv + 0x8080808080808080ull) ^ 0x8080808080808080ull;
    unsigned char* lr = cs.limbR + (size_t)b * kLimbBuf + t;
    PSL_CHK(in_buf(lr + 7 * kLimbStride, cs.limbR, 2 * kLimbBuf), 8);
#pragma unroll
    for (int d = 0; d < 8; ++d) lr[d * kLimbStride] = (unsigned char)(dr >> (8 * d));
  }
#ifdef PSL_ABLATE_STAGE
  return;
#endif
  // thread -> base word q of one direction: bytes 4q..4q+7 of the base copy
  // from one bit window, copy a word q = base bytes 4q+a..4q+a+3
  auto stage = [&](int idx, uint2 pw) {
    int dir;
    const int p0 = stage_p0(idx, dir);
    const int q = dir ? idx - kW : idx;
    // fwd: byte i <-> position p0 + i; rev: byte i <-> position p0 - i (i = 0..7)
    const int lo = dir == 0 ? p0 : p0 - 7, hi = lo + 7;
    uint32_t w0 = 0, w1 = 0;
    if (hi >= 0 && lo < L) {
      if (lo >= 0 && hi < L) {
        PSL_CHK(sb_ok((lo >> 5) + 2, io.L), 9);
#if PSL_STAGE_PRE
        uint32_t x = __funnelshift_r(pw.x, pw.y, (uint32_t)lo & 31) & 0xFFu;
#else
        (void)pw;
        uint32_t x = __funnelshift_r(sb[(lo >> 5) + 1], sb[(lo >> 5) + 2], (uint32_t)lo & 31) & 0xFFu;
#endif
        if (dir) x = __brev(x) >> 24;
        w0 = nib_bytes(x & 0xFu);
        w1 = nib_bytes(x >> 4);
      } else {
        for (int i = 0; i < 4; ++i) {
          w0 |= sbyte(sb, dir == 0 ? p0 + i : p0 - i, io.L) << (8 * i);
          w1 |= sbyte(sb, dir == 0 ? p0 + 4 + i : p0 - 4 - i, io.L) << (8 * i);
        }
      }
    }
    unsigned char* dst = (dir == 0 ? cs.winF : cs.winV) + (size_t)b * kWinBuf + 4 * q;
    PSL_CHK(in_buf(dst + 3 * kWinBytes, dir == 0 ? cs.winF : cs.winV, 2 * kWinBuf, 4), 10);
    *reinterpret_cast<uint32_t*>(dst) = w0;
    *reinterpret_cast<uint32_t*>(dst + kWinBytes) = __funnelshift_r(w0, w1, 8);
    *reinterpret_cast<uint32_t*>(dst + 2 * kWinBytes) = __funnelshift_r(w0, w1, 16);
    *reinterpret_cast<uint32_t*>(dst + 3 * kWinBytes) = __funnelshift_r(w0, w1, 24);
  };
  // 2 kW = 784 words per chunk: one per thread, the other 272 to the warps that
  // stage no sequence cores and issue no reversed MMAs before the barrier
  // (11, 12, 13, 15), so the chunk barrier waits for no doubly loaded warp
#if !PSL_STAGE_PRE
  const uint2 pw0 = make_uint2(0u, 0u), pw1 = pw0;
#endif
  stage((int)t, pw0);
  if ((int)(t + kCC) < 2 * kW) stage((int)(t + kCC), pw1);
}

// Tail chunks c0 <= c < nch (every shift past M_hi: H4 = R4 = 0, the term of
// every row is e2 = |C_k|^alpha).  No staging and no per-chunk barrier: each
// thread streams its shift of four chunks at a time from C (loads first), folds
// the move, writes C back (and the lazy local snapshot's pre-fold value),
// collects PSL / high sidelobes and adds 4 e2 to the window constant part[2] --
// the same per-thread serial order and term count as cert_build, so the
// rounding budget of the window sums is unchanged.
__device__ __forceinline__ void cert_tail(const CertIO& io, uint32_t c0, uint32_t nch,
                                          const uint32_t* sb, int32_t& pmax, double (&part)[5]) {
#ifndef PSL_TAIL_U
#define PSL_TAIL_U 8                // (4: +1.0 % at m20, 16: spills)
#endif
  constexpr uint32_t U = PSL_TAIL_U;   // chunks per streamed group (loads first)
  const uint32_t t = threadIdx.x;
#pragma unroll 1
  for (uint32_t c = c0; c < nch; c += U) {
    int32_t cp[U];
    uint2 fw[U];
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      const uint32_t k = cert_kb((int32_t)(c + u)) + t;
      const bool in = c + u < nch && k < io.L;
      PSL_CHK(!in || k >= 1, 11);
      cp[u] = in ? __ldcg(io.Csrc + k) : 0;
      fw[u] = (in && io.F == 1) ? cert_fold_words(io, c + u, sb) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (uint32_t u = 0; u < U; ++u) {
      if (c + u >= nch) break;                         // warp-uniform
      const uint32_t k = cert_kb((int32_t)(c + u)) + t;
      bool want = false;
      int32_t cv = 0;
      if (k < io.L) {
        cv = cp[u];
        if (io.Cloc) io.Cloc[k] = cv;                  // lazy local snapshot: pre-fold
        if (io.F == 1) {
          const uint32_t f = io.f1;
          const int bA = (int)((fw[u].x >> ((f - k) & 31)) & 1u), bB = (int)((fw[u].y >> ((f + k) & 31)) & 1u);
          const int acc = (k <= f ? 1 - 2 * bA : 0) + (f + k < io.L ? 1 - 2 * bB : 0);
          cv += 2 * io.sf1 * acc;
        } else if (io.F) {
          SweepIO fio;
          fio.L = io.L; fio.flips = io.flips; fio.F = io.F;
          cv = fold_flips(cv, k, fio, sb);
        }
        const int32_t a = abs(cv);
        if (io.fsum) part[3] = __dadd_rn(part[3], io.lut[a]);
        if (io.Cdst) io.Cdst[k] = cv;
        pmax = max(pmax, a);
        want = io.hlist != nullptr && a >= io.hthr;
        part[2] = __dadd_rn(part[2], __dmul_rn(4.0, io.lut[a]));
      }
      if (io.hlist) {
        const uint32_t m = __ballot_sync(FULL, want);
        if (m) {
          const int lane = t & 31, leader = __ffs(m) - 1;
          uint32_t base = 0;
          if (lane == leader) base = atomicAdd(io.hcount, (uint32_t)__popc(m));
          base = __shfl_sync(FULL, base, leader);
          PSL_CHK(!want || base + __popc(m & ((1u << lane) - 1)) < io.L, 12);
          if (want) io.hlist[base + __popc(m & ((1u << lane) - 1))] = make_int2((int)k, cv);
        }
      }
    }
  }
}

// Zero digit cores for chunk c (ring slots of chunks past the end / before the start)
__device__ __forceinline__ void cert_zero_digits(const CertSmem& cs, long long c) {
  constexpr uint32_t kCores = kCC / 16, kParts = kCores * 8;   // 16-byte parts per mapping
  for (uint32_t i = threadIdx.x; i < 2 * kParts; i += blockDim.x) {
    const uint32_t part = i % kParts, map = i / kParts;
    unsigned char* p = dcore(cs, (long long)kCores * c + part / 8) + 16 * (part & 7) + map * kRing * 128;
    PSL_CHK(in_buf(p, cs.dring, kDRing, 16), 13);
    *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
  }
}

// 20 sequence bytes for positions p0 + dir * x, x = 0..19, as 5 words (0 outside [0, L))
__device__ __forceinline__ void seq20(const uint32_t* sb, int32_t p0, int dir, int32_t L, uint32_t (&w)[5]) {
  const int32_t lo = dir > 0 ? p0 : p0 - 19, hi = lo + 19;
  if (lo >= 0 && hi < L) {
    PSL_CHK(sb_ok((lo >> 5) + 2, (uint32_t)L), 14);
    uint32_t x = __funnelshift_r(sb[(lo >> 5) + 1], sb[(lo >> 5) + 2], (uint32_t)lo & 31) & 0xFFFFFu;
    if (dir < 0) x = __brev(x) >> 12;
#pragma unroll
    for (int q = 0; q < 5; ++q) w[q] = nib_bytes((x >> (4 * q)) & 0xFu);
  } else {
#pragma unroll
    for (int q = 0; q < 5; ++q) w[q] = 0u;
    if (hi >= 0 && lo < L)
      for (int i = 0; i < 20; ++i) w[i >> 2] |= sbyte(sb, p0 + dir * i, (uint32_t)L) << (8 * (i & 3));
  }
}

// Sequence cores of iteration c (buffer c & 1): forward kappa-chunk c
// (core m row i = s[JT + kb + 8m + i + x]) and reversed kappa'-chunk c - kLag
// (core m row i = s[JT + 127 - kb' - 8m - i - x]).  Core row (m, i) is the 16
// bytes at position offset r = 8m + i (address 16 r); a thread expands 20 bytes
// once and emits the four rows r0..r0+3 by byte shifts.
__device__ __forceinline__ void cert_cores(const CertIO& io, const CertSmem& cs, int32_t c,
                                           const uint32_t* sb, bool fwd, bool rev) {
  unsigned char* base = cs.acore + (size_t)(c & 1) * kABuf;
  constexpr uint32_t kQuads = kACores * 2;    // 100 groups of 4 rows per direction
  const uint32_t t = threadIdx.x;
  // forward quads on threads 0..163, reversed on 192..355: no warp runs both
  // directions' code (a mixed warp took twice as long and held up the barrier)
  constexpr uint32_t kRevT = (kQuads + 31) / 32 * 32;
  uint32_t dir, g;
  if (t < kQuads) { dir = 0; g = t; }
  else if (t >= kRevT && t < kRevT + kQuads) { dir = 1; g = t - kRevT; }
  else return;
  if (dir == 0 ? !fwd : !rev) return;
#ifdef PSL_ABLATE_CORES
  return;
#endif
  const int32_t p0 = dir == 0 ? io.JT + (int32_t)cert_kb(c) + 4 * (int32_t)g
                              : io.JT + 127 - (int32_t)cert_kb(c - (int32_t)kLag) - 4 * (int32_t)g;
  uint32_t w[5];
  seq20(sb, p0, dir == 0 ? 1 : -1, (int32_t)io.L, w);
  uint4* dst = reinterpret_cast<uint4*>(base + (size_t)dir * kACores * 128 + 64 * g);
  PSL_CHK(in_buf(dst + 3, cs.acore, 2 * kABuf, 16), 15);
  // row r of the quad = the 16 bytes from byte r; rows in a lane-rotated order
  // (r = i + g/2 mod 4) so each quarter-warp store covers 8 distinct 16-byte bank groups
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t r = (uint32_t)(i + (g >> 1)) & 3u, sh = 8u * r;
    dst[r] = make_uint4(__funnelshift_r(w[0], w[1], sh), __funnelshift_r(w[1], w[2], sh),
                        __funnelshift_r(w[2], w[3], sh), __funnelshift_r(w[3], w[4], sh));
  }
}

// ---- tcgen05 plumbing
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100), SWIZZLE_NONE, base offset 0
  return d;
}
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(mbar)) : "memory");
}

// One tcgen05 MMA issued by a whole warp: warp-uniform descriptors, one lane
// elected inside the asm (no per-MMA waterfall over a divergent thread).
__device__ __forceinline__ void umma_i8_elect(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}

// One direction's MMAs of iteration c (dir 0: forward kappa-chunk c, 1:
// reversed kappa'-chunk c - kLag), K-steps s0 <= s < s1, issued by a whole warp;
// with `commit` the warp then commits them (and its earlier ones) to the
// iteration's barrier.  The commit also arrives when the warp issued nothing (two
// issuing warps, one barrier arrival each per iteration).  The 16 K-steps are
// issued in two halves around other work: the issuing thread blocks while the
// tensor pipe's queue (2-3 MMAs) is full, so each half mostly finds it drained.
__device__ __forceinline__ void cert_issue_dir(const CertSmem& cs, uint32_t tmem, int32_t c, int dir,
                                               bool active, uint32_t started, uint64_t* mbar,
                                               int s0, int s1, bool commit) {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (active) {
    const uint32_t abuf = smem_u32(cs.acore) + (uint32_t)(c & 1) * (uint32_t)kABuf +
                          (dir ? (uint32_t)(kACores * 128) : 0u);
    const uint32_t ring = smem_u32(cs.dring);
    const long long q0 = dir ? (long long)(kCC / 16) * (c - (int32_t)kLag) : (long long)(kCC / 16) * c - 56;
    uint64_t da = umma_desc(abuf, 256, 128) + (uint64_t)(s0 * (512 >> 4));
    uint64_t db = umma_desc(ring + (uint32_t)((((q0 % kRing) + kRing) % kRing) * 128), 128, 1024) +
                  (uint64_t)(s0 * (256 >> 4));
    const uint32_t bit = dir ? 2u : 1u;
#pragma unroll 4
    for (int s = s0; s < s1; ++s) {
      umma_i8_elect(tmem + (dir ? 64u : 0u), da, db, (s > 0 || (started & bit)) ? 1u : 0u);
      da += 512 >> 4;
      db += 256 >> 4;
    }
  }
  if (commit)
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(mbar)) : "memory");
}

// ---- the cross term on mma.sync (zone-1 chunks)
__device__ __forceinline__ void imma_s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                        uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// s_{j+k} s_{j-k} as +-1 bytes from two +-1 byte words
__device__ __forceinline__ uint32_t uv_bytes(uint32_t f, uint32_t v) { return (f ^ v) | 0x01010101u; }

template <int OFF>
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
  return v;
}

// Per-lane shared addresses (buffer 0) of this warp's cross-MMA operands.  Row
// rho = 64 w + 16 r + g (+8 for a1/a3), fragment layout of mma.m16n8k32:
//   forward word m (bytes 8m..8m+3 past base_f = 64w + g + 4t) = s_{j+k} for
//     m = 2r + 4c + {0: a0, 1: a1, 2: a2, 3: a3}
//   reversed word m' (past base_v = kY0 - 64w - g + 4t) = s_{j-k} for
//     m' = 4c - 2r + {0: a0, -1: a1, 2: a2, 1: a3}
struct CertLane {
  uint32_t f, v, bd;
};
__device__ __forceinline__ CertLane cert_lane(const CertSmem& cs) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t gid = lane >> 2, tig = lane & 3;
  const uint32_t base_f = 64 * w + gid + 4 * tig, af = gid & 3;
  const uint32_t base_v = kY0 - 64 * w - gid + 4 * tig, av = base_v & 3;
  CertLane l;
  l.f = smem_u32(cs.winF) + af * kWinBytes + (base_f - af);
  l.v = smem_u32(cs.winV) + av * kWinBytes + (base_v - av);
  l.bd = smem_u32(cs.limbR) + gid * kLimbStride + 4 * tig;
  return l;
}

struct Quad {
  uint32_t x, y, z, w;
};
template <int E>
__device__ __forceinline__ Quad qfe(uint32_t f) {
  return {lds32<32 * E>(f), lds32<32 * E + 8>(f), lds32<32 * E + 16>(f), lds32<32 * E + 24>(f)};
}
template <int E>
__device__ __forceinline__ Quad qfo(uint32_t f) {
  return {lds32<32 * E + 16>(f), lds32<32 * E + 24>(f), lds32<32 * E + 32>(f), lds32<32 * E + 40>(f)};
}
template <int E>
__device__ __forceinline__ Quad qve(uint32_t v) {
  return {lds32<32 * E>(v), lds32<32 * E - 8>(v), lds32<32 * E + 16>(v), lds32<32 * E + 8>(v)};
}
template <int E>
__device__ __forceinline__ Quad qvo(uint32_t v) {
  return {lds32<32 * E - 16>(v), lds32<32 * E - 24>(v), lds32<32 * E>(v), lds32<32 * E - 8>(v)};
}
__device__ __forceinline__ void imma_q(int (&d)[4], const Quad& a, uint32_t b0, uint32_t b1) {
  imma_s8(d, a.x, a.y, a.z, a.w, b0, b1);
}
__device__ __forceinline__ Quad uv_q(const Quad& f, const Quad& v) {
  return {uv_bytes(f.x, v.x), uv_bytes(f.y, v.y), uv_bytes(f.z, v.z), uv_bytes(f.w, v.w)};
}

// n consecutive 32-k columns of cross MMAs.  Tile r = 2i (+1) of column c
// reads the forward quad E (O) at e = c + i and the reversed quad E (O) at
// e = c - i (i = 0, 1).  The odd quads are halves of neighbouring even quads
// (fo(e) = {F(e).z, F(e).w, F(e+1).x, F(e+1).y}, vo(e) = {V(e-1).z, V(e-1).w,
// V(e).x, V(e).y}), so each column loads one new even quad per window: rings
// of three (slot = e mod 3, resolved at compile time).
__device__ __forceinline__ void cert_cross_run(uint32_t f, uint32_t v, uint32_t bd, int n,
                                               int (&acc)[kCertTiles][4]) {
  Quad F[3], V[3];
  F[0] = qfe<0>(f); F[1] = qfe<1>(f); F[2] = qfe<2>(f);
  V[0] = qve<0>(v); V[2] = qve<-1>(v);                      // V(-1) -> slot 2
  V[1] = {0u, 0u, lds32<-48>(v), lds32<-56>(v)};            // V(-2): only z, w are used
  auto column = [&](auto U_) {
    constexpr int U = decltype(U_)::value;                  // column mod 3
    const uint32_t b0 = lds32<0>(bd), b1 = lds32<16>(bd);
    const Quad& f0 = F[U];
    const Quad& f1 = F[(U + 1) % 3];
    const Quad& f2 = F[(U + 2) % 3];
    const Quad& v0 = V[U];
    const Quad& v1 = V[(U + 2) % 3];
    const Quad& v2 = V[(U + 1) % 3];
    imma_q(acc[0], uv_q(f0, v0), b0, b1);
    imma_q(acc[1], uv_q(Quad{f0.z, f0.w, f1.x, f1.y}, Quad{v1.z, v1.w, v0.x, v0.y}), b0, b1);
    imma_q(acc[2], uv_q(f1, v1), b0, b1);
    imma_q(acc[3], uv_q(Quad{f1.z, f1.w, f2.x, f2.y}, Quad{v2.z, v2.w, v1.x, v1.y}), b0, b1);
    // advance: F(c + 3) -> slot U, V(c + 1) -> slot U + 1
    f += 32; v += 32; bd += 32;
    F[U] = qfe<2>(f);
    V[(U + 1) % 3] = qve<0>(v);
  };
  int c = 0;
#pragma unroll 1
  for (; c + 3 <= n; c += 3) {
    column(std::integral_constant<int, 0>{});
    column(std::integral_constant<int, 1>{});
    column(std::integral_constant<int, 2>{});
  }
  if (c < n) column(std::integral_constant<int, 0>{});
  if (c + 1 < n) column(std::integral_constant<int, 1>{});
}

#if PSL_XTMEM
// ---- the cross term with TMEM-parked accumulators.  Warp w scores row group
// g = (w & 3) | (w >> 3) << 2 (rows 128 g .. 128 g + 127, 8 m16 tiles) over
// the column half h = (w >> 2) & 1 of every zone-1 chunk (columns 8h .. 8h + 7):
// per column one new forward and one new reversed quad feed 8 MMAs (half the
// shared-memory loads per MMA of 4 tiles x 16 columns).  The 32 accumulator
// registers live in TMEM between chunks (lanes 32 (w & 3) + lane, columns
// 128 + 32 (w >> 2)); warps w and w + 4 hold the two halves of the same rows.
constexpr int kXTiles = 8;
__device__ __forceinline__ uint32_t cert_xgroup(uint32_t w) { return (w & 3u) | ((w >> 3) << 2); }
__device__ __forceinline__ uint32_t cert_xhalf(uint32_t w) { return (w >> 2) & 1u; }
__device__ __forceinline__ uint32_t cert_xtaddr(uint32_t tmem, uint32_t w) {
  return tmem + ((32u * (w & 3u)) << 16) + 128u + 32u * (w >> 2);
}
__device__ __forceinline__ CertLane cert_lane8(const CertSmem& cs) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t gid = lane >> 2, tig = lane & 3;
  const uint32_t g = cert_xgroup(w), h = cert_xhalf(w);
  const uint32_t base_f = 128 * g + gid + 4 * tig, af = gid & 3;
  const uint32_t base_v = kY0 - 128 * g - gid + 4 * tig, av = base_v & 3;
  CertLane l;
  l.f = smem_u32(cs.winF) + af * kWinBytes + (base_f - af) + 256 * h;
  l.v = smem_u32(cs.winV) + av * kWinBytes + (base_v - av) + 256 * h;
  l.bd = smem_u32(cs.limbR) + gid * kLimbStride + 4 * tig + 256 * h;
  return l;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&a)[kXTiles][4]) {
  __syncwarp();
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(a[0][0]), "=r"(a[0][1]), "=r"(a[0][2]), "=r"(a[0][3]), "=r"(a[1][0]), "=r"(a[1][1]),
        "=r"(a[1][2]), "=r"(a[1][3]), "=r"(a[2][0]), "=r"(a[2][1]), "=r"(a[2][2]), "=r"(a[2][3]),
        "=r"(a[3][0]), "=r"(a[3][1]), "=r"(a[3][2]), "=r"(a[3][3]), "=r"(a[4][0]), "=r"(a[4][1]),
        "=r"(a[4][2]), "=r"(a[4][3]), "=r"(a[5][0]), "=r"(a[5][1]), "=r"(a[5][2]), "=r"(a[5][3]),
        "=r"(a[6][0]), "=r"(a[6][1]), "=r"(a[6][2]), "=r"(a[6][3]), "=r"(a[7][0]), "=r"(a[7][1]),
        "=r"(a[7][2]), "=r"(a[7][3])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const int (&a)[kXTiles][4]) {
  __syncwarp();
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(a[0][0]), "r"(a[0][1]), "r"(a[0][2]), "r"(a[0][3]), "r"(a[1][0]), "r"(a[1][1]),
        "r"(a[1][2]), "r"(a[1][3]), "r"(a[2][0]), "r"(a[2][1]), "r"(a[2][2]), "r"(a[2][3]),
        "r"(a[3][0]), "r"(a[3][1]), "r"(a[3][2]), "r"(a[3][3]), "r"(a[4][0]), "r"(a[4][1]),
        "r"(a[4][2]), "r"(a[4][3]), "r"(a[5][0]), "r"(a[5][1]), "r"(a[5][2]), "r"(a[5][3]),
        "r"(a[6][0]), "r"(a[6][1]), "r"(a[6][2]), "r"(a[6][3]), "r"(a[7][0]), "r"(a[7][1]),
        "r"(a[7][2]), "r"(a[7][3]) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// n consecutive columns for 8 tiles: tile 2i (+1), i = 0..3, reads the forward
// quad E (O) at e = c + i and the reversed quad E (O) at e = c - i; rings of
// five (F(c .. c+4), V(c-4 .. c); slot = e mod 5, resolved at compile time).
__device__ __forceinline__ void cert_cross_run8(uint32_t f, uint32_t v, uint32_t bd, int n,
                                                int (&acc)[kXTiles][4]) {
  constexpr int R = 5;
  Quad F[R], V[R];
  F[0] = qfe<0>(f); F[1] = qfe<1>(f); F[2] = qfe<2>(f); F[3] = qfe<3>(f); F[4] = qfe<4>(f);
  V[0] = qve<0>(v); V[4] = qve<-1>(v); V[3] = qve<-2>(v); V[2] = qve<-3>(v);   // V(e) -> slot e mod 5
  V[1] = {0u, 0u, lds32<-112>(v), lds32<-120>(v)};                            // V(-4): only z, w are used
  auto column = [&](auto U_) {
    constexpr int U = decltype(U_)::value;                  // column mod 5
    const uint32_t b0 = lds32<0>(bd), b1 = lds32<16>(bd);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const Quad& fa = F[(U + i) % R];
      const Quad& fb = F[(U + i + 1) % R];
      const Quad& va = V[(U - i + 2 * R) % R];
      const Quad& vb = V[(U - i - 1 + 2 * R) % R];
      imma_q(acc[2 * i], uv_q(fa, va), b0, b1);
      imma_q(acc[2 * i + 1], uv_q(Quad{fa.z, fa.w, fb.x, fb.y}, Quad{vb.z, vb.w, va.x, va.y}), b0, b1);
    }
    // advance: F(c + 5) -> slot U, V(c + 1) -> slot U + 1
    f += 32; v += 32; bd += 32;
    F[U] = qfe<4>(f);
    V[(U + 1) % R] = qve<0>(v);
  };
  // always the full half chunk: columns past m_lo have R4 = 0 (zero digit rows)
  (void)n;
  column(std::integral_constant<int, 0>{}); column(std::integral_constant<int, 1>{});
  column(std::integral_constant<int, 2>{}); column(std::integral_constant<int, 3>{});
  column(std::integral_constant<int, 4>{}); column(std::integral_constant<int, 0>{});
  column(std::integral_constant<int, 1>{}); column(std::integral_constant<int, 2>{});
}

// The cross MMAs of zone-1 chunk c (buffer c & 1) for this warp's rows and
// column half; the accumulators come from / go back to TMEM (zero at chunk 0,
// the first zone-1 chunk of every pass).
#ifndef PSL_XT_NOINLINE
#define PSL_XT_NOINLINE 0
#endif
#if PSL_XT_NOINLINE
__device__ __noinline__ void cert_cross_chunk(const CertIO& io, const CertSmem& cs, const CertLane& ln, uint32_t c,
                                              uint32_t tmem, uint32_t& nmma) {
#else
__device__ __forceinline__ void cert_cross_chunk(const CertIO& io, const CertSmem& cs, const CertLane& ln, uint32_t c,
                                                 uint32_t tmem, uint32_t& nmma) {
#endif
  const uint32_t kb = cert_kb(c);
  if (kb > io.m_lo) return;
#ifdef PSL_ABLATE_MMA
  return;
#endif
  const uint32_t w = threadIdx.x >> 5, g = cert_xgroup(w), h = cert_xhalf(w);
  const int rw_lo = max(128 * (int)g, (int)io.r_lo), rw_hi = min(128 * (int)g + 127, (int)io.r_hi - 1);
  if (rw_lo > rw_hi) return;
  // columns whose first shift is still in zone 1 (the rest of the chunk has R4 = 0), this half
  const int nall = (int)min((uint32_t)kCCols, (io.m_lo - kb) / 32 + 1);
  if (nall <= 8 * (int)h) return;
  const int n = 8;            // the whole half: its columns past m_lo add zero digits
  const uint32_t b = c & 1;
#ifdef PSL_DEBUG_BOUNDS
  {
    // every LDS whose value is used stays inside its own window copy / digit row
    // (the final ring refill after the last column is dead: it may read one
    // column past the copy, still inside the CTA's shared memory)
    const uint32_t wf = smem_u32(cs.winF), wv = smem_u32(cs.winV), lb = smem_u32(cs.limbR);
    const uint32_t f0 = ln.f + b * (uint32_t)kWinBuf - wf, v0 = ln.v + b * (uint32_t)kWinBuf - wv;
    const uint32_t cf = f0 % kWinBytes, cvv = v0 % kWinBytes;
    const uint32_t cb = ((ln.bd + b * (uint32_t)kLimbBuf - lb) % (uint32_t)kLimbBuf) % (uint32_t)kLimbStride;
    PSL_CHK(cf + 32u * (uint32_t)n + 124u <= (uint32_t)kWinBytes, 16);
    PSL_CHK(cvv >= 120u && cvv + 32u * (uint32_t)n - 12u <= (uint32_t)kWinBytes, 17);
    PSL_CHK(cb + 32u * (uint32_t)n - 12u <= (uint32_t)kLimbStride, 18);
  }
#endif
  nmma += (uint32_t)(n * kXTiles);
  int acc[kXTiles][4];
  const uint32_t ta = cert_xtaddr(tmem, w);
  if (c == 0) {
#pragma unroll
    for (int r = 0; r < kXTiles; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[r][e] = 0;
  } else {
    tmem_ld32(ta, acc);
  }
  cert_cross_run8(ln.f + b * (uint32_t)kWinBuf, ln.v + b * (uint32_t)kWinBuf,
                  ln.bd + b * (uint32_t)kLimbBuf, n, acc);
  tmem_st32(ta, acc);
}

// Cross accumulators -> per-row doubles: the half-0 warp of each row group adds
// its partner's (column half 1) int32 digit sums exactly, then rows 128 g + 16 r
// + gid (+8) as before (weights 256^d x 2^qR).  Call after a barrier with
// tcgen05.fence::after_thread_sync.
__device__ __forceinline__ void cert_cross_rows(uint32_t tmem, uint32_t m_lo, double unitR, double* xrow) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  if (cert_xhalf(w) != 0) return;
  const uint32_t g = cert_xgroup(w);
  int acc[kXTiles][4], acc1[kXTiles][4];
  const bool s0 = m_lo >= 1, s1 = m_lo >= 1 + 256;       // the halves ran in chunk 0 (zone 1 is a prefix)
  tmem_ld32(cert_xtaddr(tmem, w), acc);
  tmem_ld32(cert_xtaddr(tmem, w + 4), acc1);
  const double w0 = ldexp(unitR, 16 * tig), w1 = ldexp(unitR, 16 * tig + 8);
#pragma unroll
  for (int r = 0; r < kXTiles; ++r) {
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[r][e] = (s0 ? acc[r][e] : 0) + (s1 ? acc1[r][e] : 0);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      double p = __dadd_rn(__dmul_rn((double)acc[r][2 * hh], w0), __dmul_rn((double)acc[r][2 * hh + 1], w1));
      p = __dadd_rn(p, __shfl_xor_sync(FULL, p, 1));
      p = __dadd_rn(p, __shfl_xor_sync(FULL, p, 2));
      if (tig == 0) xrow[128 * g + 16 * r + gid + 8 * hh] = p;
    }
  }
}
#else
// The cross MMAs of zone-1 chunk c (buffer c & 1) for this warp's 128 rows.
__device__ __forceinline__ void cert_cross_chunk(const CertIO& io, const CertSmem& cs, const CertLane& ln, uint32_t c,
                                                 int (&acc)[kCertTiles][4], uint32_t& nmma) {
  const uint32_t kb = cert_kb(c);
  if (kb > io.m_lo) return;
#ifdef PSL_ABLATE_MMA
  return;
#endif
  const uint32_t w = threadIdx.x >> 5;
  const int rw_lo = max(64 * (int)w, (int)io.r_lo), rw_hi = min(64 * (int)w + 63, (int)io.r_hi - 1);
  if (rw_lo > rw_hi) return;
  // columns whose first shift is still in zone 1 (the rest of the chunk has R4 = 0)
  const int n = (int)min((uint32_t)kCCols, (io.m_lo - kb) / 32 + 1);
  const uint32_t b = c & 1;
#ifdef PSL_DEBUG_BOUNDS
  {
    // every LDS whose value is used stays inside its own window copy / digit row
    // (cert_cross_run's final ring refill after the last column is dead: it may
    // read one column past the copy, still inside the CTA's shared memory)
    const uint32_t wf = smem_u32(cs.winF), wv = smem_u32(cs.winV), lb = smem_u32(cs.limbR);
    const uint32_t f0 = ln.f + b * (uint32_t)kWinBuf - wf, v0 = ln.v + b * (uint32_t)kWinBuf - wv;
    const uint32_t cf = f0 % kWinBytes, cvv = v0 % kWinBytes;
    const uint32_t cb = ((ln.bd + b * (uint32_t)kLimbBuf - lb) % (uint32_t)kLimbBuf) % (uint32_t)kLimbStride;
    PSL_CHK(cf + 32u * (uint32_t)n + 28u <= (uint32_t)kWinBytes, 16);
    PSL_CHK(cvv >= 56u && cvv + 32u * (uint32_t)n - 12u <= (uint32_t)kWinBytes, 17);
    PSL_CHK(cb + 32u * (uint32_t)n - 12u <= (uint32_t)kLimbStride, 18);
  }
#endif
  nmma += (uint32_t)(n * kCertTiles);
  cert_cross_run(ln.f + b * (uint32_t)kWinBuf, ln.v + b * (uint32_t)kWinBuf,
                 ln.bd + b * (uint32_t)kLimbBuf, n, acc);
}

// Cross accumulator digits -> per-row doubles (rows 64w + 16r + g (+8)); the
// quad holds digit columns 2 tig, 2 tig + 1 (weights 256^d x 2^qR).
__device__ __forceinline__ void cert_cross_rows(const int (&acc)[kCertTiles][4], double unitR,
                                                double* xrow) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  const double w0 = ldexp(unitR, 16 * tig), w1 = ldexp(unitR, 16 * tig + 8);
#pragma unroll
  for (int r = 0; r < kCertTiles; ++r) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      double p = __dadd_rn(__dmul_rn((double)acc[r][2 * hh], w0), __dmul_rn((double)acc[r][2 * hh + 1], w1));
      p = __dadd_rn(p, __shfl_xor_sync(FULL, p, 1));
      p = __dadd_rn(p, __shfl_xor_sync(FULL, p, 2));
      if (tig == 0) xrow[64 * warp + 16 * r + gid + 8 * hh] = p;
    }
  }
}

#endif  // PSL_XTMEM

// TMEM accumulators -> per-row doubles, all 16 warps: warps 0-7 the forward
// accumulators (-> linrow), 8-15 the reversed ones (-> linrev); warp w reads TMEM
// lanes 32 (w & 3) .. + 31 and N-groups 4 ((w >> 2) & 1) .. + 3, four loads in
// flight before one wait.  Forward lane rho, N-group g -> u = rho + 128 (7 - g);
// reversed lane r -> u = 127 - r + 128 g; value = sum_d digit-column d x 256^d x 2^qH.
// The row's linear term is linrow + linrev (one rounding, as fwd then += rev).
__device__ __forceinline__ void cert_lin_rows(uint32_t tmem, uint32_t started, double unitH, const CertIO& io,
                                              double* linrow, double* linrev) {
  const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rev = w >= 8;
  const uint32_t rho = 32 * (w & 3) + lane, g0 = 4 * ((w >> 2) & 1);
  const uint32_t col0 = rev ? 64u : 0u;
  const bool have = (started >> (rev ? 1 : 0)) & 1u;
  uint32_t v[4][8];
#pragma unroll
  for (int gg = 0; gg < 4; ++gg) {
    const uint32_t addr = tmem + ((32u * (w & 3)) << 16) + col0 + 8 * (g0 + gg);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[gg][0]), "=r"(v[gg][1]), "=r"(v[gg][2]), "=r"(v[gg][3]), "=r"(v[gg][4]),
                   "=r"(v[gg][5]), "=r"(v[gg][6]), "=r"(v[gg][7])
                 : "r"(addr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  double* out = rev ? linrev : linrow;
#pragma unroll
  for (int gg = 0; gg < 4; ++gg) {
    const uint32_t g = g0 + gg;
    double x = 0.0;
    if (have) {
#pragma unroll
      for (int d = 7; d >= 0; --d) x = __dadd_rn(__dmul_rn(x, 256.0), (double)(int32_t)v[gg][d]);
      x = __dmul_rn(x, unitH);
    }
    const uint32_t u = rev ? 127 - rho + 128 * g : rho + 128 * (7 - g);
    const uint32_t r = io.r_lo + u;
    if (u < io.r_hi - io.r_lo && r < (uint32_t)kGroup) out[r] = x;
  }
}

// Band 1 (k in (m_lo, m_hi], <= n shifts wide), scored exactly per cell after
// the chunk loop.  In band 1 row j's cell is two-sided for k <= m_j and
// one-sided past it (s_{j+k} for rows left of the middle, s_{j-k} right of
// it; m_hi <= (L-1)/2 <= M_j), so with du = [s_{j+k} != s_j], dv = [s_{j-k} != s_j]
// its term is entry code of the shift's 8-entry record
//   code = 2 du + dv (two-sided: e4, e2, e2, e0),  4 + dw (one-sided: e3, e1),
// e_x = pow_int(|C_k - 2(x - 2)|, alpha).  The records live in the digit ring
// (free once the MMAs drained): one LDS.64 per cell, no dependent lookups.
constexpr int kBandRows = kGroup / kCertThreads;    // rows per thread (rho = kBandRows t + m)
constexpr uint32_t kBandRec = 8;                     // doubles per band record
static_assert((size_t)kGroup * kBandRec * sizeof(double) <= kDRing, "band records fit the digit ring");

// The pivot words band 1 reads (logical word w = sb[w + 1]), staged in the
// record buffer: forward positions j + k, backward j - k - 31, the rows' own bits.
constexpr uint32_t kBandWF = 80, kBandWB = 80, kBandWR = 40;
static_assert((kBandWF + kBandWB + kBandWR) * 4 <= kCertRecBuf * 2, "band bit windows fit the record buffer");
struct BandBits {
  long long f0, b0, r0;     // first logical word of each window
};
__device__ __forceinline__ BandBits cert_band_bits(const CertIO& io) {
  const long long jlo = (long long)io.j0 + io.r_lo, jhi = (long long)io.j0 + io.r_hi - 1;
  const long long blo = (long long)io.m_lo + 1, bhi = min((long long)io.m_hi, (long long)io.L - 1);
  BandBits w;
  w.f0 = (jlo + blo) >> 5;
  w.b0 = (jlo - bhi - 62) >> 5;
  w.r0 = jlo >> 5;
  return w;
}

// Records of the band shifts and the staged pivot words (all threads; C after
// the fold, visible after a barrier).
__device__ __forceinline__ void cert_band_records(const CertIO& io, const CertSmem& cs, const int32_t* Cf,
                                                  const uint32_t* sb) {
  const uint32_t blo = io.m_lo + 1, bhi = min(io.m_hi, io.L - 1);
  {
    const BandBits bw = cert_band_bits(io);
    const long long jlo = (long long)io.j0 + io.r_lo, jhi = (long long)io.j0 + io.r_hi - 1;
    const uint32_t nf = (uint32_t)(((jhi + bhi + 63) >> 5) - bw.f0 + 1);
    const uint32_t nb = (uint32_t)(((jhi - (long long)blo) >> 5) + 2 - bw.b0);
    const uint32_t nr = (uint32_t)((jhi >> 5) - bw.r0 + 1);
    PSL_CHK(nf <= kBandWF && nb <= kBandWB && nr <= kBandWR, 21);
    uint32_t* wf = reinterpret_cast<uint32_t*>(cs.rec);
    for (uint32_t i = threadIdx.x; i < nf + nb + nr; i += blockDim.x) {
      const long long lw = i < nf ? bw.f0 + i : (i < nf + nb ? bw.b0 + (i - nf) : bw.r0 + (i - nf - nb));
      const uint32_t slot = i < nf ? i : (i < nf + nb ? kBandWF + (i - nf) : kBandWF + kBandWB + (i - nf - nb));
      PSL_CHK(sb_ok(lw + 1, io.L), 21);
      wf[slot] = sb[lw + 1];
    }
  }
  double* tab = reinterpret_cast<double*>(cs.dring);
  for (uint32_t i = threadIdx.x; blo + i <= bhi; i += blockDim.x) {
    PSL_CHK(i < (uint32_t)kGroup && blo + i >= 1 && blo + i < io.L, 19);
    const int32_t c = __ldcg(Cf + blo + i);
    const double e4 = io.lut[abs(c - 4)], e3 = io.lut[abs(c - 2)], e2 = io.lut[abs(c)];
    const double e1 = io.lut[abs(c + 2)], e0 = io.lut[abs(c + 4)];
    double2* r = reinterpret_cast<double2*>(tab + (size_t)kBandRec * i);
    r[0] = make_double2(e4, e2);
    r[1] = make_double2(e2, e0);
    r[2] = make_double2(e3, e1);
    r[3] = make_double2(0.0, 0.0);
  }
}

// 4 bits -> 4 bytes (bit i -> byte i = 0 / 1)
__device__ __forceinline__ uint32_t spread4(uint32_t x) { return ((x & 0xFu) * 0x00204081u) & 0x01010101u; }

// Row sums of band-1 cells for this thread's rows (in ascending k, two
// interleaved partial sums per row: depth <= n / 2 + 2, inside the gamma_2100
// budget of the bound).
__device__ __forceinline__ void cert_band_rows(const CertIO& io, const CertSmem& cs, double (&Bs)[kBandRows]) {
  const uint32_t blo = io.m_lo + 1, bhi = min(io.m_hi, io.L - 1);
  if (blo > bhi) return;
  const uint32_t L = io.L;
  const unsigned char* tab = cs.dring;
  const BandBits bw = cert_band_bits(io);
  const uint32_t* sF = reinterpret_cast<const uint32_t*>(cs.rec);
  const uint32_t* sB = sF + kBandWF;
  const uint32_t* sR = sB + kBandWB;
#ifdef PSL_ABLATE_BAND
  return;
#endif
#pragma unroll 1
  for (int m = 0; m < kBandRows; ++m) {
    const uint32_t rho = kBandRows * threadIdx.x + m;
    if (rho < io.r_lo || rho >= io.r_hi) continue;
    const uint32_t j = (uint32_t)(io.j0 + (int32_t)rho);
    const uint32_t mj = min(j, L - 1 - j);
    const bool left = j <= L - 1 - j;                  // one-sided cells use s_{j+k}
    const uint32_t sjm = ((sR[(long long)(j >> 5) - bw.r0] >> (j & 31)) & 1u) ? 0xFFFFFFFFu : 0u;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll 1
    for (uint32_t k0 = blo; k0 <= bhi; k0 += 32) {
      // bit q: s_{j+k0+q} and s_{j-k0-q} (1 <-> -1; zero pads beyond the ends are never selected)
      const long long pB = (long long)j + k0, pA = (long long)j - k0 - 31;
      const int32_t wB = (int32_t)((pB >> 5) - bw.f0), wA = (int32_t)((pA >> 5) - bw.b0);
      PSL_CHK(wB >= 0 && wB + 1 < (int32_t)kBandWF && wA >= 0 && wA + 1 < (int32_t)kBandWB, 20);
      const uint32_t Du = __funnelshift_r(sF[wB], sF[wB + 1], (uint32_t)(pB & 31)) ^ sjm;
      const uint32_t Dv = __brev(__funnelshift_r(sB[wA], sB[wA + 1], (uint32_t)(pA & 31))) ^ sjm;
      // two-sided cells: q < d = m_j - k0 + 1
      const int d = (int)mj - (int)k0 + 1;
      const uint32_t A = d >= 32 ? 0xFFFFFFFFu : (d <= 0 ? 0u : (1u << d) - 1u);
      const uint32_t W4 = ~A, W2 = Du & A, W1 = left ? ((A & Dv) | (~A & Du)) : Dv;
      const unsigned char* base = tab + (k0 - blo) * (uint32_t)(kBandRec * sizeof(double));
      const uint32_t nq = min(32u, bhi - k0 + 1);     // CTA-uniform
      // 8 x code per byte, 4 cells per word; blocks where every lane of the warp is
      // two-sided (code 2du + dv) or one-sided (4 + dw) skip the third bit plane
      const uint32_t am = __activemask();
      const bool allA = __all_sync(am, d >= 32), allB = __all_sync(am, d <= 0);
      uint32_t c8[8];
      if (allA) {
#pragma unroll
        for (int g = 0; g < 8; ++g) c8[g] = ((spread4(Du >> (4 * g)) << 1) + spread4(Dv >> (4 * g))) << 3;
      } else if (allB) {
        const uint32_t Dw = left ? Du : Dv;
#pragma unroll
        for (int g = 0; g < 8; ++g) c8[g] = 0x20202020u + (spread4(Dw >> (4 * g)) << 3);
      } else {
#pragma unroll
        for (int g = 0; g < 8; ++g)
          c8[g] = ((((spread4(W4 >> (4 * g)) << 1) + spread4(W2 >> (4 * g))) << 1) + spread4(W1 >> (4 * g))) << 3;
      }
      PSL_CHK(k0 - blo + nq <= (uint32_t)kGroup, 20);
      if (nq == 32) {                                   // full block: branch-free, loads hoisted
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double e[16];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            e[q] = *reinterpret_cast<const double*>(
                base + __byte_perm(c8[4 * h + (q >> 2)], 0u, 0x4440u + (uint32_t)(q & 3)) +
                (16 * h + q) * kBandRec * sizeof(double));
#pragma unroll
          for (int q = 0; q < 16; q += 2) { s0 = __dadd_rn(s0, e[q]); s1 = __dadd_rn(s1, e[q + 1]); }
        }
      } else {
#pragma unroll 1
        for (uint32_t q = 0; q < nq; ++q) {
          const uint32_t off = (((W4 >> q) & 1u) << 5) | (((W2 >> q) & 1u) << 4) | (((W1 >> q) & 1u) << 3);
          const double e = *reinterpret_cast<const double*>(base + off + q * kBandRec * sizeof(double));
          if (q & 1) s1 = __dadd_rn(s1, e); else s0 = __dadd_rn(s0, e);
        }
      }
    }
    Bs[m] = __dadd_rn(s0, s1);
  }
}

// fitness() of the folded table (sequence.cpp:131-141): one thread adds the
// chunk's terms lut[|C_k|] in ascending k to the serial double chain.
__device__ __forceinline__ void cert_chain_chunk(const CertIO& io, const CertSmem& cs, uint32_t c,
                                                 double& chain) {
  const uint32_t kb = cert_kb(c);
  const uint32_t nk = min(kCC, io.L - kb);
  const int32_t* rec = cs.rec + (size_t)(c & 1) * kCC;
  for (uint32_t i = 0; i < nk; ++i) chain = __dadd_rn(chain, io.lut[abs(rec[i])]);
}

// Band 2 (k in (M_lo, M_hi]): row j's constant is sum_{k <= M_j} 4M_k +
// sum_{k > M_j} 4 e2_k.  b2M becomes its inclusive prefix sums, b2E its
// inclusive suffix sums, over the whole CTA (two elements per thread, warp
// shuffle scans, one pass over the warp totals in `wsum` [2][32] shared):
// every sum has depth <= 2 + 5 + 5 + 2, inside the bound's gamma_128.
__device__ __forceinline__ void cert_band2_scan(const CertIO& io, uint32_t nb2, double* wsum) {
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5, nwp = blockDim.x >> 5;
  const uint32_t i0 = 2 * t, i1 = 2 * t + 1;          // b2M index / b2E index from the top
  PSL_CHK(nb2 <= 2 * blockDim.x && nb2 <= (uint32_t)kGroup, 5);
  const double m0 = i0 < nb2 ? __ldcg(io.b2M + i0) : 0.0, m1 = i1 < nb2 ? __ldcg(io.b2M + i1) : 0.0;
  const double e0 = i0 < nb2 ? __ldcg(io.b2E + (nb2 - 1 - i0)) : 0.0;
  const double e1 = i1 < nb2 ? __ldcg(io.b2E + (nb2 - 1 - i1)) : 0.0;
  const double qm = __dadd_rn(m0, m1), qe = __dadd_rn(e0, e1);
  double pm = qm, pe = qe;                              // inclusive over the warp's pairs
  for (int o = 1; o < 32; o <<= 1) {
    const double a = __shfl_up_sync(FULL, pm, o), b = __shfl_up_sync(FULL, pe, o);
    if ((int)lane >= o) { pm = __dadd_rn(pm, a); pe = __dadd_rn(pe, b); }
  }
  double xm = __shfl_up_sync(FULL, pm, 1), xe = __shfl_up_sync(FULL, pe, 1);   // exclusive
  if (lane == 0) { xm = 0.0; xe = 0.0; }
  if (lane == 31) { wsum[warp] = pm; wsum[32 + warp] = pe; }
  __syncthreads();
  if (warp == 0) {                                      // exclusive scan of the warp totals
    double a = lane < nwp ? wsum[lane] : 0.0, b = lane < nwp ? wsum[32 + lane] : 0.0;
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(FULL, a, o), v = __shfl_up_sync(FULL, b, o);
      if ((int)lane >= o) { a = __dadd_rn(a, u); b = __dadd_rn(b, v); }
    }
    double ea = __shfl_up_sync(FULL, a, 1), eb = __shfl_up_sync(FULL, b, 1);
    if (lane == 0) { ea = 0.0; eb = 0.0; }
    __syncwarp();
    if (lane < nwp) { wsum[lane] = ea; wsum[32 + lane] = eb; }
  }
  __syncthreads();
  const double cm = __dadd_rn(wsum[warp], xm), ce = __dadd_rn(wsum[32 + warp], xe);
  const double am = __dadd_rn(cm, m0), ae = __dadd_rn(ce, e0);
  if (i0 < nb2) { io.b2M[i0] = am; io.b2E[nb2 - 1 - i0] = ae; }
  if (i1 < nb2) { io.b2M[i1] = __dadd_rn(am, m1); io.b2E[nb2 - 1 - i1] = __dadd_rn(ae, e1); }
}
__device__ __forceinline__ double cert_band2_const(const CertIO& io, uint32_t nb2, uint32_t i) {
  return __dadd_rn(i > 0 ? io.b2M[i - 1] : 0.0, i < nb2 ? io.b2E[i] : 0.0);
}

// gamma_n = n u / (1 - n u), u = 2^-53 (Higham)
__device__ __forceinline__ double gamma_n(double n) {
  const double u = 0x1p-53;
  return n * u / (1.0 - n * u);
}
