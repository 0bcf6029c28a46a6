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
// so with zones over the 1024-row window (m_j = min(j, L-1-j), M_j = L-1-m_j):
//   4T(j) = S_P + S_M + S_E                       (window-wide constants, k in Z1/Z3/Z5)
//         + s_j sum_k H4_k (s_{j+k} + s_{j-k})    (H4 = 4Q in Z1, 4N in Z3: a correlation)
//         + sum_{k in Z1} 4R_k s_{j+k} s_{j-k}    (the both-sides cross term)
//         + 4 * (exact terms of the two <= n-wide bands where the zone depends on j)
// The two correlations run on the tensor cores (mma.sync s8): the sequence as
// +-1 bytes (A, rows = neighbours, Hankel in k), H4 / R4 as 8 balanced base-256
// digits of a fixed-point value (B, one digit per column), int32 accumulation
// (exact).  Everything else is per-k work in the builder.
#pragma once

constexpr int kCertTiles = 8;                 // m16 row tiles per warp (128 rows)
constexpr int kCertCols = kChunk / 32;        // k columns of 32 per chunk
constexpr int kLimbStride = kChunk + 16;      // bytes per digit row (bank spread)
constexpr int kWinBytes = 1568;               // staged bytes per copy (392 words, = 8 mod 32)
constexpr int kY0 = 1031;                     // origin of the reversed window
constexpr size_t kLimbBuf = 8ull * kLimbStride;          // one table, one buffer
constexpr size_t kWinBuf = 4ull * kWinBytes;             // one direction (4 copies), one buffer
constexpr size_t kCertRecBuf = (size_t)kChunk * sizeof(int32_t);
constexpr size_t kCertRowBytes = (size_t)kGroup * sizeof(double);
constexpr size_t kCertCBuf = (size_t)kChunk * sizeof(int32_t);     // C_k prefetch ring slot
constexpr size_t kCertB2 = (size_t)kGroup * sizeof(double);        // band-2 constants
// [digits 2][win_f 2][win_r 2][rec 2][xrow][C ring 3][band2 M, E]
constexpr size_t kCertBytes = 2 * kLimbBuf + 4 * kWinBuf + 2 * kCertRecBuf + kCertRowBytes +
                              3 * kCertCBuf + 2 * kCertB2;
// fixed-point digits per shift: H4 (the correlation coefficient) in digit
// columns 0..4 (40 bits), R4 (the cross coefficient) in columns 5..7 (24 bits),
// each with its own power-of-two unit; the MMA accumulates both into one
// m16n8 tile (B of the linear MMAs carries zeros in 5..7, the cross MMA's in 0..4)
constexpr int kDigH = 5, kDigR = 3;
constexpr long long kMaxH = 0x7F7F7F7F7Fll, kMaxR = 0x7F7F7Fll;
constexpr uint32_t kCertMinL = 2048;

struct CertIO {
  uint32_t L, n, nchunks;
  int32_t j0;                                 // rows j = j0 + rho (may be < 0 for inactive rows)
  uint32_t r_lo, r_hi;                        // active rows of this pass: r_lo <= rho < r_hi
  const int32_t* Csrc;
  int32_t* Cdst;
  int32_t* Cloc;
  const uint32_t* flips;
  uint32_t F;
  uint32_t f1;                                // flips[0] and s_{f1} (after) when F == 1
  int sf1;
  uint32_t alpha;
  const double* lut;                          // PowerTable of the phase (covers |C_k| + 4)
  int2* hlist;
  uint32_t* hcount;
  int32_t hthr;
  double scaleH, scaleR;                      // 2^-qH, 2^-qR
  uint32_t m_lo, m_hi, M_lo, M_hi;            // zone bounds (see above)
};

struct CertSmem {
  unsigned char* limbH;   // [2][8][kLimbStride] digit rows (H4: 0-4, R4: 5-7)
  unsigned char* winF;    // [2][4][kWinBytes]  F[x] = s_{j0+kb+x}
  unsigned char* winV;    // [2][4][kWinBytes]  V[y] = s_{j0-kb+kY0-y}
  int32_t* rec;           // [2][kChunk]        C_k (band chunks only)
  double* xrow;           // [1024]             cross-term sums per row
  int32_t* cring;         // [3][kChunk]        C_k of chunks c+1, c+2 in flight (cp.async)
  double* b2M;            // [1024] 4M_k = 2(e3+e1), k = M_lo+1+i (band 2: one side or none)
  double* b2E;            // [1024] 4 e2_k
};

__device__ __forceinline__ CertSmem cert_carve(unsigned char* base) {
  CertSmem m;
  m.limbH = base;
  m.winF = base + 2 * kLimbBuf;
  m.winV = base + 2 * kLimbBuf + 2 * kWinBuf;
  m.rec = reinterpret_cast<int32_t*>(base + 2 * kLimbBuf + 4 * kWinBuf);
  m.xrow = reinterpret_cast<double*>(base + 2 * kLimbBuf + 4 * kWinBuf + 2 * kCertRecBuf);
  m.cring = reinterpret_cast<int32_t*>(base + 2 * kLimbBuf + 4 * kWinBuf + 2 * kCertRecBuf +
                                       kCertRowBytes);
  m.b2M = reinterpret_cast<double*>(base + 2 * kLimbBuf + 4 * kWinBuf + 2 * kCertRecBuf +
                                    kCertRowBytes + 3 * kCertCBuf);
  m.b2E = m.b2M + kGroup;
  return m;
}

__device__ __forceinline__ bool cert_band_chunk(const CertIO& io, uint32_t c) {
  const uint32_t kb = 1 + c * kChunk, ke = kb + kChunk - 1;
  return kb <= io.m_hi && ke > io.m_lo;      // band 1 (band 2 is linear: MMA + prefix sums)
}

// any k column with nonzero H4 / R4 (Z1, Z3, band 2) in the chunk starting at kb
__device__ __forceinline__ bool cert_mma_work(const CertIO& io, uint32_t kb) {
  return kb <= io.m_lo || (kb + kChunk - 1 > io.m_hi && kb <= io.M_hi);
}

// +-1 / 0 bytes of the staged windows
__device__ __forceinline__ uint32_t nib_bytes(uint32_t nib) {
  return ((nib * 0x00204081u) & 0x01010101u) * 0xFEu + 0x01010101u;
}
__device__ __forceinline__ uint32_t sbyte(const uint32_t* sb, long long p, uint32_t L) {
  if (p < 0 || p >= (long long)L) return 0u;
  return ((sb[(p >> 5) + 1] >> (p & 31)) & 1u) ? 0xFFu : 0x01u;
}

// C_k of this thread's two shifts of chunk c -> ring slot c % 3, asynchronously
// (cp.async, zero-filled past L); the thread itself consumes them in cert_build
__device__ __forceinline__ void cert_prefetch(const CertIO& io, const CertSmem& cs, uint32_t c) {
  const uint32_t k = 1 + c * kChunk + 2 * threadIdx.x;
  int32_t* dst = cs.cring + (size_t)(c % 3) * kChunk + 2 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool in = k + i < io.L;
    const int32_t* src = io.Csrc + (in ? k + i : 0);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst + i)), "l"(src),
                 "r"(in ? 4 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ int2 cert_take(const CertSmem& cs, uint32_t c, bool newest_pending) {
  if (newest_pending) asm volatile("cp.async.wait_group 1;" ::: "memory");
  else asm volatile("cp.async.wait_group 0;" ::: "memory");
  const int32_t* p = cs.cring + (size_t)(c % 3) * kChunk + 2 * threadIdx.x;
  return make_int2(p[0], p[1]);
}

// Builder for chunk c into buffer b: fold pending flips into C, write C back,
// collect high sidelobes, expand into the fixed-point digit rows of H4 / R4,
// the window constants and (band chunks) the exact term records; stage the
// sequence windows the MMAs read.
__device__ __forceinline__ void cert_build(const CertIO& io, const CertSmem& cs, uint32_t c,
                                           uint32_t b, const uint32_t* sb, int32_t& pmax,
                                           double (&part)[5], int2 cpre, bool& ovf) {
  const uint32_t t = threadIdx.x;
  const uint32_t kb = 1 + c * kChunk;
  const bool band = cert_band_chunk(io, c);
  int32_t* rec = cs.rec + (size_t)b * kChunk;
  uint64_t VD[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const uint32_t r = 2 * t + i;
    const uint32_t k = kb + r;
    bool want = false;
    int32_t cv = 0;
    if (k < io.L) {
      cv = i == 0 ? cpre.x : cpre.y;
      if (io.F == 1) {
        // the common single move: C_k += 2 s_f (s_{f-k} + s_{f+k}), s_f after the flip
        const uint32_t f = io.f1;
        const int acc = (k <= f ? sval(sb, f - k) : 0) + (f + k < io.L ? sval(sb, f + k) : 0);
        cv += 2 * io.sf1 * acc;
      } else if (io.F) {
        SweepIO fio;
        fio.L = io.L; fio.flips = io.flips; fio.F = io.F;
        cv = fold_flips(cv, k, fio, sb);
      }
      if (io.Cdst) io.Cdst[k] = cv;
      if (io.Cloc) io.Cloc[k] = cv;
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
        if (want) io.hlist[base + __popc(m & ((1u << lane) - 1))] = make_int2((int)k, cv);
      }
    }
    // per zone only the terms it needs (PowerTable lookups, e_x = E_k(x))
    double H = 0.0, R = 0.0;
    if (k < io.L) {
      if (k <= io.m_lo) {                               // Z1: both sides for every row
        const double e4 = __ldg(io.lut + abs(cv - 4)), e0 = __ldg(io.lut + abs(cv + 4));
        const double e2 = __ldg(io.lut + abs(cv));
        H = __dsub_rn(e4, e0);
        R = __dsub_rn(__dadd_rn(e4, e0), __dmul_rn(2.0, e2));
        part[0] = __dadd_rn(part[0], __dadd_rn(__dadd_rn(e4, e0), __dmul_rn(2.0, e2)));
      } else if (k <= io.m_hi) {                        // band 1: exact terms per row
      } else if (k <= io.M_hi) {                        // Z3 / band 2: one side or none
        const double e3 = __ldg(io.lut + abs(cv - 2)), e1 = __ldg(io.lut + abs(cv + 2));
        H = __dmul_rn(2.0, __dsub_rn(e3, e1));
        const double m4 = __dmul_rn(2.0, __dadd_rn(e3, e1));
        if (k <= io.M_lo) {
          part[1] = __dadd_rn(part[1], m4);
        } else {                                        // band 2: per-row prefix sums
          cs.b2M[k - io.M_lo - 1] = m4;
          cs.b2E[k - io.M_lo - 1] = __dmul_rn(4.0, __ldg(io.lut + abs(cv)));
        }
      } else {                                          // Z5: no side for any row
        part[2] = __dadd_rn(part[2], __dmul_rn(4.0, __ldg(io.lut + abs(cv))));
      }
    }
    // fixed point -> balanced base-256 digits: H4 in bytes 0..4, R4 in 5..7
    const long long hv = __double2ll_rn(__dmul_rn(H, io.scaleH));
    const long long rv = __double2ll_rn(__dmul_rn(R, io.scaleR));
    ovf |= hv > kMaxH || hv < -kMaxH || rv > kMaxR || rv < -kMaxR;
    const unsigned long long dh = ((unsigned long long)hv + 0x8080808080ull) ^ 0x8080808080ull;
    const unsigned long long dr = ((unsigned long long)rv + 0x808080ull) ^ 0x808080ull;
    VD[i] = (dh & 0xFFFFFFFFFFull) | ((dr & 0xFFFFFFull) << 40);
    if (band) rec[r] = cv;
  }
  if (!cert_mma_work(io, kb)) return;   // no MMA reads this chunk's digits / windows
  // digit d of the two k's -> one u16 per digit row (PRMT gathers byte d of each)
  unsigned char* lh = cs.limbH + (size_t)b * kLimbBuf + 2 * t;
  const uint32_t h0l = (uint32_t)VD[0], h0h = (uint32_t)(VD[0] >> 32);
  const uint32_t h1l = (uint32_t)VD[1], h1h = (uint32_t)(VD[1] >> 32);
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const uint32_t sel = (uint32_t)(d & 3) | ((uint32_t)(4 + (d & 3)) << 4);
    const uint32_t h = __byte_perm(d < 4 ? h0l : h0h, d < 4 ? h1l : h1h, sel);
    *reinterpret_cast<uint16_t*>(lh + d * kLimbStride) = (uint16_t)h;
  }
  // sequence windows: 4 copies x 392 words per direction, only the directions
  // some row still has in range
#ifdef PSL_ABLATE_STAGE
  return;
#endif
  const int L = (int)io.L, j0 = io.j0;
  const bool nf = j0 + (int)io.r_lo + (int)kb < L, nv = (int)kb <= j0 + (int)io.r_hi - 1;
  constexpr int kW = kWinBytes / 4;
  // thread -> base word q of one direction: bytes 4q..4q+7 of the base copy
  // from one bit window, copy a word q = base bytes 4q+a..4q+a+3
  const int total = (nf ? kW : 0) + (nv ? kW : 0);
  for (int idx = (int)t; idx < total; idx += kThreads) {
    const int dir = nf ? (idx >= kW ? 1 : 0) : 1;
    const int q = nf && dir ? idx - kW : idx;
    // fwd: byte i <-> position p0 + i; rev: byte i <-> position p0 - i (i = 0..7)
    const int p0 = dir == 0 ? j0 + (int)kb + 4 * q : j0 - (int)kb + kY0 - 4 * q;
    const int lo = dir == 0 ? p0 : p0 - 7, hi = lo + 7;
    uint32_t w0 = 0, w1 = 0;
    if (hi >= 0 && lo < L) {
      if (lo >= 0 && hi < L) {
        uint32_t x = __funnelshift_r(sb[(lo >> 5) + 1], sb[(lo >> 5) + 2], (uint32_t)lo & 31) & 0xFFu;
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
    *reinterpret_cast<uint32_t*>(dst) = w0;
    *reinterpret_cast<uint32_t*>(dst + kWinBytes) = __funnelshift_r(w0, w1, 8);
    *reinterpret_cast<uint32_t*>(dst + 2 * kWinBytes) = __funnelshift_r(w0, w1, 16);
    *reinterpret_cast<uint32_t*>(dst + 3 * kWinBytes) = __funnelshift_r(w0, w1, 24);
  }
}

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

// Per-lane shared addresses (buffer 0) of this warp's MMA operands.  Row rho =
// 128 w + 16 r + g (+8 for a1/a3), fragment layout of mma.m16n8k32 (row.col):
//   forward word m (bytes 8m..8m+3 past base_f = 128w + g + 4t) = s_{j+k} for
//     m = 2r + 4c + {0: a0, 1: a1, 2: a2, 3: a3}
//   reversed word m' (past base_v = kY0 - 128w - g + 4t) = s_{j-k} for
//     m' = 4c - 2r + {0: a0, -1: a1, 2: a2, 1: a3}
struct CertLane {
  uint32_t f, v, bd;
  bool dh;                    // this lane's B column (= g) is an H4 digit (g < 5)
};
__device__ __forceinline__ CertLane cert_lane(const CertSmem& cs) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t gid = lane >> 2, tig = lane & 3;
  const uint32_t base_f = 128 * w + gid + 4 * tig, af = gid & 3;
  const uint32_t base_v = kY0 - 128 * w - gid + 4 * tig, av = base_v & 3;
  CertLane l;
  l.f = smem_u32(cs.winF) + af * kWinBytes + (base_f - af);
  l.v = smem_u32(cs.winV) + av * kWinBytes + (base_v - av);
  l.bd = smem_u32(cs.limbH) + gid * kLimbStride + 4 * tig;
  l.dh = gid < (uint32_t)kDigH;
  return l;
}

struct Quad {
  uint32_t x, y, z, w;
};
// tile-quads of the sliding windows (see cert_run): forward E/O at e, reversed E/O at e
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

// n consecutive 32-k columns of one warp-uniform mode.  Tile r = 2i (+1) of
// relative column c reads the forward quad E (O) at e = c + i and the reversed
// quad E (O) at e = c - i: each column loads one new quad per window (ring of
// four, slot = e mod 4, resolved at compile time) instead of all eight.
template <bool FWD, bool REV, bool CRS>
__device__ __forceinline__ void cert_run(uint32_t f, uint32_t v, uint32_t bd, bool dh, int n,
                                         int (&acc)[kCertTiles][4]) {
  constexpr bool F = FWD || CRS, V = REV || CRS;
  Quad fe[4], fo[4], ve[4], vo[4];
  if (F) { fe[0] = qfe<0>(f); fo[0] = qfo<0>(f); fe[1] = qfe<1>(f); fo[1] = qfo<1>(f);
           fe[2] = qfe<2>(f); fo[2] = qfo<2>(f); fe[3] = qfe<3>(f); fo[3] = qfo<3>(f); }
  // reversed quads e = 0, -1, -2, -3 -> slots 0, 3, 2, 1
  if (V) { ve[0] = qve<0>(v); vo[0] = qvo<0>(v); ve[3] = qve<-1>(v); vo[3] = qvo<-1>(v);
           ve[2] = qve<-2>(v); vo[2] = qvo<-2>(v); ve[1] = qve<-3>(v); vo[1] = qvo<-3>(v); }
  auto column = [&](auto U) {
    constexpr int u = decltype(U)::value;       // relative column mod 4
    uint32_t bl0 = 0, bl1 = 0, bx0 = 0, bx1 = 0;
    {
      const uint32_t b0 = lds32<0>(bd), b1 = lds32<16>(bd);
      if (FWD || REV) { bl0 = dh ? b0 : 0u; bl1 = dh ? b1 : 0u; }
      if (CRS) { bx0 = dh ? 0u : b0; bx1 = dh ? 0u : b1; }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (FWD) {
        imma_q(acc[2 * i], fe[(u + i) & 3], bl0, bl1);
        imma_q(acc[2 * i + 1], fo[(u + i) & 3], bl0, bl1);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (REV) {
        imma_q(acc[2 * i], ve[(u - i + 8) & 3], bl0, bl1);
        imma_q(acc[2 * i + 1], vo[(u - i + 8) & 3], bl0, bl1);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (CRS) {
        imma_q(acc[2 * i], uv_q(fe[(u + i) & 3], ve[(u - i + 8) & 3]), bx0, bx1);
        imma_q(acc[2 * i + 1], uv_q(fo[(u + i) & 3], vo[(u - i + 8) & 3]), bx0, bx1);
      }
    }
    // advance: forward e = c + 4 -> slot u; reversed e = c + 1 -> slot u + 1
    f += 32; v += 32; bd += 32;
    if (F) { fe[u] = qfe<3>(f); fo[u] = qfo<3>(f); }
    if (V) { ve[(u + 1) & 3] = qve<0>(v); vo[(u + 1) & 3] = qvo<0>(v); }
  };
  int c = 0;
#pragma unroll 1
  for (; c + 4 <= n; c += 4) {
    column(std::integral_constant<int, 0>{});
    column(std::integral_constant<int, 1>{});
    column(std::integral_constant<int, 2>{});
    column(std::integral_constant<int, 3>{});
  }
  if (c < n) column(std::integral_constant<int, 0>{});
  if (c + 1 < n) column(std::integral_constant<int, 1>{});
  if (c + 2 < n) column(std::integral_constant<int, 2>{});
}

// The tensor-core part of chunk c (buffer b) for this warp's 128 rows: the
// accumulator's digit columns 0..4 collect H4 x (s_{j+k} + s_{j-k}), columns
// 5..7 collect R4 x s_{j+k} s_{j-k}.  Columns are grouped into runs of one
// mode (zones and row ranges are monotone in k: a chunk has few runs).
template <bool kCross>
__device__ __forceinline__ void cert_mma_chunk(const CertIO& io, const CertLane& ln, uint32_t c,
                                               uint32_t b, int (&acc)[kCertTiles][4],
                                               uint32_t& nmma) {
  const uint32_t kb = 1 + c * kChunk;
  if (!cert_mma_work(io, kb)) return;
#ifdef PSL_ABLATE_MMA
  return;
#endif
  const uint32_t w = threadIdx.x >> 5;
  // this warp's active rows (none: no MMAs)
  const int rw_lo = max(128 * (int)w, (int)io.r_lo), rw_hi = min(128 * (int)w + 127, (int)io.r_hi - 1);
  if (rw_lo > rw_hi) return;
  const long long jw_lo = (long long)io.j0 + rw_lo, jw_hi = (long long)io.j0 + rw_hi;
  const uint32_t fo = b * (uint32_t)kWinBuf, bo = b * (uint32_t)kLimbBuf;
  auto mode = [&](int cc) -> int {
    const uint32_t k0 = kb + 32 * cc, k1 = k0 + 31;
    if (k0 >= io.L) return 0;
    const bool lin = k0 <= io.m_lo || (k1 > io.m_hi && k0 <= io.M_hi);
    const bool fwd = lin && jw_lo + k0 < (long long)io.L;
    const bool rev = lin && (long long)k0 <= jw_hi;
    const bool crs = kCross && k0 <= io.m_lo;
    return (fwd ? 1 : 0) | (rev ? 2 : 0) | (crs ? 4 : 0);
  };
  // runs of equal mode: lane l < 16 evaluates column l, run starts by ballot
  const uint32_t lane = threadIdx.x & 31;
  const int my = mode((int)(lane & 15));
  const int prev = __shfl_up_sync(FULL, my, 1);
  uint32_t starts = __ballot_sync(FULL, lane < 16 && (lane == 0 || my != prev));
  while (starts) {
    const int cc = __ffs(starts) - 1;
    starts &= starts - 1;
    const int ce = starts ? __ffs(starts) - 1 : kCertCols;
    const int md = __shfl_sync(FULL, my, cc);
    const uint32_t f = ln.f + fo + 32 * cc, v = ln.v + fo + 32 * cc, bd = ln.bd + bo + 32 * cc;
    const int n = ce - cc;
    nmma += (uint32_t)(n * kCertTiles) * (uint32_t)((md & 1) + ((md >> 1) & 1) + ((md >> 2) & 1));
    switch (md) {
      case 1: cert_run<true, false, false>(f, v, bd, ln.dh, n, acc); break;
      case 2: cert_run<false, true, false>(f, v, bd, ln.dh, n, acc); break;
      case 3: cert_run<true, true, false>(f, v, bd, ln.dh, n, acc); break;
      case 7: if (kCross) cert_run<true, true, true>(f, v, bd, ln.dh, n, acc); break;
      case 5: if (kCross) cert_run<true, false, true>(f, v, bd, ln.dh, n, acc); break;
      case 6: if (kCross) cert_run<false, true, true>(f, v, bd, ln.dh, n, acc); break;
      case 4: if (kCross) cert_run<false, false, true>(f, v, bd, ln.dh, n, acc); break;
      default: break;
    }
  }
}

// Accumulator digits -> per-row doubles (rows 128w + 16r + g (+8)).  The quad
// holds digit columns 2 tig, 2 tig + 1: columns 0..4 are H4 digits (weight
// 256^d x 2^qH), 5..7 R4 digits (256^(d-5) x 2^qR).
__device__ __forceinline__ void cert_rows(const int (&acc)[kCertTiles][4], double unitH,
                                          double unitR, double* lrow, double* xrow) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tig = lane & 3;
  const int d0 = 2 * tig, d1 = 2 * tig + 1;
  const double w0 = d0 < kDigH ? ldexp(unitH, 8 * d0) : ldexp(unitR, 8 * (d0 - kDigH));
  const double w1 = d1 < kDigH ? ldexp(unitH, 8 * d1) : ldexp(unitR, 8 * (d1 - kDigH));
  const bool h0 = d0 < kDigH, h1 = d1 < kDigH;
#pragma unroll
  for (int r = 0; r < kCertTiles; ++r) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const double x0 = __dmul_rn((double)acc[r][2 * hh], w0);
      const double x1 = __dmul_rn((double)acc[r][2 * hh + 1], w1);
      double pl = __dadd_rn(h0 ? x0 : 0.0, h1 ? x1 : 0.0);
      double px = __dadd_rn(h0 ? 0.0 : x0, h1 ? 0.0 : x1);
      pl = __dadd_rn(pl, __shfl_xor_sync(FULL, pl, 1));
      px = __dadd_rn(px, __shfl_xor_sync(FULL, px, 1));
      pl = __dadd_rn(pl, __shfl_xor_sync(FULL, pl, 2));
      px = __dadd_rn(px, __shfl_xor_sync(FULL, px, 2));
      if (tig == 0) {
        const uint32_t rho = 128 * warp + 16 * r + gid + 8 * hh;
        lrow[rho] = pl;
        xrow[rho] = px;
      }
    }
  }
}

// Exact band-1 terms of chunk c for this thread's rows rho = 4t + m: per cell
// pow_int(|C_k - 2x|, alpha), x = s_j (s_{j-k} [k <= j] + s_{j+k} [j+k < L]).
__device__ __forceinline__ void cert_band_cells(const CertIO& io, const CertSmem& cs, uint32_t c,
                                                uint32_t b, const uint32_t* __restrict__ sb,
                                                double (&Bs)[kJ]) {
  const uint32_t kb = 1 + c * kChunk;
  const uint32_t ke = min(kb + kChunk - 1, io.L - 1);
  const int32_t* rec = cs.rec + (size_t)b * kChunk;
  const uint32_t L = io.L;
#ifdef PSL_ABLATE_BAND
  return;
#endif
  const double* __restrict__ lut = io.lut;
  {
    const uint32_t blo = max(kb, io.m_lo + 1);
    const uint32_t bhi = min(ke, io.m_hi);
    if (blo > bhi) return;
#pragma unroll
    for (int m = 0; m < kJ; ++m) {
      const uint32_t rho = 4 * threadIdx.x + m;
      if (rho < io.r_lo || rho >= io.r_hi) continue;
      const uint32_t j = (uint32_t)(io.j0 + (int32_t)rho);
      const uint32_t sjb = (sb[(j >> 5) + 1] >> (j & 31)) & 1u;
      double s = Bs[m];
#pragma unroll 1
      for (uint32_t k0 = blo; k0 <= bhi; k0 += 32) {
        // bit q: s_{j+k0+q} and s_{j-k0-q} (1 <-> -1; zero pads beyond the ends)
        const long long pB = (long long)j + k0, pA = (long long)j - k0 - 31;
        const long long wB = pB >> 5, wA = pA >> 5;
        const uint32_t Bw = __funnelshift_r(sb[wB + 1], sb[wB + 2], (uint32_t)(pB & 31));
        const uint32_t Aw = __brev(__funnelshift_r(sb[wA + 1], sb[wA + 2], (uint32_t)(pA & 31)));
        const uint32_t nq = min(32u, bhi - k0 + 1);
        for (uint32_t q = 0; q < nq; ++q) {
          const uint32_t k = k0 + q;
          const int u = ((Bw >> q) & 1u) == sjb ? 1 : -1;
          const int v = ((Aw >> q) & 1u) == sjb ? 1 : -1;
          const int x = (k <= j ? v : 0) + (j + k < L ? u : 0);
          s = __dadd_rn(s, __ldg(lut + abs(rec[k - kb] - 2 * x)));
        }
      }
      Bs[m] = s;
    }
  }
}

// Band 2 (k in (M_lo, M_hi]): row j's constant is sum_{k <= M_j} 4M_k +
// sum_{k > M_j} 4 e2_k.  Warp 0 turns b2M into inclusive prefix sums and b2E
// into inclusive suffix sums (32 serial terms per lane + a shuffle scan).
__device__ __forceinline__ void cert_band2_scan(const CertSmem& cs, uint32_t nb2) {
  if (threadIdx.x >= 32) return;
  const uint32_t lane = threadIdx.x;
  const uint32_t per = (nb2 + 31) / 32, lo = lane * per, hi = min(nb2, lo + per);
  double sm = 0.0, se = 0.0;
  for (uint32_t i = lo; i < hi; ++i) { sm = __dadd_rn(sm, cs.b2M[i]); cs.b2M[i] = sm; }
  for (uint32_t i = hi; i-- > lo;) { se = __dadd_rn(se, cs.b2E[i]); cs.b2E[i] = se; }
  double pm = sm, ps = se;   // inclusive scans over lanes (prefix for M, suffix for E)
  for (int o = 1; o < 32; o <<= 1) {
    const double a = __shfl_up_sync(FULL, pm, o), bb = __shfl_down_sync(FULL, ps, o);
    if ((int)lane >= o) pm = __dadd_rn(pm, a);
    if ((int)lane + o < 32) ps = __dadd_rn(ps, bb);
  }
  const double offm = __dsub_rn(pm, sm), offe = __dsub_rn(ps, se);   // exclusive carries
  for (uint32_t i = lo; i < hi; ++i) {
    cs.b2M[i] = __dadd_rn(cs.b2M[i], offm);
    cs.b2E[i] = __dadd_rn(cs.b2E[i], offe);
  }
}
__device__ __forceinline__ double cert_band2_const(const CertSmem& cs, uint32_t nb2, uint32_t i) {
  return __dadd_rn(i > 0 ? cs.b2M[i - 1] : 0.0, i < nb2 ? cs.b2E[i] : 0.0);
}

// gamma_n = n u / (1 - n u), u = 2^-53 (Higham)
__device__ __forceinline__ double gamma_n(double n) {
  const double u = 0x1p-53;
  return n * u / (1.0 - n * u);
}
