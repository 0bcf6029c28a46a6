// psl_api.cu -- the C ABI (include/pslb200.h): host logic above the kernels.
//
// Mirrors the reference's public surface (/root/reference/proj): parameter
// defaults and validation (search.cpp:19-94), pow_int (sequence.cpp:95-105),
// the ScanJob operator seam (search.cpp:156-175), neighborhood_scan
// (search.cpp:296-321), evaluate_neighbor (sequence.cpp:180-196),
// SidelobeTable::build (sequence.cpp:46-60), apply_flip
// (sequence.cpp:198-224) and run_search (search.cpp:327-430), with the same
// error classes (errors.hpp) mapped to status codes and the same messages.
// There is no CPU fallback: without a CUDA device every compute entry point
// returns PSL_ERR_CUDA.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "psl_internal.h"

using namespace pslb;

struct psl_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;   // warm-start uploads overlapped with the table builds
  uint32_t launches = 0;
  int scan_mode = PSL_SCAN_AUTO;
  uint64_t stats[5] = {0, 0, 0, 0, 0};
  int cert_check = 0;
  uint64_t chk[5] = {0, 0, 0, 0, 0};
  double chk_max[2] = {0.0, 0.0};
  // pinned staging of host-packed warm starts (grow-only) and the event after
  // its last upload (the next packing waits for it)
  uint32_t* pack_host = nullptr;
  size_t pack_cap = 0;
  cudaEvent_t pack_done = nullptr;
};

struct psl_walks {
  psl_ctx* ctx = nullptr;
  psl_params params{};
  uint32_t n_walks = 0;
  RunArgs a{};
  // device allocations
  WalkState* st = nullptr;
  int32_t* Cpiv = nullptr;
  int32_t* Cloc = nullptr;
  uint32_t* bits = nullptr;  // piv | loc | best | used, each n_walks * w_stride
  int2* hlist = nullptr;
  uint32_t* flips = nullptr;
  psl_event* events = nullptr;
  psl_trace* traces = nullptr;
  uint64_t* seeds = nullptr;
  uint32_t* packed = nullptr;   // device copy of the host-packed warm starts (setup only)
  int8_t* sol = nullptr;        // unpack scratch for solutions
  int8_t* sol_direct = nullptr; // host buffer the run kernel wrote the solutions into (psl_run_walks)
  double* lut = nullptr;        // [2][lut_n] power tables
  double* b2 = nullptr;         // certified-scan band-2 scratch
  double* lo_buf = nullptr;     // certified-scan per-row lower bounds (n_lmt > 1024)
  double* iv_buf = nullptr;     // certified-scan row intervals of a group
  uint64_t stats_read[5] = {0, 0, 0, 0, 0};   // scan statistics already added to ctx->stats
  uint64_t chk_read[5] = {0, 0, 0, 0, 0};     // ... certificate-check counts
};

namespace {

const char* kVersion = "0.1.0";  // version.hpp:5

void set_err(char* err, size_t errlen, const std::string& msg) {
  if (err && errlen) {
    std::strncpy(err, msg.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

int cuda_fail(char* err, size_t errlen, cudaError_t e, const char* what) {
  set_err(err, errlen, std::string(what) + ": " + cudaGetErrorString(e));
  return PSL_ERR_CUDA;
}

#define CK(call)                                                        \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) return cuda_fail(err, errlen, e_, #call);    \
  } while (0)

constexpr uint32_t kMinLength = 2;            // sequence.hpp:12
constexpr uint32_t kMaxLength = 1u << 20;     // sequence.hpp:13

std::string overflow_msg(bool neighbor, uint32_t L, uint32_t alpha) {
  // search.cpp:276-280 (neighbour) / sequence.cpp:11-15 (fitness)
  return std::string(neighbor ? "neighbor fitness is not finite at length "
                              : "fitness sum is not finite at length ") +
         std::to_string(L) + " with exponent " + std::to_string(alpha) +
         "; lower the exponent (alpha2, then alpha1) until |C_k|^alpha sums stay "
         "inside double range";
}

std::vector<uint32_t> pack_bits(const int8_t* s, uint32_t L, uint32_t pad) {
  const uint32_t nw = (L + 31) / 32;
  std::vector<uint32_t> b(nw + pad, 0u);
  for (uint32_t i = 0; i < L; ++i)
    if (s[i] < 0) b[i >> 5] |= 1u << (i & 31);
  return b;
}

int check_sequence(const int8_t* s, uint32_t L, char* err, size_t errlen) {
  // BinarySequence ctor (sequence.cpp:20-35)
  if (L < kMinLength || L > kMaxLength) {
    set_err(err, errlen, "sequence length " + std::to_string(L) + " out of supported range [" +
                             std::to_string(kMinLength) + ", " + std::to_string(kMaxLength) + "]");
    return PSL_ERR_CONFIG;
  }
  for (uint32_t i = 0; i < L; ++i) {
    if (s[i] != 1 && s[i] != -1) {
      set_err(err, errlen, "sequence element at position " + std::to_string(i) + " is " +
                               std::to_string((int)s[i]) + "; elements must be +1 or -1");
      return PSL_ERR_CONFIG;
    }
  }
  return PSL_OK;
}

int device_ready(psl_ctx* ctx, char* err, size_t errlen) {
  if (!ctx) { set_err(err, errlen, "null context"); return PSL_ERR_CUDA; }
  CK(cudaSetDevice(ctx->device));
  return PSL_OK;
}

// Stream-ordered device scratch for one C-ABI call: allocations come from the
// device's memory pool (kept across calls, psl_ctx_create), so a call costs no
// cudaMalloc / cudaFree round trip; freed in stream order when the call ends.
struct Scratch {
  cudaStream_t s;
  std::vector<void*> p;
  explicit Scratch(cudaStream_t st) : s(st) {}
  template <class T>
  cudaError_t get(T** out, size_t bytes) {
    void* q = nullptr;
    const cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(bytes, 16), s);
    if (e == cudaSuccess) { p.push_back(q); *out = static_cast<T*>(q); }
    return e;
  }
  ~Scratch() { for (void* q : p) cudaFreeAsync(q, s); }
};

// One walk's warm start -> nw bit words (bit = 1 <-> -1), validating every
// element as the BinarySequence ctor does (sequence.cpp:20-35).  Returns the first
// offending position + 1 (0 when valid) and its value in *badv.  8 elements per
// 64-bit word: (b + 1) mod 256 in {0x00, 0x02} <=> b in {+1, -1}; the sign bits
// are gathered by the 0x0102040810204080 multiply.
uint64_t pack_walk(const int8_t* s, uint32_t L, uint32_t* dst, int* badv) {
  const uint32_t full = L / 32;
  for (uint32_t i = 0; i < full; ++i) {
    uint32_t word = 0;
    uint64_t badm = 0;
    for (int q = 0; q < 4; ++q) {
      uint64_t v;
      std::memcpy(&v, s + 32 * (size_t)i + 8 * q, 8);
      const uint64_t inc = ((v & 0x7F7F7F7F7F7F7F7Full) + 0x0101010101010101ull) ^ (v & 0x8080808080808080ull);
      badm |= inc & 0xFDFDFDFDFDFDFDFDull;
      word |= (uint32_t)((((v >> 7) & 0x0101010101010101ull) * 0x0102040810204080ull) >> 56) << (8 * q);
    }
    if (badm) {
      for (uint32_t j = 0; j < 32; ++j) {
        const int8_t e = s[32 * (size_t)i + j];
        if (e != 1 && e != -1) { *badv = e; return 32ull * i + j + 1; }
      }
    }
    dst[i] = word;
  }
  if (full * 32 < L) {
    uint32_t word = 0;
    for (uint32_t j = full * 32; j < L; ++j) {
      const int8_t e = s[j];
      if (e != 1 && e != -1) { *badv = e; return (uint64_t)j + 1; }
      word |= (uint32_t)(e < 0) << (j & 31);
    }
    dst[full] = word;
  }
  return 0;
}

}  // namespace

extern "C" {

const char* psl_version(void) { return kVersion; }

int psl_ctx_create(int device, psl_ctx** out, char* err, size_t errlen) {
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_err(err, errlen, std::string("no CUDA device available (") +
                             (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") +
                             "); the B200 engine has no CPU fallback");
    return PSL_ERR_CUDA;
  }
  if (device < 0 || device >= n) {
    set_err(err, errlen, "device index " + std::to_string(device) + " out of range");
    return PSL_ERR_CUDA;
  }
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) {
    set_err(err, errlen, std::string("device ") + prop.name +
                             " is not sm_100 (Blackwell); this build targets sm_100a only");
    return PSL_ERR_CUDA;
  }
  psl_ctx* c = new psl_ctx;
  c->device = device;
  if (const char* env = std::getenv("PSLB200_SCAN"))
    c->scan_mode = std::string(env) == "exact" ? PSL_SCAN_EXACT : PSL_SCAN_AUTO;
  CK(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->stream = c->own;
  // keep freed walk buffers in the pool (no release back to the OS between calls)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return PSL_OK;
}

void psl_ctx_destroy(psl_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->pack_done) { cudaEventSynchronize(ctx->pack_done); cudaEventDestroy(ctx->pack_done); }
  if (ctx->pack_host) cudaFreeHost(ctx->pack_host);
  delete ctx;
}

int psl_ctx_set_stream(psl_ctx* ctx, void* stream) {
  if (!ctx) return PSL_ERR_CUDA;
  ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
  return PSL_OK;
}

void* psl_ctx_stream(psl_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

uint32_t psl_kernel_launches(psl_ctx* ctx) { return ctx ? ctx->launches : 0; }

int psl_ctx_set_scan_mode(psl_ctx* ctx, int mode) {
  if (!ctx || (mode != PSL_SCAN_AUTO && mode != PSL_SCAN_EXACT)) return PSL_ERR_CONFIG;
  ctx->scan_mode = mode;
  return PSL_OK;
}

int psl_ctx_scan_mode(psl_ctx* ctx) { return ctx ? ctx->scan_mode : -1; }

int psl_ctx_scan_stats(psl_ctx* ctx, uint64_t* certified, uint64_t* refined, uint64_t* chains,
                       uint64_t* mma, uint64_t* umma) {
  if (!ctx) return PSL_ERR_CONFIG;
  if (umma) *umma = ctx->stats[4];
  if (certified) *certified = ctx->stats[0];
  if (refined) *refined = ctx->stats[1];
  if (chains) *chains = ctx->stats[2];
  if (mma) *mma = ctx->stats[3];
  return PSL_OK;
}

int psl_ctx_set_cert_check(psl_ctx* ctx, int on) {
  if (!ctx) return PSL_ERR_CONFIG;
  ctx->cert_check = on ? 1 : 0;
  return PSL_OK;
}

int psl_ctx_cert_check_stats(psl_ctx* ctx, uint64_t counts[5], double maxima[2]) {
  if (!ctx) return PSL_ERR_CONFIG;
  for (int i = 0; i < 5; ++i) if (counts) counts[i] = ctx->chk[i];
  for (int i = 0; i < 2; ++i) if (maxima) maxima[i] = ctx->chk_max[i];
  return PSL_OK;
}

int psl_probe_umma(psl_ctx* ctx, double* mma_per_s, char* err, size_t errlen) {
  int rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
  const int n = probe_umma(nsm, ctx->stream, mma_per_s);
  if (n < 0) return cuda_fail(err, errlen, take_launch_error(), "probe_umma");
  ctx->launches += (uint32_t)n;
  return PSL_OK;
}

int psl_probe_imma(psl_ctx* ctx, double* mma_per_s, char* err, size_t errlen) {
  int rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
  const int n = probe_imma(nsm, ctx->stream, mma_per_s);
  if (n < 0) return cuda_fail(err, errlen, take_launch_error(), "probe_imma");
  ctx->launches += (uint32_t)n;
  return PSL_OK;
}

int psl_probe_peaks(psl_ctx* ctx, double* dadd_cells_per_s, double* lds_cells_per_s,
                    double* sm_mhz, char* err, size_t errlen) {
  int rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
  const int n = probe_peaks(nsm, ctx->stream, dadd_cells_per_s, lds_cells_per_s, sm_mhz);
  if (n < 0) return cuda_fail(err, errlen, take_launch_error(), "probe_peaks");
  ctx->launches += (uint32_t)n;
  return PSL_OK;
}

// ---------------------------------------------------------------- params

uint32_t psl_default_alpha2(uint32_t length) {
  if (length < (1u << 18) - 1) return 13;
  if (length < (1u << 19) - 1) return 11;
  return 10;
}
uint32_t psl_default_n_lmt(uint32_t length) { return std::min(length, 1024u); }
uint32_t psl_default_flip_lmt(uint32_t length) { return std::min(length, 10u); }

void psl_default_params(uint32_t length, psl_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->length = length;
  p->seed = 1;
  p->alpha1 = 4;
  p->alpha2 = psl_default_alpha2(length);
  p->ls_lmt = 2000;
  p->flip_lmt = psl_default_flip_lmt(length);
  p->n_lmt = psl_default_n_lmt(length);
  p->workers = 1;
}

int psl_validate_params(const psl_params* in, psl_params* out, char* warning, size_t warnlen,
                        char* err, size_t errlen) {
  psl_params p = *in;
  std::string warn;
  auto fail = [&](const std::string& m) { set_err(err, errlen, m); return PSL_ERR_CONFIG; };
  if (p.length < kMinLength || p.length > kMaxLength)
    return fail("length " + std::to_string(p.length) + " out of supported range [" +
                std::to_string(kMinLength) + ", " + std::to_string(kMaxLength) + "]");
  if (p.alpha1 < 1 || p.alpha2 < 1) return fail("fitness exponents alpha1/alpha2 must be >= 1");
  if (p.ls_lmt < 1) return fail("ls-lmt must be >= 1");
  if (p.flip_lmt < 1) return fail("flip-lmt must be >= 1");
  if (p.n_lmt < 1) return fail("n-lmt must be >= 1");
  if (p.workers < 1 || p.workers > 4096) return fail("workers must be in [1, 4096]");
  if (!p.has_max_nse && !p.has_max_seconds)
    return fail("a stop condition is required: max-nse and/or max-seconds");
  if (p.has_max_nse && p.max_nse < 1) return fail("max-nse must be >= 1");
  if (p.has_max_seconds && !(std::isfinite(p.max_seconds) && p.max_seconds > 0))
    return fail("max-seconds must be a positive finite number");
  if (p.init) {
    int rc = check_sequence(p.init, p.length, err, errlen);
    if (rc) return rc;
  }
  if (p.n_lmt > p.length) {
    warn += "n-lmt " + std::to_string(p.n_lmt) + " exceeds the " + std::to_string(p.length) +
            " distinct one-flip neighbors; clamped to the length\n";
    p.n_lmt = p.length;
  }
  if (p.flip_lmt > p.length) {
    warn += "flip-lmt " + std::to_string(p.flip_lmt) + " exceeds the length; clamped to " +
            std::to_string(p.length) + "\n";
    p.flip_lmt = p.length;
  }
  if (warning && warnlen) set_err(warning, warnlen, warn);
  if (out) *out = p;
  return PSL_OK;
}

double psl_pow_int(double base, uint32_t exp) {
  double result = 1.0, factor = base;
  uint32_t e = exp;
  while (e != 0) {
    if (e & 1u) result *= factor;
    e >>= 1;
    if (e != 0) factor *= factor;
  }
  return result;
}

// ---------------------------------------------------------------- scans

namespace {

// The sequence bits in the walks' padded layout (walks_create): nw + 48 zero
// words on both sides, because the sweep's sliding windows run past either end
// of the sequence unclamped.  Word i sits at [sb0 + 1 + i].
std::vector<uint32_t> padded_bits(const int8_t* seq, uint32_t L, size_t* sb0) {
  const size_t nw = (L + 31) / 32, front = nw + 48;
  std::vector<uint32_t> bits(front + nw + nw + 48 + kBitsPad, 0u);
  for (uint32_t i = 0; i < L; ++i)
    if (seq[i] < 0) bits[front + (i >> 5)] |= 1u << (i & 31);
  *sb0 = front - 1;
  return bits;
}

// values[1..n], psls[1..n] of the n neighbours (start+i)%L of one pivot.
int run_scan(psl_ctx* ctx, const int8_t* seq, const int32_t* table, uint32_t L, uint32_t start,
             uint32_t n, const double* lut, uint32_t lut_size, double* values, int32_t* psls,
             char* err, size_t errlen) {
  int rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  const uint32_t nw = (L + 31) / 32;
  size_t sb0 = 0;
  const std::vector<uint32_t> bits = padded_bits(seq, L, &sb0);
  cudaStream_t s = ctx->stream;
  Scratch d(s);
  ScanArgs a{};
  double* dv = nullptr;
  int32_t* dp = nullptr;
  uint32_t* db = nullptr;
  int32_t* dc = nullptr;
  double* dl = nullptr;
  CK(d.get(&db, bits.size() * 4));
  CK(d.get(&dc, (size_t)L * 4));
  CK(d.get(&dl, (size_t)lut_size * 8));
  CK(d.get(&a.hlist, (size_t)L * sizeof(int2)));
  CK(d.get(&a.P, 4));
  CK(d.get(&a.hcount, 4));
  CK(d.get(&dv, ((size_t)n + 1) * 8));
  CK(d.get(&dp, ((size_t)n + 1) * 4));
  CK(cudaMemcpyAsync(db, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dc, table, (size_t)L * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dl, lut, (size_t)lut_size * 8, cudaMemcpyHostToDevice, s));
  a.L = L; a.n = n; a.start = start; a.nwords = nw;
  a.nchunks = (L - 1 + kChunk - 1) / kChunk;
  a.lut_size = lut_size;
  a.bits = db + sb0; a.C = dc; a.lut = dl; a.values = dv; a.psls = dp;
  const int nl = launch_scan(a, s);
  if (nl < 0) return cuda_fail(err, errlen, take_launch_error(), "scan_kernel");
  ctx->launches += (uint32_t)nl;
  CK(cudaMemcpyAsync(values + 1, dv + 1, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(psls + 1, dp + 1, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return PSL_OK;
}

}  // namespace

int psl_scan(psl_ctx* ctx, const psl_scan_job* job, char* err, size_t errlen) {
  if (!job || !job->seq || !job->table || !job->lut || !job->values || !job->psls) {
    set_err(err, errlen, "psl_scan: null pointer in job");
    return PSL_ERR_CONFIG;
  }
  if (job->length < kMinLength || job->start >= job->length || job->n < 1 ||
      job->n > job->length) {
    set_err(err, errlen, "psl_scan: job out of range");
    return PSL_ERR_CONFIG;
  }
  // the reference's ScanJob reads PowerTable(L, alpha) (L + 1 entries,
  // search.cpp:337-338): any |C_k +- 4| <= L is a valid index
  if (job->lut_size < job->length + 1) {
    set_err(err, errlen, "power table too small for sequence length");
    return PSL_ERR_CONFIG;
  }
  return run_scan(ctx, job->seq, job->table, job->length, job->start, job->n, job->lut,
                  job->lut_size, job->values, job->psls, err, errlen);
}

int psl_neighborhood_scan(psl_ctx* ctx, const int8_t* seq, const int32_t* table,
                          const double* lut, uint32_t lut_size, uint32_t alpha, uint32_t L,
                          uint32_t start, uint32_t n, psl_scan_result* out, char* err,
                          size_t errlen) {
  int rc = check_sequence(seq, L, err, errlen);
  if (rc) return rc;
  // search.cpp:300-312
  if (start >= L) {
    set_err(err, errlen, "scan start position " + std::to_string(start) +
                             " out of range for length " + std::to_string(L));
    return PSL_ERR_CONFIG;
  }
  if (n < 1 || n > L) { set_err(err, errlen, "scan size must be in [1, length]"); return PSL_ERR_CONFIG; }
  if (lut_size < L + 1) { set_err(err, errlen, "power table too small for sequence length"); return PSL_ERR_CONFIG; }
  std::vector<double> values((size_t)n + 1);
  std::vector<int32_t> psls((size_t)n + 1);
  rc = run_scan(ctx, seq, table, L, start, n, lut, lut_size, values.data(), psls.data(), err, errlen);
  if (rc) return rc;
  // reduce_scan (search.cpp:271-292)
  uint32_t bi = 1, pi = 1;
  double v = values[1];
  int32_t pm = psls[1];
  for (uint32_t i = 1; i <= n; ++i) {
    if (!std::isfinite(values[i])) {
      set_err(err, errlen, overflow_msg(true, L, alpha));
      return PSL_ERR_OVERFLOW;
    }
    if (values[i] < v) { v = values[i]; bi = i; }
    if (psls[i] < pm) { pm = psls[i]; pi = i; }
  }
  out->best_index = (uint32_t)(((uint64_t)start + bi) % L);
  out->value_step = v;
  out->best_neighbor_psl = pm;
  out->best_psl_index = (uint32_t)(((uint64_t)start + pi) % L);
  return PSL_OK;
}

int psl_evaluate_neighbor(psl_ctx* ctx, const int8_t* seq, const int32_t* table,
                          const double* lut, uint32_t lut_size, uint32_t alpha, uint32_t L,
                          uint32_t j, double* fitness, int32_t* psl, char* err, size_t errlen) {
  int rc = check_sequence(seq, L, err, errlen);
  if (rc) return rc;
  // sequence.cpp:182-192
  if (j >= L) {
    set_err(err, errlen, "neighbor position " + std::to_string(j) + " out of range for length " +
                             std::to_string(L));
    return PSL_ERR_CONFIG;
  }
  if (lut_size < L + 1) { set_err(err, errlen, "power table too small for sequence length"); return PSL_ERR_CONFIG; }
  double values[2];
  int32_t psls[2];
  rc = run_scan(ctx, seq, table, L, (j + L - 1) % L, 1, lut, lut_size, values, psls, err, errlen);
  if (rc) return rc;
  if (!std::isfinite(values[1])) {
    set_err(err, errlen, overflow_msg(false, L, alpha));
    return PSL_ERR_OVERFLOW;
  }
  *fitness = values[1];
  *psl = psls[1];
  return PSL_OK;
}

int psl_build_table(psl_ctx* ctx, const int8_t* seq, uint32_t L, int32_t* table_out, char* err,
                    size_t errlen) {
  int rc = check_sequence(seq, L, err, errlen);
  if (rc) return rc;
  rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  const uint32_t nw = (L + 31) / 32;
  const std::vector<uint32_t> bits = pack_bits(seq, L, kBitsPad);
  cudaStream_t s = ctx->stream;
  Scratch d(s);
  uint32_t* db = nullptr;
  int32_t* dc = nullptr;
  CK(d.get(&db, bits.size() * 4));
  CK(d.get(&dc, (size_t)L * 4));
  CK(cudaMemcpyAsync(db, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, s));
  if (launch_table_only(db, dc, L, nw, s) < 0)
    return cuda_fail(err, errlen, take_launch_error(), "build_tables_kernel");
  ctx->launches += 1;
  CK(cudaMemcpyAsync(table_out, dc, (size_t)L * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return PSL_OK;
}

int psl_verify_sequence(psl_ctx* ctx, const int8_t* seq, uint32_t L, int32_t* psl,
                        double* merit_factor, int64_t* energy, uint64_t* histogram,
                        uint32_t hist_cap, char* err, size_t errlen) {
  int rc = check_sequence(seq, L, err, errlen);
  if (rc) return rc;
  rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  const uint32_t nw = (L + 31) / 32;
  std::vector<uint32_t> bits = pack_bits(seq, L, kBitsPad);
  cudaStream_t s = ctx->stream;
  uint32_t* db = nullptr;
  int32_t* dc = nullptr;
  int32_t* dpsl = nullptr;
  unsigned long long* den = nullptr;
  unsigned long long* dh = nullptr;
  CK(cudaMallocAsync(&db, bits.size() * 4, s));
  CK(cudaMallocAsync(&dc, (size_t)L * 4, s));
  CK(cudaMallocAsync(&dpsl, 4, s));
  CK(cudaMallocAsync(&den, 8, s));
  CK(cudaMallocAsync(&dh, ((size_t)L + 1) * 8, s));
  CK(cudaMemcpyAsync(db, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(dpsl, 0, 4, s));
  CK(cudaMemsetAsync(den, 0, 8, s));
  CK(cudaMemsetAsync(dh, 0, ((size_t)L + 1) * 8, s));
  if (launch_table_only(db, dc, L, nw, s) < 0 || launch_verify(dc, L, dpsl, den, dh, s) < 0)
    return cuda_fail(err, errlen, take_launch_error(), "verify");
  ctx->launches += 2;
  int32_t hpsl = 0;
  unsigned long long hen = 0;
  CK(cudaMemcpyAsync(&hpsl, dpsl, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&hen, den, 8, cudaMemcpyDeviceToHost, s));
  if (histogram && hist_cap)
    CK(cudaMemcpyAsync(histogram, dh, std::min<size_t>(hist_cap, (size_t)L + 1) * 8,
                       cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (void* p : {(void*)db, (void*)dc, (void*)dpsl, (void*)den, (void*)dh}) cudaFreeAsync(p, s);
  *psl = hpsl;
  if (energy) *energy = (int64_t)hen;
  if (merit_factor) *merit_factor = ((double)L * (double)L) / (2.0 * (double)(int64_t)hen);
  return PSL_OK;
}

int psl_apply_flip(psl_ctx* ctx, int8_t* seq, int32_t* table, uint32_t L, uint32_t j, char* err,
                   size_t errlen) {
  int rc = check_sequence(seq, L, err, errlen);
  if (rc) return rc;
  if (j >= L) {
    set_err(err, errlen, "flip position " + std::to_string(j) + " out of range for length " +
                             std::to_string(L));
    return PSL_ERR_CONFIG;
  }
  rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  const std::vector<uint32_t> bits = pack_bits(seq, L, kBitsPad);
  cudaStream_t s = ctx->stream;
  Scratch d(s);
  uint32_t* db = nullptr;
  int32_t* dc = nullptr;
  CK(d.get(&db, bits.size() * 4));
  CK(d.get(&dc, (size_t)L * 4));
  CK(cudaMemcpyAsync(db, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dc, table, (size_t)L * 4, cudaMemcpyHostToDevice, s));
  if (launch_apply_flip(db, dc, L, j, s) < 0)
    return cuda_fail(err, errlen, take_launch_error(), "apply_flip_kernel");
  ctx->launches += 2;
  CK(cudaMemcpyAsync(table, dc, (size_t)L * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  seq[j] = (int8_t)-seq[j];
  return PSL_OK;
}

int psl_flip_deltas(psl_ctx* ctx, const int8_t* seq, uint32_t L, uint32_t j, int32_t* out, char* err,
                    size_t errlen) {
  int rc = check_sequence(seq, L, err, errlen);
  if (rc) return rc;
  if (!out) { set_err(err, errlen, "flip_deltas: null output"); return PSL_ERR_CONFIG; }
  if (j >= L) {   // sequence.cpp:156-160
    set_err(err, errlen, "flip position " + std::to_string(j) + " out of range for length " +
                             std::to_string(L));
    return PSL_ERR_CONFIG;
  }
  rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  const std::vector<uint32_t> bits = pack_bits(seq, L, kBitsPad);
  cudaStream_t s = ctx->stream;
  Scratch d(s);
  uint32_t* db = nullptr;
  int32_t* dout = nullptr;
  CK(d.get(&db, bits.size() * 4));
  CK(d.get(&dout, (size_t)L * 4));
  CK(cudaMemcpyAsync(db, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, s));
  if (launch_flip_deltas(db, L, j, dout, s) < 0)
    return cuda_fail(err, errlen, take_launch_error(), "flip_deltas_kernel");
  ctx->launches += 1;
  CK(cudaMemcpyAsync(out, dout, (size_t)L * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return PSL_OK;
}

int psl_fitness(psl_ctx* ctx, const int32_t* table, uint32_t L, const double* lut, uint32_t lut_size,
                uint32_t alpha, double* fitness, char* err, size_t errlen) {
  if (!table || !lut || !fitness) { set_err(err, errlen, "fitness: null pointer"); return PSL_ERR_CONFIG; }
  if (L < 1) { set_err(err, errlen, "fitness: empty table"); return PSL_ERR_CONFIG; }
  int32_t amax = 0;
  for (uint32_t k = 1; k < L; ++k) amax = std::max(amax, std::abs(table[k]));
  if ((uint64_t)lut_size <= (uint64_t)amax) {
    set_err(err, errlen, "power table too small for the table's sidelobes");
    return PSL_ERR_CONFIG;
  }
  int rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  cudaStream_t s = ctx->stream;
  Scratch d(s);
  int32_t* dc = nullptr;
  double* dl = nullptr;
  double* dout = nullptr;
  CK(d.get(&dc, (size_t)L * 4));
  CK(d.get(&dl, (size_t)lut_size * 8));
  CK(d.get(&dout, 8));
  CK(cudaMemcpyAsync(dc, table, (size_t)L * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dl, lut, (size_t)lut_size * 8, cudaMemcpyHostToDevice, s));
  if (launch_fitness_chain(dc, L, dl, dout, s) < 0)
    return cuda_fail(err, errlen, take_launch_error(), "fitness_chain_kernel");
  ctx->launches += 1;
  double v = 0.0;
  CK(cudaMemcpyAsync(&v, dout, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (!std::isfinite(v)) {   // sequence.cpp:139
    set_err(err, errlen, overflow_msg(false, L, alpha));
    return PSL_ERR_OVERFLOW;
  }
  *fitness = v;
  return PSL_OK;
}

// ---------------------------------------------------------------- walks

void psl_walks_destroy(psl_walks* w) {
  if (!w) return;
  cudaSetDevice(w->ctx->device);
  cudaStream_t s = w->ctx->stream;
  for (void* p : {(void*)w->st, (void*)w->Cpiv, (void*)w->Cloc, (void*)w->bits, (void*)w->hlist,
                  (void*)w->flips, (void*)w->events, (void*)w->traces, (void*)w->seeds,
                  (void*)w->packed, (void*)w->sol, (void*)w->lut, (void*)w->b2,
                  (void*)w->lo_buf, (void*)w->iv_buf})
    if (p) cudaFreeAsync(p, s);
  delete w;
}

namespace {

int walks_create(psl_ctx* ctx, const psl_params* params, uint32_t n_walks, const uint64_t* seeds,
                 const int8_t* inits, uint64_t events_cap, uint64_t traces_cap, psl_walks** out,
                 char* err, size_t errlen) {
  *out = nullptr;
  psl_params p;
  int rc = psl_validate_params(params, &p, nullptr, 0, err, errlen);
  if (rc) return rc;
  if (n_walks < 1) { set_err(err, errlen, "n_walks must be >= 1"); return PSL_ERR_CONFIG; }
  rc = device_ready(ctx, err, errlen);
  if (rc) return rc;
  psl_walks* W = new psl_walks;
  W->ctx = ctx;
  W->params = p;
  W->n_walks = n_walks;
  const uint32_t L = p.length;
  const uint32_t nw = (L + 31) / 32;
  RunArgs& a = W->a;
  a.L = L; a.n = p.n_lmt; a.alpha1 = p.alpha1; a.alpha2 = p.alpha2;
  a.ls_lmt = p.ls_lmt; a.flip_lmt = p.flip_lmt;
  a.nwords = nw;
  a.nchunks = (L - 1 + kChunk - 1) / kChunk;
  a.has_max_nse = p.has_max_nse; a.max_nse = p.max_nse;
  a.has_max_seconds = p.has_max_seconds; a.max_seconds = p.max_seconds;
  a.step_budget = 0xffffffffu;
  a.record_events = events_cap > 0;
  a.record_traces = traces_cap > 0;
  a.cert = ctx->scan_mode == PSL_SCAN_AUTO && !a.record_traces;
  a.cert_slack = 0.0;
  if (const char* env = std::getenv("PSLB200_CERT_SLACK")) a.cert_slack = std::max(0.0, std::atof(env));
  a.events_cap = events_cap;
  a.traces_cap = traces_cap;
  a.c_stride = ((size_t)L + 31) & ~size_t(31);
  // per-walk bit regions: nw+48 zero words in front and behind the sequence, so
  // the scan's sliding windows never need bounds clamps
  a.w_front = (size_t)nw + 48 - 1;
  a.w_stride = ((size_t)nw + 48 + nw + (size_t)nw + 48 + kBitsPad + 3) & ~size_t(3);
  a.h_stride = L;
  a.f_stride = std::max<uint32_t>(p.flip_lmt, 1);
  cudaStream_t s = ctx->stream;
  auto fail = [&](cudaError_t e, const char* what) {
    psl_walks_destroy(W);
    return cuda_fail(err, errlen, e, what);
  };
  cudaError_t e;
  // stream-ordered allocations from the device's default pool: repeated
  // psl_run_walks calls reuse the memory instead of re-mapping gigabytes
#define AL(ptr, bytes) \
  if ((e = cudaMallocAsync(&(ptr), (bytes), s)) != cudaSuccess) return fail(e, "cudaMallocAsync " #ptr);
  AL(W->st, sizeof(WalkState) * n_walks);
  AL(W->Cpiv, a.c_stride * 4 * n_walks);
  AL(W->Cloc, a.c_stride * 4 * n_walks);
  AL(W->bits, a.w_stride * 4 * n_walks * 4);
  AL(W->hlist, a.h_stride * sizeof(int2) * n_walks);
  AL(W->flips, a.f_stride * 4 * n_walks);
  AL(W->seeds, 8ull * n_walks);
  if (events_cap) AL(W->events, sizeof(psl_event) * events_cap * n_walks);
  if (traces_cap) AL(W->traces, sizeof(psl_trace) * traces_cap * n_walks);
  a.lut_n = L + 8;
  AL(W->lut, 2ull * a.lut_n * sizeof(double));
  a.lut1 = W->lut; a.lut2 = W->lut + a.lut_n;
  AL(W->b2, 2ull * kGroup * sizeof(double) * n_walks);
  a.b2 = W->b2;
  AL(W->lo_buf, (size_t)p.n_lmt * sizeof(double) * n_walks);
  a.lo_buf = W->lo_buf;
  AL(W->iv_buf, 3ull * kGroup * sizeof(double) * n_walks);
  a.iv_buf = W->iv_buf;
  a.st = W->st; a.Cpiv = W->Cpiv; a.Cloc = W->Cloc;
  a.bits_piv = W->bits;
  a.bits_loc = W->bits + a.w_stride * n_walks;
  a.bits_best = W->bits + 2 * a.w_stride * n_walks;
  a.used = W->bits + 3 * a.w_stride * n_walks;
  a.hlist = W->hlist; a.flips = W->flips; a.events = W->events; a.traces = W->traces;
  std::vector<uint64_t> sd(n_walks);
  for (uint32_t w = 0; w < n_walks; ++w) sd[w] = seeds ? seeds[w] : p.seed + w;
  if ((e = cudaMemcpyAsync(W->seeds, sd.data(), 8ull * n_walks, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return fail(e, "seeds");
  // Warm starts are validated and bit-packed on the host (8x fewer PCIe bytes
  // than the int8 elements), by all host threads, walk by walk in order; a batch
  // of packed walks is uploaded on the copy stream as soon as it is complete, and
  // its validation / table build runs while the next batch is still being packed.
  const bool shared_init = !inits && p.init;
  const uint32_t nbatch = (inits && L >= 8192 && n_walks >= 32) ? 4u : 1u;
  if (inits || p.init) {
    const size_t words = (shared_init ? 1 : (size_t)n_walks) * nw;
    if (ctx->pack_done) cudaEventSynchronize(ctx->pack_done);   // staging free again
    else if ((e = cudaEventCreateWithFlags(&ctx->pack_done, cudaEventDisableTiming)) != cudaSuccess)
      return fail(e, "event");
    if (ctx->pack_cap < words) {
      if (ctx->pack_host) cudaFreeHost(ctx->pack_host);
      ctx->pack_host = nullptr;
      ctx->pack_cap = 0;
      if ((e = cudaHostAlloc(&ctx->pack_host, words * 4, cudaHostAllocPortable)) != cudaSuccess)
        return fail(e, "pinned staging");
      ctx->pack_cap = words;
    }
    AL(W->packed, words * 4);
    if (nbatch > 1 && !ctx->copy &&
        (e = cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking)) != cudaSuccess)
      return fail(e, "copy stream");
  }
#undef AL
  if (launch_power_tables(W->lut, a.lut_n, p.alpha1, p.alpha2, s) < 0)
    return fail(take_launch_error(), "power_tables_kernel");
  ctx->launches += 1;
  // host packing: walks claimed in order by the worker threads; done[b] counts the
  // packed walks of batch b; the first invalid element over all walks is reported
  std::atomic<uint32_t> next{0};
  std::vector<std::atomic<uint32_t>> done(nbatch);
  for (auto& d : done) d.store(0);
  std::atomic<uint64_t> bad_flat{UINT64_MAX};
  int bad_val = 0;
  std::mutex bad_mu;
  const uint32_t n_pack = shared_init ? 0u : (inits ? n_walks : 0u);
  // batch boundaries: a small first batch (1/16 of the walks) so the first
  // table builds start after little packing; the GPU is the slower stage after it
  auto bound = [&](uint32_t b) -> uint32_t {
    static const uint32_t num[5] = {0, 1, 4, 8, 16};
    return nbatch == 4 ? (uint32_t)((uint64_t)n_walks * num[b] / 16) : (uint32_t)((uint64_t)n_walks * b / nbatch);
  };
  auto batch_of = [&](uint32_t w) {
    uint32_t b = 0;
    while (b + 1 < nbatch && w >= bound(b + 1)) ++b;
    return b;
  };
  auto worker = [&]() {
    for (;;) {
      const uint32_t w = next.fetch_add(1);
      if (w >= n_pack) return;
      int bv = 0;
      const uint64_t b = pack_walk(inits + (size_t)w * L, L, ctx->pack_host + (size_t)w * nw, &bv);
      if (b) {
        const uint64_t flat = (uint64_t)w * L + b - 1;
        std::lock_guard<std::mutex> lk(bad_mu);
        if (flat < bad_flat.load()) { bad_flat.store(flat); bad_val = bv; }
      }
      done[batch_of(w)].fetch_add(1);
    }
  };
  std::vector<std::thread> pool;
  if (shared_init) {
    int bv = 0;
    pack_walk(p.init, L, ctx->pack_host, &bv);              // validated by psl_validate_params
  } else if (n_pack) {
    const uint32_t hw = std::max(1u, std::thread::hardware_concurrency());
    const uint32_t nt = ((size_t)n_pack * L < (1u << 20)) ? 0u : std::min({hw, 16u, n_pack});
    for (uint32_t i = 0; i < nt; ++i) pool.emplace_back(worker);
    if (nt == 0) worker();
  }
  auto join_pool = [&]() { for (auto& th : pool) if (th.joinable()) th.join(); };
  for (uint32_t bi = 0; bi < nbatch; ++bi) {
    const uint32_t w0 = bound(bi);
    const uint32_t cnt = bound(bi + 1) - w0;
    const uint32_t* dpacked = nullptr;
    size_t pstride = 0;
    if (n_pack) {
      while (done[bi].load() < cnt) std::this_thread::yield();
      if (bad_flat.load() != UINT64_MAX) break;                // reported below
      cudaStream_t cs_ = nbatch > 1 ? ctx->copy : s;
      if (nbatch > 1) {
        cudaEvent_t ready;
        if ((e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming)) != cudaSuccess) {
          join_pool();
          return fail(e, "event");
        }
        cudaEventRecord(ready, s);                           // W->packed is stream-ordered on s
        cudaStreamWaitEvent(cs_, ready, 0);
        cudaEventDestroy(ready);
      }
      if ((e = cudaMemcpyAsync(W->packed + (size_t)w0 * nw, ctx->pack_host + (size_t)w0 * nw,
                               (size_t)cnt * nw * 4, cudaMemcpyHostToDevice, cs_)) != cudaSuccess) {
        join_pool();
        return fail(e, "warm starts");
      }
      if (nbatch > 1) {
        cudaEvent_t landed;
        if ((e = cudaEventCreateWithFlags(&landed, cudaEventDisableTiming)) != cudaSuccess) {
          join_pool();
          return fail(e, "event");
        }
        cudaEventRecord(landed, cs_);
        cudaStreamWaitEvent(s, landed, 0);
        cudaEventDestroy(landed);
      }
      dpacked = W->packed + (size_t)w0 * nw;
      pstride = nw;
    } else if (shared_init) {
      if (bi == 0 && (e = cudaMemcpyAsync(W->packed, ctx->pack_host, (size_t)nw * 4,
                                          cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return fail(e, "warm start");
      dpacked = W->packed;
      pstride = 0;
    }
    const RunArgs ab = walk_offset(a, w0);
    const int ni = launch_init_walks(ab, cnt, W->seeds + w0, dpacked, pstride, s);
    if (ni < 0) { join_pool(); return fail(take_launch_error(), "init_walks_kernel"); }
    // SidelobeTable::build: exact NTT correlation for long sequences (O(L log L)),
    // bit-parallel popcount kernel (O(L^2/32)) for short ones
    const int nb = L >= 8192 ? launch_build_tables_ntt(ab, cnt, s) : launch_build_tables(ab, cnt, s);
    if (nb < 0) { join_pool(); return fail(take_launch_error(), "build_tables"); }
    ctx->launches += (uint32_t)ni + (uint32_t)nb;
  }
  join_pool();
  if (n_pack && bad_flat.load() != UINT64_MAX) {
    const uint64_t flat = bad_flat.load();
    cudaStreamSynchronize(s);
    psl_walks_destroy(W);
    set_err(err, errlen, "sequence element at position " + std::to_string(flat % L) + " is " +
                             std::to_string(bad_val) + "; elements must be +1 or -1");
    return PSL_ERR_CONFIG;
  }
  if (W->packed) {
    cudaEventRecord(ctx->pack_done, nbatch > 1 ? ctx->copy : s);   // staging reusable after this
    cudaFreeAsync(W->packed, s);
    W->packed = nullptr;
  }
  *out = W;
  return PSL_OK;
}

int walks_launch(psl_walks* W, uint32_t steps, char* err, size_t errlen) {
  RunArgs a = W->a;
  a.step_budget = steps;
  a.cert_check = W->ctx->cert_check;
  if (launch_run(a, W->n_walks, W->ctx->stream) < 0)
    return cuda_fail(err, errlen, take_launch_error(), "run_kernel");
  W->ctx->launches += 1;
  return PSL_OK;
}

}  // namespace

int psl_walks_create(psl_ctx* ctx, const psl_params* params, uint32_t n_walks,
                     const uint64_t* seeds, const int8_t* inits, psl_walks** out, char* err,
                     size_t errlen) {
  return walks_create(ctx, params, n_walks, seeds, inits, 0, 0, out, err, errlen);
}

int psl_walks_step(psl_walks* w, uint32_t steps, char* err, size_t errlen) {
  if (!w) return PSL_ERR_CONFIG;
  int rc = device_ready(w->ctx, err, errlen);
  if (rc) return rc;
  return walks_launch(w, steps, err, errlen);
}

int psl_walks_run(psl_walks* w, char* err, size_t errlen) {
  return psl_walks_step(w, 0xffffffffu, err, errlen);
}

int psl_walks_records(psl_walks* w, psl_walk_record* records, int8_t* solutions, char* err,
                      size_t errlen) {
  if (!w) return PSL_ERR_CONFIG;
  int rc = device_ready(w->ctx, err, errlen);
  if (rc) return rc;
  cudaStream_t s = w->ctx->stream;
  std::vector<WalkState> st(w->n_walks);
  CK(cudaMemcpyAsync(st.data(), w->st, sizeof(WalkState) * w->n_walks, cudaMemcpyDeviceToHost, s));
  const uint32_t L = w->a.L;
  bool direct = false;
  if (solutions && w->sol_direct == solutions) {
    // written by the run kernel as each walk stopped -- valid if every walk stopped cleanly
    CK(cudaStreamSynchronize(s));
    direct = true;
    for (const WalkState& S : st) direct = direct && S.done && S.status == PSL_OK;
  }
  if (solutions && !direct) {
    // unpack on the device, one D2H of n_walks * L int8
    if (!w->sol) CK(cudaMallocAsync(&w->sol, (size_t)w->n_walks * L, s));
    if (launch_unpack(w->a.bits_best + w->a.w_front + 1, w->a.w_stride, L, w->n_walks, w->sol, s) < 0)
      return cuda_fail(err, errlen, take_launch_error(), "unpack_kernel");
    w->ctx->launches += 1;
    CK(cudaMemcpyAsync(solutions, w->sol, (size_t)w->n_walks * L, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  for (uint32_t i = 0; i < w->n_walks; ++i) {
    const WalkState& S = st[i];
    psl_walk_record& r = records[i];
    r.seed = S.seed;
    r.nse = S.nse;
    const uint64_t end = S.end_ns ? S.end_ns : S.t0_ns;
    r.elapsed_seconds = S.t0_ns ? (double)(end - S.t0_ns) * 1e-9 : 0.0;
    r.psl_best = S.psl_best < 0 ? S.P : S.psl_best;
    r.status = S.status;
    r.energy = S.energy_best;
    r.merit_factor = ((double)L * (double)L) / (2.0 * (double)S.energy_best);
    r.switches = S.switches;
    r.steps = S.steps;
  }
  uint64_t tot[5] = {0, 0, 0, 0, 0};
  for (const WalkState& S : st) {
    tot[0] += S.n_cert; tot[1] += S.n_refine; tot[2] += S.n_vlchain; tot[3] += S.n_mma;
    tot[4] += S.n_umma;
  }
  for (int i = 0; i < 5; ++i) {
    w->ctx->stats[i] += tot[i] - w->stats_read[i];
    w->stats_read[i] = tot[i];
  }
  uint64_t chk[5] = {0, 0, 0, 0, 0};
  for (const WalkState& S : st) {
    chk[0] += S.chk_steps; chk[1] += S.chk_rows; chk[2] += S.chk_viol; chk[3] += S.chk_dec;
    chk[4] += S.chk_dec_bad;
    w->ctx->chk_max[0] = std::max(w->ctx->chk_max[0], S.chk_tight);
    w->ctx->chk_max[1] = std::max(w->ctx->chk_max[1], S.chk_relw);
  }
  for (int i = 0; i < 5; ++i) {
    w->ctx->chk[i] += chk[i] - w->chk_read[i];
    w->chk_read[i] = chk[i];
  }
  return PSL_OK;
}

int psl_run_walks(psl_ctx* ctx, const psl_params* params, uint32_t n_walks, const uint64_t* seeds,
                  const int8_t* inits, psl_walk_record* records, int8_t* solutions, char* err,
                  size_t errlen) {
  psl_walks* w = nullptr;
  int rc = psl_walks_create(ctx, params, n_walks, seeds, inits, &w, err, errlen);
  if (rc) return rc;
  if (solutions) {
    // a pinned (mapped) caller buffer: each walk's kernel writes its best
    // sequence there when it stops, overlapping the D2H with later walks' steps
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, solutions) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer) {
      w->a.sol_out = static_cast<int8_t*>(pa.devicePointer);
      w->sol_direct = solutions;
    }
    cudaGetLastError();
  }
  rc = psl_walks_run(w, err, errlen);
  if (!rc) rc = psl_walks_records(w, records, solutions, err, errlen);
  psl_walks_destroy(w);
  return rc;
}

int psl_run_walks_multi(const int* devices, uint32_t n_devices, const psl_params* params,
                        uint32_t n_walks, const uint64_t* seeds, const int8_t* inits,
                        psl_walk_record* records, int8_t* solutions, uint32_t* best_walk,
                        double* device_seconds, char* err, size_t errlen) {
  if (!devices || n_devices < 1) { set_err(err, errlen, "at least one device is required"); return PSL_ERR_CONFIG; }
  if (!params || !records) { set_err(err, errlen, "null params or records"); return PSL_ERR_CONFIG; }
  psl_params p;
  int rc = psl_validate_params(params, &p, nullptr, 0, err, errlen);
  if (rc) return rc;
  if (n_walks < n_devices) {
    set_err(err, errlen, "n_walks (" + std::to_string(n_walks) + ") must be >= the number of devices (" +
                             std::to_string(n_devices) + ")");
    return PSL_ERR_CONFIG;
  }
  const uint32_t L = p.length;
  std::vector<uint64_t> sd(n_walks);
  for (uint32_t w = 0; w < n_walks; ++w) sd[w] = seeds ? seeds[w] : p.seed + w;
  struct Part {
    int rc = PSL_OK;
    std::string err;
    double seconds = 0.0;
  };
  std::vector<Part> parts(n_devices);
  auto run_part = [&](uint32_t d) {
    Part& pt = parts[d];
    const uint32_t w0 = (uint32_t)((uint64_t)n_walks * d / n_devices);
    const uint32_t w1 = (uint32_t)((uint64_t)n_walks * (d + 1) / n_devices);
    char e[1024] = {0};
    const auto t0 = std::chrono::steady_clock::now();
    psl_ctx* ctx = nullptr;
    pt.rc = psl_ctx_create(devices[d], &ctx, e, sizeof e);
    if (pt.rc == PSL_OK) {
      pt.rc = psl_run_walks(ctx, &p, w1 - w0, sd.data() + w0, inits ? inits + (size_t)w0 * L : nullptr,
                            records + w0, solutions ? solutions + (size_t)w0 * L : nullptr, e, sizeof e);
      psl_ctx_destroy(ctx);
    }
    pt.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (pt.rc != PSL_OK)
      pt.err = "device " + std::to_string(devices[d]) + ": " + e;
  };
  if (n_devices == 1) {
    run_part(0);
  } else {
    std::vector<std::thread> th;
    th.reserve(n_devices);
    for (uint32_t d = 0; d < n_devices; ++d) th.emplace_back(run_part, d);
    for (auto& t : th) t.join();
  }
  for (uint32_t d = 0; d < n_devices; ++d) {
    if (device_seconds) device_seconds[d] = parts[d].seconds;
    if (parts[d].rc != PSL_OK) {
      set_err(err, errlen, parts[d].err);
      return parts[d].rc;
    }
  }
  if (best_walk) {
    uint64_t best = UINT64_MAX;
    for (uint32_t w = 0; w < n_walks; ++w) {
      if (records[w].status != PSL_OK) continue;
      const uint64_t key = ((uint64_t)(uint32_t)records[w].psl_best << 32) | w;
      best = std::min(best, key);
    }
    *best_walk = best == UINT64_MAX ? UINT32_MAX : (uint32_t)(best & 0xffffffffu);
  }
  return PSL_OK;
}

// ---------------------------------------------------------------- run_search

int psl_run_search(psl_ctx* ctx, const psl_params* params, const psl_hooks* hooks,
                   psl_run_record* out, int8_t* solution_best, char* err, size_t errlen) {
  const bool want_traces = hooks && hooks->on_scan;
  // device event/trace buffer capacity per drain (PSLB200_DRAIN_CAP overrides,
  // used by the tests to force many drain/resume cycles)
  uint64_t cap = 1u << 16;
  if (const char* env = std::getenv("PSLB200_DRAIN_CAP")) cap = std::max<uint64_t>(2, std::strtoull(env, nullptr, 10));
  const uint64_t ecap = cap, tcap = want_traces ? cap : 0;
  psl_walks* W = nullptr;
  int rc = walks_create(ctx, params, 1, nullptr, nullptr, ecap, tcap, &W, err, errlen);
  if (rc) return rc;
  cudaStream_t s = ctx->stream;
  std::vector<psl_event> ev;
  std::vector<psl_trace> tr;
  uint64_t n_ev = 0, n_tr = 0;
  WalkState S{};
  for (;;) {
    rc = walks_launch(W, 0xffffffffu, err, errlen);
    if (rc) break;
    cudaError_t e = cudaMemcpyAsync(&S, W->st, sizeof(S), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { rc = cuda_fail(err, errlen, e, "run_search"); break; }
    // drain (all buffered entries are final when the kernel returns)
    ev.resize(S.n_events);
    tr.resize(S.n_traces);
    if (S.n_events)
      e = cudaMemcpyAsync(ev.data(), W->events, sizeof(psl_event) * S.n_events, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && S.n_traces)
      e = cudaMemcpyAsync(tr.data(), W->traces, sizeof(psl_trace) * S.n_traces, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { rc = cuda_fail(err, errlen, e, "drain"); break; }
    // hooks fire in event order; traces after the events of the same step are
    // interleaved by nse (an event never has a larger nse than its step's trace)
    size_t ie = 0, it = 0;
    while (ie < ev.size() || it < tr.size()) {
      if (ie < ev.size() && (it >= tr.size() || ev[ie].nse <= tr[it].nse)) {
        if (hooks && hooks->on_event) hooks->on_event(&ev[ie], hooks->user);
        ++ie;
      } else {
        if (hooks && hooks->on_scan) hooks->on_scan(&tr[it], hooks->user);
        ++it;
      }
    }
    n_ev += S.n_events;
    n_tr += S.n_traces;
    if (S.n_events || S.n_traces) {
      WalkState reset = S;
      reset.n_events = 0;
      reset.n_traces = 0;
      e = cudaMemcpyAsync(W->st, &reset, sizeof(reset), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) { rc = cuda_fail(err, errlen, e, "reset"); break; }
    }
    if (S.status != PSL_OK) {
      const uint32_t L = W->a.L;
      set_err(err, errlen, overflow_msg(S.err_kind == 2, L, S.err_alpha));
      rc = PSL_ERR_OVERFLOW;
      break;
    }
    if (S.done) break;
  }
  if (rc == PSL_OK) {
    psl_walk_record r{};
    rc = psl_walks_records(W, &r, solution_best, err, errlen);
    if (rc == PSL_OK) {
      out->nse = r.nse;
      out->elapsed_seconds = r.elapsed_seconds;
      out->psl_best = r.psl_best;
      out->merit_factor = r.merit_factor;
      out->energy = r.energy;
      out->n_events = n_ev;
      out->n_traces = n_tr;
      out->switches = r.switches;
    }
  }
  psl_walks_destroy(W);
  return rc;
}

}  // extern "C"
