// psl_internal.h -- shared between the kernels (psl_kernels.cu) and the C-ABI
// host layer (psl_api.cu).  Not part of the public boundary (include/pslb200.h).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/pslb200.h"

namespace pslb {

constexpr int kThreads = 256;      // one CTA per walk
constexpr int kJ = 4;              // adjacent neighbours scored per thread
constexpr int kGroup = kThreads * kJ;  // neighbours per sweep (1024)
constexpr int kChunk = 512;        // k records staged in shared memory per chunk
constexpr int kRecDoubles = 8;     // per-k record: BOTH[e4,e2,e2,e0] ONE[e3,e1,e1,e2]
constexpr int kHCap = 1024;        // filtered high-sidelobe list kept in smem
constexpr int kBitsPad = 8;        // zero words after each global bit array

// Per-walk device state (global memory), resumable across launches.
struct WalkState {
  uint64_t rng[4];
  uint64_t seed;
  uint64_t nse;
  uint64_t unimproved;
  uint64_t switches;
  uint64_t steps;
  uint64_t t0_ns;
  uint64_t end_ns;
  uint64_t n_events;
  uint64_t n_traces;
  double value_local;
  int64_t energy_best;
  int32_t psl_best;
  int32_t P;            // PSL of the pivot table after the last pass
  int32_t P_local;      // PSL of the phase-local snapshot table
  uint32_t phase;
  uint32_t n_pending;   // pending flips the next pass folds into C
  uint32_t src_local;   // next pass reads C from the local snapshot (restart)
  uint32_t local_pending;    // next pass copies its PRE-fold C into the local snapshot
                             // (the snapshot is materialised lazily: only when the
                             // pivot first moves away from the local best)
  uint32_t loc_at_pivot;     // the local best IS the current pivot (snapshot not
                             // materialised; its table is Cpiv after the next fold)
  uint32_t fitness_pending;  // next pass runs the serial pivot-fitness chain
  int32_t status;       // PSL_OK / PSL_ERR_OVERFLOW
  uint32_t err_alpha;
  uint32_t err_kind;    // 1 fitness(), 2 reduce_scan()
  uint32_t done;        // stop condition reached
  uint32_t trace_patch; // 1: last trace waits for value_local
  uint32_t switch_pending;  // 1: last event is a provisional phase-switch
  uint32_t vl_exact;    // value_local is the serial double (else only [vl_lo, vl_hi] is known,
                        // and the exact value is fitness() of the local snapshot table)
  double vl_lo, vl_hi;
  uint64_t n_cert;      // steps decided by the certified scan alone
  uint64_t n_refine;    // certified steps that needed the exact sweep
  uint64_t n_vlchain;   // exact value_local chains over the local snapshot
  uint64_t n_mma;       // tensor-core mma.sync m16n8k32 instructions (per warp) issued
  uint64_t n_umma;      // tcgen05.mma M128 N64 K32 (kind::i8) instructions issued
  // certificate check mode (RunArgs::cert_check): every certified step is also
  // re-scored by the exact sweep and each row's serial double is tested
  // against the row's interval [lo, hi]
  uint64_t chk_steps;   // certified steps checked
  uint64_t chk_rows;    // rows checked
  uint64_t chk_viol;    // rows whose exact serial double fell outside [lo, hi]
  uint64_t chk_dec;     // steps the intervals decided on their own
  uint64_t chk_dec_bad; // ... whose decision (argmin, value_local order) differs from the exact one
  double chk_tight;     // max |V - mid| / (half-width on V's side) over checked rows (<= 1)
  double chk_relw;      // max (hi - lo) / mid over checked rows
};

struct RunArgs {
  uint32_t L, n, alpha1, alpha2, ls_lmt, flip_lmt;
  uint32_t nwords, nchunks;
  int32_t has_max_nse, has_max_seconds;
  uint64_t max_nse;
  double max_seconds;
  uint32_t step_budget;
  int32_t record_events, record_traces;
  int32_t cert;         // certified scan allowed (decision-exact; never with traces)
  double cert_slack;    // test hook: extra relative interval width (forces the exact fallbacks)
  int32_t cert_check;   // test hook: re-score every certified step exactly and check the intervals
  uint64_t events_cap, traces_cap;
  WalkState* st;
  int32_t* Cpiv;
  int32_t* Cloc;
  size_t c_stride;
  uint32_t* bits_piv;
  uint32_t* bits_loc;
  uint32_t* bits_best;
  uint32_t* used;
  size_t w_stride;   // words per walk region: [front pad][nwords][back pad]
  size_t w_front;    // walk base = region + w_front, word i at base[i + 1]
  int2* hlist;
  size_t h_stride;
  uint32_t* flips;
  size_t f_stride;
  psl_event* events;
  psl_trace* traces;
  double* b2;           // certified scan scratch: [walk][2][1024] band-2 constants
  double* lo_buf;       // certified scan scratch: [walk][n] per-row lower bounds (n > 1024)
  double* iv_buf;       // certified scan scratch: [walk][3][1024] a row group's mid / lo / hi
  const double* lut1;   // PowerTable(L, alpha1) / (L, alpha2) on the device (sequence.hpp:72-84)
  const double* lut2;
  uint32_t lut_n;       // entries per table (> max |C_k| + 4)
  int8_t* sol_out;      // optional: mapped pinned host [walk][L]; a walk that stops writes its
                        // best sequence there from the kernel (overlaps later walks' steps)
};

struct ScanArgs {
  uint32_t L, n, start, nwords, nchunks, lut_size;
  int32_t* P;           // device: PSL of the given table (scan_prep_kernel)
  uint32_t* hcount;     // device: entries in hlist
  const uint32_t* bits;
  const int32_t* C;
  const double* lut;
  int2* hlist;          // device: all k with |C_k| >= P - 8 (any order)
  double* values;       // [n+1]
  int32_t* psls;        // [n+1]
};

size_t run_smem_bytes(bool cert);

// The CUDA error a launcher saw (per host thread): launchers record it when
// they return -1, the C ABI reports it (cudaGetLastError() would already have
// been cleared by the launcher).
inline cudaError_t& launch_error_slot() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}
inline int launch_status(int launches) {
  const cudaError_t e = cudaGetLastError();
  launch_error_slot() = e;
  return e == cudaSuccess ? launches : -1;
}
inline int launch_fail(cudaError_t e) {
  launch_error_slot() = e == cudaSuccess ? cudaErrorUnknown : e;
  return -1;
}
inline cudaError_t take_launch_error() {
  const cudaError_t e = launch_error_slot();
  launch_error_slot() = cudaSuccess;
  return e == cudaSuccess ? cudaErrorUnknown : e;
}

// Launchers (return the number of kernels launched, or -1 on launch error).
// packed: warm starts as nw bit words per walk (stride 0: one shared start), or
// nullptr for random_sequence starts drawn on the device
int launch_init_walks(const RunArgs& a, uint32_t n_walks, const uint64_t* d_seeds,
                      const uint32_t* d_packed, size_t packed_stride, cudaStream_t s);
// RunArgs whose per-walk arrays start at walk w0 (batched setup)
RunArgs walk_offset(const RunArgs& a, uint32_t w0);
int launch_verify(const int32_t* C, uint32_t L, int32_t* psl, unsigned long long* energy,
                  unsigned long long* hist, cudaStream_t s);
int launch_unpack(const uint32_t* bits, size_t w_stride, uint32_t L, uint32_t n_walks, int8_t* out,
                  cudaStream_t s);
int launch_build_tables(const RunArgs& a, uint32_t n_walks, cudaStream_t s);
int launch_build_tables_ntt(const RunArgs& a, uint32_t n_walks, cudaStream_t s);
int launch_run(const RunArgs& a, uint32_t n_walks, cudaStream_t s);
int launch_scan(const ScanArgs& a, cudaStream_t s);
int launch_table_only(const uint32_t* d_bits, int32_t* d_C, uint32_t L, uint32_t nwords,
                      cudaStream_t s);
int launch_power_tables(double* lut, uint32_t lut_n, uint32_t alpha1, uint32_t alpha2,
                        cudaStream_t s);
int launch_apply_flip(uint32_t* d_bits, int32_t* d_C, uint32_t L, uint32_t j, cudaStream_t s);
int launch_flip_deltas(const uint32_t* d_bits, uint32_t L, uint32_t j, int32_t* d_out, cudaStream_t s);
int launch_fitness_chain(const int32_t* d_C, uint32_t L, const double* d_lut, double* d_out,
                         cudaStream_t s);
int probe_peaks(int nsm, cudaStream_t s, double* dadd_cps, double* lds_cps, double* mhz);
int probe_imma(int nsm, cudaStream_t s, double* mma_per_s);
int probe_umma(int nsm, cudaStream_t s, double* mma_per_s);

}  // namespace pslb
