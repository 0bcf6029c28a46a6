/*
 * pslb200.h -- C ABI of the B200-native low-PSL search engine.
 *
 * The drop-in boundary for the reference's search hot path (pslopt,
 * /root/reference/proj).  Plain pointers and sizes only; every entry point
 * names the reference interface it replaces (file:line under proj/).
 * Host buffers in, host buffers out; device memory, streams and kernels are
 * owned by the opaque context.  All calls return a status code:
 *
 *   PSL_OK            0
 *   PSL_ERR_CONFIG    1  -> pslopt::ConfigError   (errors.hpp:15-18)
 *   PSL_ERR_OVERFLOW  2  -> pslopt::OverflowError (errors.hpp:22-25)
 *   PSL_ERR_CUDA      3  device missing / CUDA failure (no CPU fallback)
 *   PSL_ERR_CAPACITY  4  internal buffer capacity (never user-visible from
 *                        psl_run_search, which drains and resumes)
 *
 * and, on error, a NUL-terminated message in (err, errlen) carrying the same
 * text the reference puts in its exception (e.g. the OverflowError message
 * names the length and the exponent and says "alpha2": search.cpp:276-280,
 * sequence.cpp:11-15).
 */
#ifndef PSLB200_H
#define PSLB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PSL_OK = 0,
  PSL_ERR_CONFIG = 1,
  PSL_ERR_OVERFLOW = 2,
  PSL_ERR_CUDA = 3,
  PSL_ERR_CAPACITY = 4
};

/* EventKind (search.hpp:74-78), same numeric order. */
enum { PSL_EVENT_IMPROVED_PSL = 0, PSL_EVENT_PHASE_SWITCH = 1, PSL_EVENT_LOCAL_BEST_IMPROVED = 2 };

/* SearchParams + StopCondition (search.hpp:21-42).  Optional fields carry an
 * explicit has_* flag; init == NULL means "no warm start". */
typedef struct {
  uint32_t length;
  uint64_t seed;
  uint32_t alpha1;
  uint32_t alpha2;
  uint32_t ls_lmt;
  uint32_t flip_lmt;
  uint32_t n_lmt;
  uint32_t workers;          /* echoed only; the device ignores it (search.hpp:37) */
  int32_t has_max_nse;
  uint64_t max_nse;
  int32_t has_max_seconds;
  double max_seconds;
  const int8_t* init;        /* length elements, each +1 / -1, or NULL */
} psl_params;

/* ConvergenceEvent (search.hpp:80-88) */
typedef struct {
  uint64_t nse;
  double elapsed_seconds;
  int32_t psl_best;
  uint32_t phase_index;
  uint32_t kind;
} psl_event;

/* ScanTrace (search.hpp:92-98) */
typedef struct {
  uint64_t nse;
  double value_step;
  double value_local;
  int32_t psl_best;
  uint32_t phase_index;
} psl_trace;

/* RunRecord scalars (search.hpp:109-120); the solution is returned through a
 * caller buffer, the events through the hooks, the params echo is the
 * normalised psl_validate_params() output. */
typedef struct {
  uint64_t nse;
  double elapsed_seconds;
  int32_t psl_best;
  double merit_factor;
  int64_t energy;            /* sum_k C_k^2 of solution_best (exact) */
  uint64_t n_events;
  uint64_t n_traces;
  uint64_t switches;
} psl_run_record;

/* SearchHooks (search.hpp:100-103): invoked on the calling host thread, in
 * event order, after the device buffers are drained. */
typedef void (*psl_event_cb)(const psl_event* ev, void* user);
typedef void (*psl_trace_cb)(const psl_trace* tr, void* user);
typedef struct {
  psl_event_cb on_event;     /* may be NULL */
  psl_trace_cb on_scan;      /* may be NULL; non-NULL enables device tracing */
  void* user;
} psl_hooks;

/* ScanJob (search.cpp:156-165): borrowed host pointers; values/psls slots
 * 1..n are written, slot 0 untouched. */
typedef struct {
  const int8_t* seq;
  const int32_t* table;
  uint32_t length;
  uint32_t start;
  uint32_t n;
  const double* lut;         /* at least max|C_k|+5 entries (PowerTable) */
  uint32_t lut_size;
  double* values;
  int32_t* psls;
} psl_scan_job;

/* ScanResult (search.hpp:136-141) */
typedef struct {
  uint32_t best_index;
  double value_step;
  int32_t best_neighbor_psl;
  uint32_t best_psl_index;
} psl_scan_result;

/* Per-walk record for the many-walk entry point. */
typedef struct {
  uint64_t seed;
  uint64_t nse;
  double elapsed_seconds;
  int32_t psl_best;
  int32_t status;            /* PSL_OK or PSL_ERR_OVERFLOW */
  double merit_factor;
  int64_t energy;
  uint64_t switches;
  uint64_t steps;
} psl_walk_record;

typedef struct psl_ctx psl_ctx;
typedef struct psl_walks psl_walks;

/* ---- context ----------------------------------------------------------- */
int psl_ctx_create(int device, psl_ctx** out, char* err, size_t errlen);
void psl_ctx_destroy(psl_ctx* ctx);
/* Launch subsequent work on this cudaStream_t (NULL = the context's own). */
int psl_ctx_set_stream(psl_ctx* ctx, void* stream);
void* psl_ctx_stream(psl_ctx* ctx);
const char* psl_version(void);                         /* version.hpp:5 */
uint32_t psl_kernel_launches(psl_ctx* ctx);            /* kernels launched so far */
/* Scan mode of subsequent runs.  PSL_SCAN_AUTO (default): steps are scored by
 * the certified tensor-core scan wherever it can decide them and by the exact
 * serial-chain sweep otherwise (records, events and solutions are identical
 * to the reference either way; runs with an on_scan hook always use the exact
 * sweep, since ScanTrace carries the serial doubles).  PSL_SCAN_EXACT: exact
 * sweep on every step.  The PSLB200_SCAN=exact environment variable sets the
 * default. */
#define PSL_SCAN_AUTO 0
#define PSL_SCAN_EXACT 1
int psl_ctx_set_scan_mode(psl_ctx* ctx, int mode);
int psl_ctx_scan_mode(psl_ctx* ctx);
/* Totals over the walks whose records were read on this context: steps decided
 * by the certified scan alone, certified steps re-scored exactly, exact
 * value_local chains, mma.sync (m16n8k32 s8) instructions per warp and
 * tcgen05.mma (M128 N64 K32, kind::i8) instructions. */
int psl_ctx_scan_stats(psl_ctx* ctx, uint64_t* certified, uint64_t* refined, uint64_t* chains,
                       uint64_t* mma, uint64_t* umma);
/* Certificate check (test/validation hook, not a reference interface): when
 * on, every step the certified scan scores (n_lmt <= 1024) is also re-scored
 * by the exact serial-chain sweep; each row's serial double is tested against
 * the row's certified interval [lo, hi] and the intervals' own decision
 * (argmin, value_step vs value_local) against the exact one.  Decisions are
 * then taken from the exact sweep.  Read back with psl_ctx_cert_check_stats:
 * counts[0..4] = steps checked, rows checked, rows outside their interval,
 * steps the intervals decided alone, of those decided differently;
 * maxima[0] = max |V - mid| / half-width, maxima[1] = max (hi - lo) / mid. */
int psl_ctx_set_cert_check(psl_ctx* ctx, int on);
int psl_ctx_cert_check_stats(psl_ctx* ctx, uint64_t counts[5], double maxima[2]);
/* Measurement helpers: mma.sync m16n8k32 s8 instructions per second and
 * tcgen05.mma kind::i8 M128 N64 K32 instructions per second (all SMs). */
int psl_probe_imma(psl_ctx* ctx, double* mma_per_s, char* err, size_t errlen);
int psl_probe_umma(psl_ctx* ctx, double* mma_per_s, char* err, size_t errlen);
/* Measurement helper for the roofline (bench.py): FP64-add pipe throughput
 * (cells/s at one DADD per cell), the divergent-LDS.64+DADD loop rate, and the
 * SM clock seen by the probe. */
int psl_probe_peaks(psl_ctx* ctx, double* dadd_cells_per_s, double* lds_cells_per_s,
                    double* sm_mhz, char* err, size_t errlen);

/* ---- parameters (host logic, search.cpp:19-94, sequence.cpp:95-105) ---- */
uint32_t psl_default_alpha2(uint32_t length);          /* search.cpp:19-23 */
uint32_t psl_default_n_lmt(uint32_t length);           /* search.cpp:25    */
uint32_t psl_default_flip_lmt(uint32_t length);        /* search.cpp:27    */
void psl_default_params(uint32_t length, psl_params* out); /* search.cpp:29-38 */
int psl_validate_params(const psl_params* in, psl_params* out, char* warning,
                        size_t warnlen, char* err, size_t errlen); /* search.cpp:40-94 */
double psl_pow_int(double base, uint32_t exp);         /* sequence.cpp:95-105 */

/* ---- operator seam ----------------------------------------------------- */
/* scan_chunk(job, 1, n+1) / ScanPool::run (search.cpp:167-175, :202-218):
 * values[i], psls[i] of neighbour (start + i) % length for i = 1..n.  lut must be
 * PowerTable(length, alpha)'s length + 1 entries (search.cpp:337-338; else
 * PSL_ERR_CONFIG).  The pivot's PSL and high-sidelobe list are built on the
 * device; device scratch comes from the context's memory pool. */
int psl_scan(psl_ctx* ctx, const psl_scan_job* job, char* err, size_t errlen);
/* neighborhood_scan (search.cpp:296-321); absolute positions in `out`. */
int psl_neighborhood_scan(psl_ctx* ctx, const int8_t* seq, const int32_t* table,
                          const double* lut, uint32_t lut_size, uint32_t alpha,
                          uint32_t length, uint32_t start, uint32_t n,
                          psl_scan_result* out, char* err, size_t errlen);
/* evaluate_neighbor (sequence.cpp:180-196). */
int psl_evaluate_neighbor(psl_ctx* ctx, const int8_t* seq, const int32_t* table,
                          const double* lut, uint32_t lut_size, uint32_t alpha,
                          uint32_t length, uint32_t j, double* fitness, int32_t* psl,
                          char* err, size_t errlen);
/* SidelobeTable::build (sequence.cpp:46-60); table_out[0] = length. */
int psl_build_table(psl_ctx* ctx, const int8_t* seq, uint32_t length, int32_t* table_out,
                    char* err, size_t errlen);
/* oracle::verify_sequence (oracle.cpp:172-197): table on the device, then PSL,
 * merit factor (exact int64 energy), and the |C_k| histogram (entries 0..
 * min(hist_cap, L+1)-1; may be NULL). */
int psl_verify_sequence(psl_ctx* ctx, const int8_t* seq, uint32_t length, int32_t* psl,
                        double* merit_factor, int64_t* energy, uint64_t* histogram,
                        uint32_t hist_cap, char* err, size_t errlen);
/* apply_flip (sequence.cpp:198-224), in place on host buffers. */
int psl_apply_flip(psl_ctx* ctx, int8_t* seq, int32_t* table, uint32_t length, uint32_t j,
                   char* err, size_t errlen);
/* flip_deltas (sequence.cpp:154-172): out[0] = 0, out[k] = delta_k = -2 s_j
 * (s_{j-k} [j-k >= 0] + s_{j+k} [j+k < L]) on the sequence before the flip;
 * out has `length` entries. */
int psl_flip_deltas(psl_ctx* ctx, const int8_t* seq, uint32_t length, uint32_t j, int32_t* out,
                    char* err, size_t errlen);
/* fitness(table, PowerTable) (sequence.cpp:131-141): the serial ascending-k
 * double sum of lut[|C_k|], k = 1..length-1, on the device (bit-identical);
 * a non-finite sum is PSL_ERR_OVERFLOW with the reference's message
 * (sequence.cpp:11-15).  lut_size must exceed max |C_k|. */
int psl_fitness(psl_ctx* ctx, const int32_t* table, uint32_t length, const double* lut,
                uint32_t lut_size, uint32_t alpha, double* fitness, char* err, size_t errlen);

/* ---- run entry points -------------------------------------------------- */
/* run_search (search.cpp:327-430).  solution_best: length bytes. */
int psl_run_search(psl_ctx* ctx, const psl_params* params, const psl_hooks* hooks,
                   psl_run_record* out, int8_t* solution_best, char* err, size_t errlen);

/* Many independent walks (one CTA each), walk w seeded seeds[w] (or
 * params->seed + w when seeds == NULL), optional per-walk warm starts
 * (inits: n_walks*length bytes).  Events/traces are not recorded. */
int psl_walks_create(psl_ctx* ctx, const psl_params* params, uint32_t n_walks,
                     const uint64_t* seeds, const int8_t* inits, psl_walks** out,
                     char* err, size_t errlen);
/* Advance every live walk by at most `steps` search steps (asynchronous on
 * the context stream).  Stop conditions in params still apply. */
int psl_walks_step(psl_walks* w, uint32_t steps, char* err, size_t errlen);
/* Run every walk to its stop condition (max_nse / max_seconds). */
int psl_walks_run(psl_walks* w, char* err, size_t errlen);
/* Synchronise and copy out records (and solutions: n_walks*length bytes, may
 * be NULL). */
int psl_walks_records(psl_walks* w, psl_walk_record* records, int8_t* solutions,
                      char* err, size_t errlen);
void psl_walks_destroy(psl_walks* w);

/* One-call form: create, run to the stop condition, copy out, destroy. When
 * `solutions` is page-locked host memory (cudaHostAlloc / cudaHostRegister,
 * mapped under UVA), each walk's kernel writes its best sequence straight into
 * it as the walk stops, so the copy-out overlaps the steps of later walks;
 * any other buffer gets one device-side unpack and a D2H copy. */
int psl_run_walks(psl_ctx* ctx, const psl_params* params, uint32_t n_walks,
                  const uint64_t* seeds, const int8_t* inits, psl_walk_record* records,
                  int8_t* solutions, char* err, size_t errlen);

/* Many independent walks over several GPUs of one node (
 * the reference's `bench` runs its seeds one after another, tools/main.cpp:
 * 162-176).  Walk w (seed seeds[w], or params->seed + w) runs on device
 * devices[d] for the contiguous block n_walks * d / n_devices <= w <
 * n_walks * (d + 1) / n_devices; one host thread per device creates its own
 * context and runs its block with psl_run_walks, so there is no per-step
 * communication.  The only cross-device step is this host gather: records[w]
 * and solutions[w] (n_walks x L, may be NULL) in global walk order, and
 * *best_walk = the walk with the smallest key (psl_best << 32) | w (the
 * smaller walk index wins PSL ties).  device_seconds (n_devices entries, may be
 * NULL) receives each device's wall time for its block.  A device index may
 * repeat (two contexts on one GPU).  Errors: the first failing device's status
 * and message, in device order. */
int psl_run_walks_multi(const int* devices, uint32_t n_devices, const psl_params* params,
                        uint32_t n_walks, const uint64_t* seeds, const int8_t* inits,
                        psl_walk_record* records, int8_t* solutions, uint32_t* best_walk,
                        double* device_seconds, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif /* PSLB200_H */
