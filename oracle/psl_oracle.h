/*
 * psl_oracle.h -- CPU restatement of the reference search hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker.  The product path (paper_2107_09801_b200) never links
 * or calls it.
 *
 * Every function restates one reference function; the citation is the
 * reference file:line under /root/reference/proj.  Arithmetic follows the
 * reference exactly: the fitness is a serial ascending-k IEEE double sum of
 * pow_int() values, compiled with -ffp-contract=off like the reference
 * (proj/src/CMakeLists.txt:14).  Parity of this restatement is pinned against
 * the reference itself (oracle/_ref, built from the reference sources) and
 * against the golden vectors in tests/golden/.
 */
#ifndef PSL_ORACLE_H
#define PSL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:18-59 : xoshiro256** seeded by splitmix64 ---------------- */
typedef struct { uint64_t s[4]; } orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);          /* rng.hpp:20-30 */
uint64_t orc_rng_next(orc_rng* r);                     /* rng.hpp:32-42 */
uint64_t orc_rng_bounded(orc_rng* r, uint64_t n);      /* rng.hpp:46-52 */
int8_t orc_rng_spin(orc_rng* r);                       /* rng.hpp:55    */

/* ---- sequence.cpp ------------------------------------------------------ */
double orc_pow_int(double base, uint32_t exp);                       /* :95-105  */
void orc_power_table(uint32_t max_abs, uint32_t alpha, double* lut); /* :107-115 */
void orc_build_table(const int8_t* s, uint32_t L, int32_t* c);       /* :46-60   */
void orc_build_table_fast(const int8_t* s, uint32_t L, int32_t* c);  /* same result, bit-parallel */
void orc_build_table_mt(const int8_t* s, uint32_t L, int32_t* c, uint32_t nthreads);
int32_t orc_psl(const int32_t* c, uint32_t L);                       /* :84-93   */
double orc_fitness(const int32_t* c, uint32_t L, const double* lut); /* :131-141 */
double orc_merit_factor(const int32_t* c, uint32_t L);               /* :143-152 */
int64_t orc_energy(const int32_t* c, uint32_t L);                    /* :146-149 */
void orc_flip_deltas(const int8_t* s, uint32_t L, uint32_t j, int32_t* out); /* :154-172 */
void orc_eval_flip(const int8_t* s, const int32_t* c, uint32_t L, uint32_t j,
                   const double* lut, double* fitness, int32_t* psl); /* sequence.hpp:126-162 */
void orc_apply_flip(int8_t* s, int32_t* c, uint32_t L, uint32_t j);  /* :198-224 */

/* ---- search.cpp -------------------------------------------------------- */
uint32_t orc_default_alpha2(uint32_t L);                             /* :19-23 */
void orc_random_sequence(orc_rng* r, uint32_t L, int8_t* s);         /* :120-129 */
/* flip_random_distinct (:131-148); `used` is caller scratch of L bytes. */
void orc_flip_random_distinct(int8_t* s, int32_t* c, uint32_t L, uint32_t count,
                              orc_rng* r, uint8_t* used);
/* scan_chunk(job, 1, n+1) (:167-175): values[i], psls[i] for i = 1..n */
void orc_scan(const int8_t* s, const int32_t* c, uint32_t L, uint32_t start,
              uint32_t n, const double* lut, double* values, int32_t* psls);
/* reduce_scan (:271-292); returns 1 on the first non-finite value (the
 * reference throws OverflowError there), else 0. */
int orc_reduce(const double* values, const int32_t* psls, uint32_t n,
               uint32_t* best_i, double* value_step, int32_t* psl_min,
               uint32_t* psl_i);

/* run_search (:327-430).  Status codes match the product C-ABI:
 * 0 ok, 1 config error, 2 overflow error, 4 event/trace capacity exceeded. */
typedef struct {
  uint32_t length;
  uint64_t seed;
  uint32_t alpha1, alpha2, ls_lmt, flip_lmt, n_lmt;
  uint64_t max_nse;          /* 0 = unset */
  const int8_t* init;        /* NULL = draw a random pivot */
} orc_params;

typedef struct {
  uint64_t nse;
  int32_t psl_best;
  uint32_t phase;
  uint32_t kind;             /* 0 improved-psl, 1 phase-switch, 2 local-best-improved */
} orc_event;

typedef struct {
  uint64_t nse;
  double value_step;
  double value_local;
  int32_t psl_best;
  uint32_t phase;
} orc_trace;

typedef struct {
  uint64_t nse;
  int32_t psl_best;
  double merit_factor;
  int64_t energy_best;
  uint64_t n_events;
  uint64_t n_traces;
  uint64_t switches;
} orc_record;

int orc_run_search(const orc_params* p, int8_t* solution_best, orc_record* rec,
                   orc_event* events, uint64_t events_cap, orc_trace* traces,
                   uint64_t traces_cap);

#ifdef __cplusplus
}
#endif
#endif
