/*
 * psl_oracle.c -- CPU restatement of the reference search hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see psl_oracle.h).  Compiled with
 * -O2 -ffp-contract=off so the double chains round exactly like the
 * reference (proj/src/CMakeLists.txt:14).  Citations are into
 * /root/reference/proj.
 */
#include "psl_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:20-30 -- splitmix64 fills the four state words in order. */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) {
    z += 0x9e3779b97f4a7c15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    r->s[i] = x ^ (x >> 31);
  }
}

/* rng.hpp:32-42 -- xoshiro256** 1.0. */
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t* s = r->s;
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

/* rng.hpp:46-52 -- masked rejection; always at least one draw. */
uint64_t orc_rng_bounded(orc_rng* r, uint64_t n) {
  const uint64_t mask = (n <= 1) ? 0 : (~0ull >> __builtin_clzll(n - 1));
  for (;;) {
    const uint64_t v = orc_rng_next(r) & mask;
    if (v < n) return v;
  }
}

/* rng.hpp:55 -- top bit 0 -> +1, 1 -> -1. */
int8_t orc_rng_spin(orc_rng* r) { return (orc_rng_next(r) >> 63) ? (int8_t)-1 : (int8_t)1; }

/* ----------------------------------------------------------- sequence.cpp */

/* sequence.cpp:95-105 -- binary exponentiation, factors lowest bit first. */
double orc_pow_int(double base, uint32_t exp) {
  double result = 1.0;
  double factor = base;
  uint32_t e = exp;
  while (e != 0) {
    if (e & 1u) result *= factor;
    e >>= 1;
    if (e != 0) factor *= factor;
  }
  return result;
}

/* sequence.cpp:107-115 */
void orc_power_table(uint32_t max_abs, uint32_t alpha, double* lut) {
  for (uint32_t a = 0; a <= max_abs; ++a) lut[a] = orc_pow_int((double)a, alpha);
}

/* sequence.cpp:46-60 -- O(L^2) direct correlation; c[0] = L. */
void orc_build_table(const int8_t* s, uint32_t L, int32_t* c) {
  c[0] = (int32_t)L;
  for (uint32_t k = 1; k < L; ++k) {
    int32_t acc = 0;
    for (uint32_t i = 0; i + k < L; ++i) acc += (int32_t)s[i] * (int32_t)s[i + k];
    c[k] = acc;
  }
}

/* Same table, bit-parallel (c_k = (L-k) - 2*#{i : s_i != s_{i+k}}); used by
 * tests at lengths where the O(L^2) byte loop is too slow.  Checked against
 * orc_build_table in tests/test_oracle.py. */
void orc_build_table_fast(const int8_t* s, uint32_t L, int32_t* c) {
  const uint32_t W = (L + 63) / 64;
  uint64_t* b = (uint64_t*)calloc((size_t)W + 2, sizeof(uint64_t));
  for (uint32_t i = 0; i < L; ++i)
    if (s[i] < 0) b[i >> 6] |= 1ull << (i & 63);
  c[0] = (int32_t)L;
  for (uint32_t k = 1; k < L; ++k) {
    const uint32_t n = L - k;  /* pairs (i, i+k), i < n */
    const uint32_t ws = k >> 6, sh = k & 63;
    int64_t diff = 0;
    for (uint32_t w = 0; w * 64 < n; ++w) {
      uint64_t hi = b[w + ws];
      uint64_t shifted = sh ? ((hi >> sh) | (b[w + ws + 1] << (64 - sh))) : hi;
      uint64_t x = b[w] ^ shifted;
      const uint32_t rem = n - w * 64;
      if (rem < 64) x &= (1ull << rem) - 1;
      diff += __builtin_popcountll(x);
    }
    c[k] = (int32_t)n - 2 * (int32_t)diff;
  }
  free(b);
}

/* orc_build_table_fast split over threads (shift k handled by thread
 * k % nthreads, so the O(L-k) work per shift is balanced). */
typedef struct { const uint64_t* b; uint32_t L; int32_t* c; uint32_t t, nt; } orc_tb_job;

static void* orc_tb_worker(void* arg) {
  const orc_tb_job* j = (const orc_tb_job*)arg;
  const uint64_t* b = j->b;
  const uint32_t L = j->L;
  for (uint32_t k = 1 + j->t; k < L; k += j->nt) {
    const uint32_t n = L - k;
    const uint32_t ws = k >> 6, sh = k & 63;
    int64_t diff = 0;
    const uint32_t full = n / 64;
    uint32_t w = 0;
    if (sh) {
      for (; w < full; ++w)
        diff += __builtin_popcountll(b[w] ^ ((b[w + ws] >> sh) | (b[w + ws + 1] << (64 - sh))));
    } else {
      for (; w < full; ++w) diff += __builtin_popcountll(b[w] ^ b[w + ws]);
    }
    if (n & 63) {
      uint64_t hi = b[w + ws];
      uint64_t shifted = sh ? ((hi >> sh) | (b[w + ws + 1] << (64 - sh))) : hi;
      diff += __builtin_popcountll((b[w] ^ shifted) & ((1ull << (n & 63)) - 1));
    }
    j->c[k] = (int32_t)n - 2 * (int32_t)diff;
  }
  return NULL;
}

void orc_build_table_mt(const int8_t* s, uint32_t L, int32_t* c, uint32_t nthreads) {
  const uint32_t W = (L + 63) / 64;
  uint64_t* b = (uint64_t*)calloc((size_t)W + 2, sizeof(uint64_t));
  for (uint32_t i = 0; i < L; ++i)
    if (s[i] < 0) b[i >> 6] |= 1ull << (i & 63);
  c[0] = (int32_t)L;
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  orc_tb_job* jobs = (orc_tb_job*)malloc(sizeof(orc_tb_job) * nthreads);
  for (uint32_t t = 0; t < nthreads; ++t) {
    jobs[t].b = b; jobs[t].L = L; jobs[t].c = c; jobs[t].t = t; jobs[t].nt = nthreads;
    pthread_create(&th[t], NULL, orc_tb_worker, &jobs[t]);
  }
  for (uint32_t t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th); free(jobs); free(b);
}

/* sequence.cpp:84-93 */
int32_t orc_psl(const int32_t* c, uint32_t L) {
  int32_t peak = 0;
  for (uint32_t k = 1; k < L; ++k) {
    const int32_t a = abs(c[k]);
    if (a > peak) peak = a;
  }
  return peak;
}

/* sequence.cpp:131-141 -- serial ascending-k double sum; the caller checks
 * finiteness (the reference throws OverflowError at :139). */
double orc_fitness(const int32_t* c, uint32_t L, const double* lut) {
  double sum = 0.0;
  for (uint32_t k = 1; k < L; ++k) sum += lut[abs(c[k])];
  return sum;
}

/* sequence.cpp:146-149 -- exact int64 energy. */
int64_t orc_energy(const int32_t* c, uint32_t L) {
  int64_t e = 0;
  for (uint32_t k = 1; k < L; ++k) e += (int64_t)c[k] * (int64_t)c[k];
  return e;
}

/* sequence.cpp:143-152 */
double orc_merit_factor(const int32_t* c, uint32_t L) {
  const double num = (double)L * (double)L;
  return num / (2.0 * (double)orc_energy(c, L));
}

/* sequence.cpp:154-172 */
void orc_flip_deltas(const int8_t* s, uint32_t L, uint32_t j, int32_t* out) {
  const int32_t sj2 = -2 * (int32_t)s[j];
  out[0] = 0;
  for (uint32_t k = 1; k < L; ++k) {
    int32_t touched = 0;
    if (j >= k) touched += s[j - k];
    if (j + k < L) touched += s[j + k];
    out[k] = sj2 * touched;
  }
}

/* sequence.hpp:126-162 (detail::eval_flip) -- three ascending k ranges. */
void orc_eval_flip(const int8_t* s, const int32_t* c, uint32_t L, uint32_t j,
                   const double* lut, double* fitness, int32_t* psl) {
  const int32_t sj2 = -2 * (int32_t)s[j];
  const uint32_t left = j, right = L - 1 - j;
  const uint32_t both_end = left < right ? left : right;
  const uint32_t one_end = left < right ? right : left;
  double sum = 0.0;
  int32_t peak = 0;
  uint32_t k = 1;
  for (; k <= both_end; ++k) {
    const int32_t a = abs(c[k] + sj2 * (int32_t)(s[j - k] + s[j + k]));
    sum += lut[a];
    if (a > peak) peak = a;
  }
  if (left >= right) {
    for (; k <= one_end; ++k) {
      const int32_t a = abs(c[k] + sj2 * (int32_t)s[j - k]);
      sum += lut[a];
      if (a > peak) peak = a;
    }
  } else {
    for (; k <= one_end; ++k) {
      const int32_t a = abs(c[k] + sj2 * (int32_t)s[j + k]);
      sum += lut[a];
      if (a > peak) peak = a;
    }
  }
  for (; k < L; ++k) {
    const int32_t a = abs(c[k]);
    sum += lut[a];
    if (a > peak) peak = a;
  }
  *fitness = sum;
  *psl = peak;
}

/* sequence.cpp:198-224 */
void orc_apply_flip(int8_t* s, int32_t* c, uint32_t L, uint32_t j) {
  const int32_t sj2 = -2 * (int32_t)s[j];
  const uint32_t left = j, right = L - 1 - j;
  const uint32_t both_end = left < right ? left : right;
  const uint32_t one_end = left < right ? right : left;
  uint32_t k = 1;
  for (; k <= both_end; ++k) c[k] += sj2 * (int32_t)(s[j - k] + s[j + k]);
  if (left >= right) {
    for (; k <= one_end; ++k) c[k] += sj2 * (int32_t)s[j - k];
  } else {
    for (; k <= one_end; ++k) c[k] += sj2 * (int32_t)s[j + k];
  }
  s[j] = (int8_t)-s[j];
}

/* ------------------------------------------------------------- search.cpp */

/* search.cpp:19-23 */
uint32_t orc_default_alpha2(uint32_t L) {
  if (L < (1u << 18) - 1) return 13;
  if (L < (1u << 19) - 1) return 11;
  return 10;
}

/* search.cpp:120-129 -- L spin draws in position order. */
void orc_random_sequence(orc_rng* r, uint32_t L, int8_t* s) {
  for (uint32_t i = 0; i < L; ++i) s[i] = orc_rng_spin(r);
}

/* search.cpp:131-148 */
void orc_flip_random_distinct(int8_t* s, int32_t* c, uint32_t L, uint32_t count,
                              orc_rng* r, uint8_t* used) {
  memset(used, 0, L);
  uint32_t done = 0;
  while (done < count) {
    const uint32_t pos = (uint32_t)orc_rng_bounded(r, L);
    if (used[pos]) continue;
    used[pos] = 1;
    orc_apply_flip(s, c, L, pos);
    ++done;
  }
}

/* search.cpp:167-175 */
void orc_scan(const int8_t* s, const int32_t* c, uint32_t L, uint32_t start,
              uint32_t n, const double* lut, double* values, int32_t* psls) {
  for (uint32_t i = 1; i <= n; ++i) {
    const uint32_t pos = (uint32_t)(((uint64_t)start + i) % L);
    orc_eval_flip(s, c, L, pos, lut, &values[i], &psls[i]);
  }
}

/* search.cpp:271-292 */
int orc_reduce(const double* values, const int32_t* psls, uint32_t n,
               uint32_t* best_i, double* value_step, int32_t* psl_min,
               uint32_t* psl_i) {
  uint32_t bi = 1, pi = 1;
  double v = values[1];
  int32_t pm = psls[1];
  for (uint32_t i = 1; i <= n; ++i) {
    if (!isfinite(values[i])) return 1;
    if (values[i] < v) { v = values[i]; bi = i; }
    if (psls[i] < pm) { pm = psls[i]; pi = i; }
  }
  *best_i = bi; *value_step = v; *psl_min = pm; *psl_i = pi;
  return 0;
}

/* search.cpp:327-430 -- Algorithm 1, restated with plain copies for the
 * phase-local and best-PSL snapshots.  Only the max_nse stop is supported
 * (the oracle must replay exactly). */
int orc_run_search(const orc_params* p, int8_t* solution_best, orc_record* rec,
                   orc_event* events, uint64_t events_cap, orc_trace* traces,
                   uint64_t traces_cap) {
  const uint32_t L = p->length;
  uint32_t n = p->n_lmt, flip = p->flip_lmt;
  if (L < 2 || L > (1u << 20) || p->alpha1 < 1 || p->alpha2 < 1 ||
      p->ls_lmt < 1 || flip < 1 || n < 1 || p->max_nse < 1)
    return 1;                                      /* validate_params :40-94 */
  if (n > L) n = L;
  if (flip > L) flip = L;

  orc_rng rng;
  orc_rng_seed(&rng, p->seed);
  int8_t* seq = (int8_t*)malloc(L);
  if (p->init) memcpy(seq, p->init, L);
  else orc_random_sequence(&rng, L, seq);          /* :332-334 */
  int32_t* table = (int32_t*)malloc(sizeof(int32_t) * L);
  orc_build_table_fast(seq, L, table);             /* :335 */

  double* pow1 = (double*)malloc(sizeof(double) * (L + 1));
  double* pow2 = (double*)malloc(sizeof(double) * (L + 1));
  orc_power_table(L, p->alpha1, pow1);             /* :337-338 */
  orc_power_table(L, p->alpha2, pow2);
  const double* lut = pow1;
  uint32_t alpha = p->alpha1;
  uint32_t phase = 1;

  int status = 0;
  double value_local = orc_fitness(table, L, lut); /* :348 */
  uint64_t nse = 1;
  int8_t* local_seq = (int8_t*)malloc(L);
  int32_t* local_table = (int32_t*)malloc(sizeof(int32_t) * L);
  int8_t* best_seq = (int8_t*)malloc(L);
  int32_t* best_table = (int32_t*)malloc(sizeof(int32_t) * L);
  double* values = (double*)malloc(sizeof(double) * (n + 1));
  int32_t* psls = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  uint8_t* used = (uint8_t*)malloc(L);
  uint64_t ne = 0, nt = 0, switches = 0;
  if (!isfinite(value_local)) { status = 2; goto done; }
  memcpy(local_seq, seq, L);
  memcpy(local_table, table, sizeof(int32_t) * L);
  memcpy(best_seq, seq, L);
  memcpy(best_table, table, sizeof(int32_t) * L);
  int32_t psl_best = orc_psl(table, L);
  uint64_t unimproved = 0;

#define EMIT(KIND)                                                        \
  do {                                                                    \
    if (ne >= events_cap) { status = 4; goto done; }                      \
    events[ne].nse = nse; events[ne].psl_best = psl_best;                 \
    events[ne].phase = phase; events[ne].kind = (KIND); ++ne;             \
  } while (0)

  while (!(nse >= p->max_nse)) {                   /* :373-374 */
    const uint32_t start = (uint32_t)orc_rng_bounded(&rng, L);
    orc_scan(seq, table, L, start, n, lut, values, psls);
    nse += n;
    uint32_t best_i, psl_i;
    double value_step;
    int32_t psl_min;
    if (orc_reduce(values, psls, n, &best_i, &value_step, &psl_min, &psl_i)) {
      status = 2; goto done;                       /* :275-281 */
    }
    if (psl_min < psl_best) {                      /* :383-389 */
      psl_best = psl_min;
      memcpy(best_seq, seq, L);
      memcpy(best_table, table, sizeof(int32_t) * L);
      orc_apply_flip(best_seq, best_table, L, (uint32_t)(((uint64_t)start + psl_i) % L));
      EMIT(0);
    }
    orc_apply_flip(seq, table, L, (uint32_t)(((uint64_t)start + best_i) % L)); /* :392 */
    if (value_step < value_local) {                /* :394-399 */
      value_local = value_step;
      memcpy(local_seq, seq, L);
      memcpy(local_table, table, sizeof(int32_t) * L);
      unimproved = 0;
      EMIT(2);
    } else if (value_step > value_local) {         /* :400-413 */
      if (++unimproved > p->ls_lmt) {
        memcpy(seq, local_seq, L);
        memcpy(table, local_table, sizeof(int32_t) * L);
        orc_flip_random_distinct(seq, table, L, flip, &rng, used);
        phase = (phase == 1) ? 2u : 1u;
        lut = (phase == 1) ? pow1 : pow2;
        alpha = (phase == 1) ? p->alpha1 : p->alpha2;
        value_local = orc_fitness(table, L, lut);
        if (!isfinite(value_local)) { status = 2; goto done; }
        nse += 1;
        unimproved = 0;
        ++switches;
        EMIT(1);
      }
    }
    if (traces) {                                  /* :417-419 */
      if (nt >= traces_cap) { status = 4; goto done; }
      traces[nt].nse = nse; traces[nt].value_step = value_step;
      traces[nt].value_local = value_local; traces[nt].psl_best = psl_best;
      traces[nt].phase = phase; ++nt;
    }
  }
#undef EMIT
  (void)alpha;
  memcpy(solution_best, best_seq, L);
  rec->nse = nse;
  rec->psl_best = psl_best;
  rec->energy_best = orc_energy(best_table, L);
  rec->merit_factor = orc_merit_factor(best_table, L);  /* :425 */
done:
  rec->n_events = ne;
  rec->n_traces = nt;
  rec->switches = switches;
  if (status != 0) rec->nse = nse;
  free(seq); free(table); free(pow1); free(pow2); free(local_seq);
  free(local_table); free(best_seq); free(best_table); free(values);
  free(psls); free(used);
  return status;
}
