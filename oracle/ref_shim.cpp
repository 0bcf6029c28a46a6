// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled together with the reference
// sources where they lie (/root/reference/proj/src/{sequence,search,oracle}.cpp)
// by oracle/Makefile into oracle/_ref/libpslref.so.  Nothing here re-implements
// the algorithm: every entry point calls the reference's own public API
// (pslopt::run_search, neighborhood_scan, detail::eval_flip, ...) or the
// reference's naive trajectory oracle (tests/reference_search.hpp).  Used to
// pin oracle/psl_oracle.c, to generate tests/golden/ fixtures, and as the CPU
// baseline ("kind": "reference") in bench.py.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pslopt/errors.hpp"
#include "pslopt/oracle.hpp"
#include "pslopt/rng.hpp"
#include "pslopt/search.hpp"
#include "pslopt/sequence.hpp"
#include "reference_search.hpp"

using namespace pslopt;

namespace {
void put_err(const std::exception& e, char* err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
}
}  // namespace

extern "C" {

struct ref_event { uint64_t nse; int32_t psl_best; uint32_t phase; uint32_t kind; double elapsed; };
struct ref_trace { uint64_t nse; double value_step; double value_local; int32_t psl_best; uint32_t phase; };

void ref_rng(uint64_t seed, uint32_t count, uint64_t* out) {
  Rng r(seed);
  for (uint32_t i = 0; i < count; ++i) out[i] = r.next();
}

void ref_random_sequence(uint64_t seed, uint32_t L, int8_t* out) {
  Rng r(seed);
  BinarySequence s = random_sequence(L, r);
  std::memcpy(out, s.data(), L);
}

int ref_build_table(const int8_t* s, uint32_t L, int32_t* c) {
  try {
    const SidelobeTable t = SidelobeTable::build(BinarySequence(std::vector<int8_t>(s, s + L)));
    std::memcpy(c, t.data(), sizeof(int32_t) * L);
    return 0;
  } catch (const ConfigError&) { return 1; }
}

double ref_pow_int(double base, uint32_t exp) { return pow_int(base, exp); }

// scan_chunk(job, 1, n+1) semantics through detail::eval_flip (search.cpp:167-175).
void ref_scan_values(const int8_t* s, const int32_t* c, uint32_t L, uint32_t start,
                     uint32_t n, const double* lut, double* values, int32_t* psls) {
  for (uint32_t i = 1; i <= n; ++i) {
    const uint32_t pos = (start + i) % L;
    const NeighborEval e = detail::eval_flip(s, c, L, pos, lut);
    values[i] = e.fitness;
    psls[i] = e.psl;
  }
}

// neighborhood_scan (search.cpp:296-321); returns 0 ok, 1 ConfigError, 2 OverflowError.
int ref_neighborhood_scan(const int8_t* s, uint32_t L, uint32_t alpha, uint32_t start,
                          uint32_t n, uint32_t* best_index, double* value_step,
                          int32_t* best_psl, uint32_t* best_psl_index, char* err,
                          size_t errlen) {
  try {
    const BinarySequence seq(std::vector<int8_t>(s, s + L));
    const SidelobeTable t = SidelobeTable::build(seq);
    const PowerTable pow(L, alpha);
    const ScanResult r = neighborhood_scan(seq, t, pow, start, n);
    *best_index = r.best_index;
    *value_step = r.value_step;
    *best_psl = r.best_neighbor_psl;
    *best_psl_index = r.best_psl_index;
    return 0;
  } catch (const OverflowError& e) { put_err(e, err, errlen); return 2; }
  catch (const ConfigError& e) { put_err(e, err, errlen); return 1; }
}

int ref_evaluate_neighbor(const int8_t* s, uint32_t L, uint32_t j, uint32_t alpha,
                          double* fitness, int32_t* psl) {
  try {
    const BinarySequence seq(std::vector<int8_t>(s, s + L));
    const SidelobeTable t = SidelobeTable::build(seq);
    const NeighborEval e = evaluate_neighbor(seq, t, j, alpha);
    *fitness = e.fitness;
    *psl = e.psl;
    return 0;
  } catch (const OverflowError&) { return 2; }
  catch (const ConfigError&) { return 1; }
}

double ref_brute_fitness(const int8_t* s, uint32_t L, uint32_t alpha) {
  return oracle::brute_fitness(BinarySequence(std::vector<int8_t>(s, s + L)), alpha);
}

// run_search (search.cpp:327-430) with hooks capturing events and traces.
int ref_run_search(uint32_t L, uint64_t seed, uint32_t alpha1, uint32_t alpha2,
                   uint32_t ls_lmt, uint32_t flip_lmt, uint32_t n_lmt, uint32_t workers,
                   uint64_t max_nse, double max_seconds, const int8_t* init,
                   int8_t* solution, int32_t* psl_best, double* merit_factor,
                   uint64_t* nse, double* elapsed, ref_event* events, uint64_t events_cap,
                   uint64_t* n_events, ref_trace* traces, uint64_t traces_cap,
                   uint64_t* n_traces, char* err, size_t errlen) {
  SearchParams p;
  p.length = L; p.seed = seed; p.alpha1 = alpha1; p.alpha2 = alpha2;
  p.ls_lmt = ls_lmt; p.flip_lmt = flip_lmt; p.n_lmt = n_lmt; p.workers = workers;
  if (max_nse) p.stop.max_nse = max_nse;
  if (max_seconds > 0) p.stop.max_seconds = max_seconds;
  if (init) p.init = std::vector<int8_t>(init, init + L);
  uint64_t ne = 0, nt = 0;
  SearchHooks hooks;
  hooks.on_event = [&](const ConvergenceEvent& e) {
    if (events && ne < events_cap)
      events[ne] = {e.nse, e.psl_best, e.phase_index,
                    e.kind == EventKind::kImprovedPsl ? 0u
                    : e.kind == EventKind::kPhaseSwitch ? 1u : 2u,
                    e.elapsed_seconds};
    ++ne;
  };
  if (traces) {
    hooks.on_scan = [&](const ScanTrace& t) {
      if (nt < traces_cap) traces[nt] = {t.nse, t.value_step, t.value_local, t.psl_best, t.phase_index};
      ++nt;
    };
  }
  try {
    const RunRecord r = run_search(p, hooks);
    std::memcpy(solution, r.solution_best.data(), L);
    *psl_best = r.psl_best;
    *merit_factor = r.merit_factor;
    *nse = r.nse;
    *elapsed = r.elapsed_seconds;
    *n_events = ne;
    *n_traces = nt;
    return 0;
  } catch (const OverflowError& e) {
    *n_events = ne; *n_traces = nt; put_err(e, err, errlen); return 2;
  } catch (const ConfigError& e) {
    *n_events = ne; *n_traces = nt; put_err(e, err, errlen); return 1;
  }
}

// reftest::reference_search (tests/reference_search.hpp:54-141): the naive
// full-rebuild trajectory oracle used by unit_search.cpp:173-227.
int ref_naive_search(uint32_t L, uint64_t seed, uint32_t alpha1, uint32_t alpha2,
                     uint32_t ls_lmt, uint32_t flip_lmt, uint32_t n_lmt, uint64_t max_nse,
                     int8_t* solution, int32_t* psl_best, uint64_t* nse, uint64_t* switches,
                     ref_trace* traces, uint64_t traces_cap, uint64_t* n_traces) {
  SearchParams p;
  p.length = L; p.seed = seed; p.alpha1 = alpha1; p.alpha2 = alpha2;
  p.ls_lmt = ls_lmt; p.flip_lmt = flip_lmt; p.n_lmt = n_lmt;
  p.stop.max_nse = max_nse;
  const reftest::RefResult r = reftest::reference_search(p);
  std::memcpy(solution, r.solution_best.data(), L);
  *psl_best = r.psl_best;
  *nse = r.nse;
  *switches = r.switches;
  uint64_t nt = 0;
  for (const auto& s : r.steps) {
    if (nt < traces_cap) traces[nt] = {s.nse, s.value_step, s.value_local, s.psl_best, s.phase};
    ++nt;
  }
  *n_traces = nt;
  return 0;
}

// CPU baseline: `threads` independent walks, one per host thread, each a
// stock run_search(default_params(L), seed0 + w, max_nse) call (workers = 1).
// Returns aggregate NSE/s = sum(nse_w) / max(elapsed_w) using each record's own
// clock (which, like the reference, excludes the O(L^2) table build), and the
// wall time including builds.
double ref_bench_walks(uint32_t L, uint64_t seed0, uint32_t threads, uint64_t max_nse,
                       uint32_t n_lmt, uint64_t* total_nse, double* max_elapsed,
                       double* wall_seconds) {
  std::vector<uint64_t> nses(threads, 0);
  std::vector<double> els(threads, 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (uint32_t w = 0; w < threads; ++w) {
    th.emplace_back([&, w] {
      SearchParams p = default_params(L);
      p.seed = seed0 + w;
      if (n_lmt) p.n_lmt = n_lmt;
      p.stop.max_nse = max_nse;
      const RunRecord r = run_search(p);
      nses[w] = r.nse;
      els[w] = r.elapsed_seconds;
    });
  }
  for (auto& t : th) t.join();
  *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t tot = 0;
  double mx = 0.0, rate = 0.0;
  for (uint32_t w = 0; w < threads; ++w) {
    tot += nses[w];
    if (els[w] > mx) mx = els[w];
    rate += static_cast<double>(nses[w]) / els[w];
  }
  *total_nse = tot;
  *max_elapsed = mx;
  return rate;
}

// CPU baseline on a bounded sample: `threads` host threads each evaluate the
// n one-flip neighbours of its own pivot `reps` times with the reference's own
// kernel detail::eval_flip (sequence.hpp:126-162), tables supplied by the
// caller.  Returns neighbour evaluations per second (aggregate).
double ref_bench_eval(const int8_t* seqs, const int32_t* tables, uint32_t L, uint32_t walks,
                      const double* lut, uint32_t n, uint32_t reps, uint32_t threads,
                      double* seconds) {
  std::atomic<uint64_t> evals{0};
  std::vector<double> sink(threads, 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (uint32_t w = 0; w < threads; ++w) {
    th.emplace_back([&, w] {
      const int8_t* s = seqs + static_cast<size_t>(w % walks) * L;
      const int32_t* c = tables + static_cast<size_t>(w % walks) * L;
      double acc = 0.0;
      uint64_t cnt = 0;
      for (uint32_t r = 0; r < reps; ++r) {
        const uint32_t start = (r * 7919u + w * 104729u) % L;
        for (uint32_t i = 1; i <= n; ++i) {
          const NeighborEval e = detail::eval_flip(s, c, L, (start + i) % L, lut);
          acc += e.fitness + e.psl;
          ++cnt;
        }
      }
      sink[w] = acc;
      evals += cnt;
    });
  }
  for (auto& t : th) t.join();
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return static_cast<double>(evals.load()) / *seconds;
}


// ---- CPU baseline: one independent walk per host thread (BASELINE.md's CPU
// plan).  Walk w starts like run_search(seed_w): Rng(seed_w), the
// pivot = random_sequence(L, rng) (search.cpp:333-334, its L spin draws); its
// table comes from the caller (the reference's O(L^2) build is excluded from
// the timed region, search.cpp:335 vs :342).  Each step is the body of the
// run_search loop (search.cpp:371-392): start = rng.bounded(L), the n one-flip
// neighbours scored by detail::eval_flip (scan_chunk, :166-175), reduce_scan's
// first-minimum argmin (:271-292) and apply_flip of the winner (:392).  The
// phase bookkeeping (O(L) copies at most) is left out.
struct RefWalks {
  uint32_t L = 0, n = 0;
  const double* lut = nullptr;
  std::vector<Rng> rng;
  std::vector<std::vector<int8_t>> s;
  std::vector<std::vector<int32_t>> c;
  std::vector<uint64_t> evals;
};

void* ref_walks_create(const uint64_t* seeds, uint32_t walks, uint32_t L, uint32_t n,
                       const int32_t* tables, const double* lut) {
  auto* h = new RefWalks;
  h->L = L; h->n = n; h->lut = lut;
  for (uint32_t w = 0; w < walks; ++w) {
    Rng r(seeds[w]);
    const BinarySequence seq = random_sequence(L, r);
    h->rng.push_back(r);
    h->s.emplace_back(seq.data(), seq.data() + L);
    h->c.emplace_back(tables + (size_t)w * L, tables + (size_t)(w + 1) * L);
  }
  h->evals.assign(walks, 0);
  return h;
}

void ref_walks_destroy(void* handle) { delete static_cast<RefWalks*>(handle); }

// Advances every walk by `steps` steps, one host thread per walk; returns the
// aggregate one-flip evaluations per second (NSE/s) of this call.
double ref_walks_step(void* handle, uint32_t steps, double* seconds, int32_t* psl_out) {
  auto* h = static_cast<RefWalks*>(handle);
  const uint32_t W = (uint32_t)h->s.size(), L = h->L, n = h->n;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (uint32_t w = 0; w < W; ++w) {
    th.emplace_back([h, w, L, n, steps] {
      int8_t* s = h->s[w].data();
      int32_t* c = h->c[w].data();
      for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t start = static_cast<uint32_t>(h->rng[w].bounded(L));
        uint32_t best = 1;
        double bv = 0.0;
        for (uint32_t i = 1; i <= n; ++i) {
          const NeighborEval e = detail::eval_flip(s, c, L, (start + i) % L, h->lut);
          if (i == 1 || e.fitness < bv) { bv = e.fitness; best = i; }
        }
        h->evals[w] += n;
        // apply_flip(seq, table, j) (sequence.cpp:198-224)
        const uint32_t j = (start + best) % L;
        const int32_t sj2 = -2 * static_cast<int32_t>(s[j]);
        for (uint32_t k = 1; k < L; ++k) {
          int32_t touched = 0;
          if (j >= k) touched += s[j - k];
          if (j + k < L) touched += s[j + k];
          c[k] += sj2 * touched;
        }
        s[j] = static_cast<int8_t>(-s[j]);
      }
    });
  }
  for (auto& t : th) t.join();
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (psl_out)
    for (uint32_t w = 0; w < W; ++w) {
      int32_t p = 0;
      for (uint32_t k = 1; k < L; ++k) p = std::max(p, std::abs(h->c[w][k]));
      psl_out[w] = p;
    }
  return (double)W * n * steps / *seconds;
}

}  // extern "C"
