// pslopt_search_b200.cpp -- the reference-side binding: pslopt's search API
// (proj/include/pslopt/search.hpp) implemented over the B200 engine's C ABI
// (include/pslb200.h).
//
// This translation unit REPLACES the reference's src/search.cpp (and
// pslopt_sequence_b200.cpp replaces src/sequence.cpp).  Link them with the
// reference's own oracle.cpp / io.cpp and any reference caller (the CLI,
// tests/acceptance.cpp, user code) and every run_search / neighborhood_scan /
// SidelobeTable::build / fitness / evaluate_neighbor / flip_deltas / apply_flip
// call executes on the GPU; nothing else changes.
// oracle/Makefile target `dropin` builds the reference's acceptance gate this
// way (oracle/_ref/acceptance_b200); tests/test_dropin.py runs it on a B200.
#include <cstdlib>
#include <string>
#include <vector>

#include "pslb200.h"
#include "pslb200_engine.hpp"
#include "pslopt/errors.hpp"
#include "pslopt/search.hpp"
#include "pslopt/version.hpp"

namespace pslopt {

namespace {

using b200::engine;
using b200::raise;

psl_params to_c(const SearchParams& p) {
  psl_params c{};
  c.length = p.length;
  c.seed = p.seed;
  c.alpha1 = p.alpha1;
  c.alpha2 = p.alpha2;
  c.ls_lmt = p.ls_lmt;
  c.flip_lmt = p.flip_lmt;
  c.n_lmt = p.n_lmt;
  c.workers = p.workers;
  c.has_max_nse = p.stop.max_nse.has_value();
  c.max_nse = p.stop.max_nse.value_or(0);
  c.has_max_seconds = p.stop.max_seconds.has_value();
  c.max_seconds = p.stop.max_seconds.value_or(0.0);
  c.init = nullptr;
  if (p.init) {
    if (p.init->size() != p.length) {
      // the C ABI reads `length` elements: the checks that precede this one
      // first (search.cpp:40-71), then the reference's message (:72-76)
      char err[512] = {0};
      const int rc = psl_validate_params(&c, nullptr, nullptr, 0, err, sizeof err);
      if (rc != PSL_OK) raise(rc, err);
      throw ConfigError("warm-start sequence has length " + std::to_string(p.init->size()) +
                        ", expected " + std::to_string(p.length));
    }
    c.init = p.init->data();
  }
  return c;
}

}  // namespace

uint32_t default_alpha2(uint32_t length) { return psl_default_alpha2(length); }
uint32_t default_n_lmt(uint32_t length) { return psl_default_n_lmt(length); }
uint32_t default_flip_lmt(uint32_t length) { return psl_default_flip_lmt(length); }

SearchParams default_params(uint32_t length) {
  psl_params c;
  psl_default_params(length, &c);
  SearchParams p;
  p.length = c.length;
  p.alpha1 = c.alpha1;
  p.alpha2 = c.alpha2;
  p.ls_lmt = c.ls_lmt;
  p.flip_lmt = c.flip_lmt;
  p.n_lmt = c.n_lmt;
  return p;
}

SearchParams validate_params(const SearchParams& params, std::string* warning) {
  const psl_params in = to_c(params);
  psl_params out;
  char warn[1024] = {0}, err[1024] = {0};
  const int rc = psl_validate_params(&in, &out, warn, sizeof warn, err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
  if (warning) *warning += warn;
  SearchParams p = params;
  p.n_lmt = out.n_lmt;
  p.flip_lmt = out.flip_lmt;
  return p;
}

const char* to_string(EventKind kind) {
  switch (kind) {
    case EventKind::kImprovedPsl: return "improved-psl";
    case EventKind::kPhaseSwitch: return "phase-switch";
    case EventKind::kLocalBestImproved: return "local-best-improved";
  }
  return "unknown";
}

EventKind event_kind_from_string(const std::string& name) {
  for (EventKind k : {EventKind::kImprovedPsl, EventKind::kPhaseSwitch,
                      EventKind::kLocalBestImproved})
    if (name == to_string(k)) return k;
  throw ParseError("unknown event kind '" + name + "'");
}

// Host-side helpers keep the reference's draw-order contract (search.hpp:126-134).
BinarySequence random_sequence(uint32_t length, Rng& rng) {
  if (length < kMinLength || length > kMaxLength)
    throw ConfigError("length " + std::to_string(length) + " out of supported range [" +
                      std::to_string(kMinLength) + ", " + std::to_string(kMaxLength) + "]");
  std::vector<int8_t> e(length);
  for (auto& x : e) x = rng.spin();
  return BinarySequence(std::move(e));
}

void flip_random_distinct(BinarySequence& s, SidelobeTable& t, uint32_t count, Rng& rng) {
  const uint32_t L = s.length();
  if (count > L)
    throw ConfigError("cannot flip " + std::to_string(count) +
                      " distinct positions in a sequence of length " + std::to_string(L));
  std::vector<uint8_t> used(L, 0);
  for (uint32_t done = 0; done < count;) {
    const uint32_t pos = static_cast<uint32_t>(rng.bounded(L));
    if (used[pos]) continue;
    used[pos] = 1;
    apply_flip(s, t, pos);
    ++done;
  }
}

ScanResult neighborhood_scan(const BinarySequence& pivot, const SidelobeTable& table,
                             const PowerTable& pow, uint32_t start, uint32_t n) {
  if (table.length() != pivot.length())
    throw ConfigError("sidelobe table length does not match sequence length");
  psl_scan_result r{};
  char err[1024] = {0};
  const int rc = psl_neighborhood_scan(engine(), pivot.data(), table.data(), pow.data(),
                                       pow.size(), pow.alpha(), pivot.length(), start, n, &r,
                                       err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
  return {r.best_index, r.value_step, r.best_neighbor_psl, r.best_psl_index};
}

namespace {
struct HookCtx {
  const SearchHooks* hooks;
  std::vector<ConvergenceEvent>* events;
};
void on_event(const psl_event* e, void* user) {
  auto* h = static_cast<HookCtx*>(user);
  h->events->push_back({e->nse, e->elapsed_seconds, e->psl_best, e->phase_index,
                        static_cast<EventKind>(e->kind)});
  if (h->hooks->on_event) h->hooks->on_event(h->events->back());
}
void on_scan(const psl_trace* t, void* user) {
  auto* h = static_cast<HookCtx*>(user);
  h->hooks->on_scan({t->nse, t->value_step, t->value_local, t->psl_best, t->phase_index});
}
}  // namespace

RunRecord run_search(const SearchParams& params, const SearchHooks& hooks) {
  const SearchParams p = validate_params(params);
  const psl_params c = to_c(p);
  std::vector<ConvergenceEvent> events;
  HookCtx hc{&hooks, &events};
  psl_hooks h{on_event, hooks.on_scan ? on_scan : nullptr, &hc};
  psl_run_record rec{};
  std::vector<int8_t> sol(p.length);
  char err[1024] = {0};
  const int rc = psl_run_search(engine(), &c, &h, &rec, sol.data(), err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
  return RunRecord{p,        BinarySequence(std::move(sol)), rec.psl_best, rec.merit_factor,
                   rec.nse,  rec.elapsed_seconds,            std::move(events), kVersion};
}

}  // namespace pslopt
