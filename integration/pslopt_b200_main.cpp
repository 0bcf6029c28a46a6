// pslopt_b200_main.cpp -- the reference CLI's `solve` / `bench` / `verify`
// subcommands (proj/tools/main.cpp:41-181) on the B200 engine.
//
// Same flags, defaults ("length-dependent defaults apply only where the user
// did not say otherwise", main.cpp:65-73), stdout lines and exit codes
// (0 ok, 1 usage/config, 2 overflow, 3 I/O or parse; main.cpp:21-26).  Output
// files are written by the reference's own io.cpp (pslopt-run v1 record,
// convergence CSV, +/- sequence file), linked unchanged; search calls go
// through integration/pslopt_search_b200.cpp to the GPU.  The reference CLI
// itself needs CLI11 (absent from the reference tree), so flags are parsed
// here by hand.  `bench` runs its seeds as concurrent walks on the device
// (psl_run_walks): same per-seed records as sequential run_search calls.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "pslb200.h"
#include "pslopt/errors.hpp"
#include "pslopt/io.hpp"
#include "pslopt/search.hpp"
#include "pslopt/sequence.hpp"

namespace {

constexpr int kExitOk = 0, kExitUsage = 1, kExitOverflow = 2, kExitIo = 3;

struct Args {
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
};

uint64_t to_u64(const std::string& s, const char* flag) {
  char* end = nullptr;
  const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
  if (s.empty() || *end) throw pslopt::ConfigError(std::string("bad value for ") + flag + ": " + s);
  return v;
}

Args parse(int argc, char** argv, int first) {
  static const std::map<std::string, std::string> alias = {{"-L", "--length"}};
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string f = argv[i];
    if (alias.count(f)) f = alias.at(f);
    if (f == "--histogram") { a.kv[f] = "1"; continue; }
    if (f.rfind("--", 0) != 0) { a.kv["positional"] = f; continue; }
    if (i + 1 >= argc) throw pslopt::ConfigError("flag " + f + " needs a value");
    a.kv[f] = argv[++i];
  }
  return a;
}

pslopt::SearchParams search_params(const Args& a) {
  if (!a.has("--length")) throw pslopt::ConfigError("--length is required");
  const uint32_t L = (uint32_t)to_u64(a.get("--length"), "--length");
  pslopt::SearchParams p = pslopt::default_params(L);   // main.cpp:65-73
  p.seed = a.has("--seed") ? to_u64(a.get("--seed"), "--seed") : 1;
  if (a.has("--alpha1")) p.alpha1 = (uint32_t)to_u64(a.get("--alpha1"), "--alpha1");
  if (a.has("--alpha2")) p.alpha2 = (uint32_t)to_u64(a.get("--alpha2"), "--alpha2");
  if (a.has("--ls-lmt")) p.ls_lmt = (uint32_t)to_u64(a.get("--ls-lmt"), "--ls-lmt");
  if (a.has("--flip-lmt")) p.flip_lmt = (uint32_t)to_u64(a.get("--flip-lmt"), "--flip-lmt");
  if (a.has("--n-lmt")) p.n_lmt = (uint32_t)to_u64(a.get("--n-lmt"), "--n-lmt");
  if (a.has("--workers")) p.workers = (uint32_t)to_u64(a.get("--workers"), "--workers");
  if (a.has("--max-nse")) p.stop.max_nse = to_u64(a.get("--max-nse"), "--max-nse");
  if (a.has("--max-seconds")) p.stop.max_seconds = std::atof(a.get("--max-seconds").c_str());
  return p;
}

int solve(const Args& a) {   // main.cpp:75-105
  pslopt::SearchParams p = search_params(a);
  if (a.has("--init")) {
    const pslopt::BinarySequence init = pslopt::io::read_sequence(a.get("--init"));
    p.init = std::vector<int8_t>(init.elements().begin(), init.elements().end());
  }
  std::string warnings;
  const pslopt::SearchParams params = pslopt::validate_params(p, &warnings);
  if (!warnings.empty()) std::fputs(warnings.c_str(), stderr);
  pslopt::SearchHooks hooks;
  const std::string log = a.get("--log");
  if (!log.empty()) {
    std::remove(log.c_str());
    hooks.on_event = [&log](const pslopt::ConvergenceEvent& e) {
      pslopt::io::append_convergence_csv(log, e);
    };
  }
  const pslopt::RunRecord rec = pslopt::run_search(params, hooks);
  if (a.has("--out")) pslopt::io::write_run_record(a.get("--out"), rec);
  if (a.has("--best")) pslopt::io::write_sequence(a.get("--best"), rec.solution_best);
  std::printf("PSL=%d NSE=%llu MF=%.6f elapsed=%.3fs\n", rec.psl_best,
              (unsigned long long)rec.nse, rec.merit_factor, rec.elapsed_seconds);
  return kExitOk;
}

int default_device() {
  const char* dev = std::getenv("PSLB200_DEVICE");
  return dev ? std::atoi(dev) : 0;
}

std::vector<int> devices(const Args& a) {
  std::string list = a.get("--devices");
  if (list.empty()) {
    const char* env = std::getenv("PSLB200_DEVICES");
    if (env) list = env;
  }
  std::vector<int> out;
  size_t pos = 0;
  while (pos < list.size()) {
    size_t end = list.find(',', pos);
    if (end == std::string::npos) end = list.size();
    out.push_back((int)to_u64(list.substr(pos, end - pos), "--devices"));
    pos = end + 1;
  }
  if (out.empty()) out.push_back(default_device());
  return out;
}

int bench(const Args& a) {   // main.cpp:142-181
  pslopt::SearchParams params = search_params(a);
  const std::string mode = a.get("--mode", "two-phase");
  const uint32_t runs = a.has("--runs") ? (uint32_t)to_u64(a.get("--runs"), "--runs") : 10;
  if (mode == "single-alpha1") params.alpha2 = params.alpha1;
  else if (mode == "single-alpha2") params.alpha1 = params.alpha2;
  else if (mode != "two-phase") throw pslopt::ConfigError("unknown bench mode '" + mode + "'");
  std::string warnings;
  params = pslopt::validate_params(params, &warnings);
  if (!warnings.empty()) std::fputs(warnings.c_str(), stderr);
  std::printf("mode=%s L=%u runs=%u alpha1=%u alpha2=%u\n", mode.c_str(), params.length, runs,
              params.alpha1, params.alpha2);
  psl_params c{};
  c.length = params.length; c.seed = params.seed; c.alpha1 = params.alpha1;
  c.alpha2 = params.alpha2; c.ls_lmt = params.ls_lmt; c.flip_lmt = params.flip_lmt;
  c.n_lmt = params.n_lmt; c.workers = params.workers;
  c.has_max_nse = params.stop.max_nse.has_value(); c.max_nse = params.stop.max_nse.value_or(0);
  c.has_max_seconds = params.stop.max_seconds.has_value();
  c.max_seconds = params.stop.max_seconds.value_or(0.0);
  // the seeds run as concurrent walks, split over the selected GPUs
  // (--devices 0,1,... or PSLB200_DEVICES; default PSLB200_DEVICE or 0)
  std::vector<int> devs = devices(a);
  if (devs.size() > runs) devs.resize(runs);
  char err[1024] = {0};
  std::vector<psl_walk_record> recs(runs);
  uint32_t best = 0;
  std::vector<double> dev_s(devs.size());
  const int rc = psl_run_walks_multi(devs.data(), (uint32_t)devs.size(), &c, runs, nullptr, nullptr,
                                     recs.data(), nullptr, &best, dev_s.data(), err, sizeof err);
  if (rc == PSL_ERR_OVERFLOW) throw pslopt::OverflowError(err);
  if (rc != PSL_OK) throw pslopt::ConfigError(err);
  uint64_t total_nse = 0, psl_sum = 0;
  double total_seconds = 0.0;
  int32_t psl_min = 0, psl_max = 0;
  for (uint32_t r = 0; r < runs; ++r) {
    const psl_walk_record& w = recs[r];
    if (w.status == PSL_ERR_OVERFLOW)
      throw pslopt::OverflowError("fitness overflow in run seed " + std::to_string(w.seed));
    std::printf("run seed=%llu psl=%d nse=%llu elapsed=%.3fs mf=%.4f\n",
                (unsigned long long)w.seed, w.psl_best, (unsigned long long)w.nse,
                w.elapsed_seconds, w.merit_factor);
    total_nse += w.nse;
    total_seconds += w.elapsed_seconds;
    psl_sum += (uint64_t)w.psl_best;
    if (r == 0 || w.psl_best < psl_min) psl_min = w.psl_best;
    if (r == 0 || w.psl_best > psl_max) psl_max = w.psl_best;
  }
  // runs execute concurrently: evals-per-sec is sum(nse) / sum(elapsed) as in
  // the reference, plus the aggregate device throughput
  double wall = 0.0;
  for (const auto& w : recs) wall = w.elapsed_seconds > wall ? w.elapsed_seconds : wall;
  std::printf("psl mean=%.3f min=%d max=%d evals-per-sec=%.1f aggregate-evals-per-sec=%.1f\n",
              (double)psl_sum / runs, psl_min, psl_max, (double)total_nse / total_seconds,
              (double)total_nse / wall);
  if (devs.size() > 1)
    std::printf("devices=%zu best seed=%llu psl=%d\n", devs.size(),
                (unsigned long long)recs[best].seed, recs[best].psl_best);
  return kExitOk;
}

int verify(const Args& a) {   // main.cpp:107-124, on the device
  const std::string path = a.get("positional");
  if (path.empty()) throw pslopt::ConfigError("verify needs a sequence file");
  const pslopt::BinarySequence seq = pslopt::io::read_sequence(path);
  psl_ctx* ctx = nullptr;
  char err[1024] = {0};
  if (psl_ctx_create(default_device(), &ctx, err, sizeof err) != PSL_OK) throw pslopt::Error(err);
  const uint32_t L = seq.length();
  std::vector<uint64_t> hist((size_t)L + 1);
  int32_t psl = 0;
  double mf = 0.0;
  int64_t energy = 0;
  const int rc = psl_verify_sequence(ctx, seq.data(), L, &psl, &mf, &energy, hist.data(),
                                     (uint32_t)hist.size(), err, sizeof err);
  psl_ctx_destroy(ctx);
  if (rc != PSL_OK) throw pslopt::ConfigError(err);
  const bool below = (int64_t)psl * psl < (int64_t)L;
  std::printf("L=%u PSL=%d MF=%.6f PSL<sqrt(L): %s\n", L, psl, mf, below ? "yes" : "no");
  if (a.has("--histogram"))
    for (int32_t v = 0; v <= psl; ++v) std::printf("|C|=%d: %llu\n", v, (unsigned long long)hist[v]);
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: pslopt_b200 {solve|bench|verify} [flags]\n");
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse(argc, argv, 2);
    if (cmd == "solve") return solve(a);
    if (cmd == "bench") return bench(a);
    if (cmd == "verify") return verify(a);
    std::fprintf(stderr, "unknown subcommand %s\n", cmd.c_str());
    return kExitUsage;
  } catch (const pslopt::OverflowError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitOverflow;
  } catch (const pslopt::ConfigError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  } catch (const pslopt::ParseError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitIo;
  } catch (const pslopt::IoError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitIo;
  } catch (const pslopt::Error& e) {            // main.cpp:253-255 (engine/device errors too)
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  } catch (const std::exception& e) {           // main.cpp:256-258
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  }
}
