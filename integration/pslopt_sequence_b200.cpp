// pslopt_sequence_b200.cpp -- the reference-side binding of pslopt's sequence
// API (proj/include/pslopt/sequence.hpp) over the B200 engine's C ABI
// (include/pslb200.h).
//
// This translation unit REPLACES the reference's src/sequence.cpp.  The O(L^2)
// table build (SidelobeTable::build, sequence.cpp:46-60), the serial fitness
// chain (fitness, :117-141), the one-flip evaluation (evaluate_neighbor,
// :174-196), the delta vector (flip_deltas, :154-172) and the in-place move
// (apply_flip, :198-224) run on the GPU.  What stays on the host is the
// reference's own bookkeeping: element validation, bounds checks and their
// exception messages, the O(L) integer psl / merit_factor / autocorrelation
// and the PowerTable ctor (pow_int is part of the bit-exact contract and is
// exported by the C ABI as psl_pow_int).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "pslb200.h"
#include "pslb200_engine.hpp"
#include "pslopt/errors.hpp"
#include "pslopt/sequence.hpp"

namespace pslopt {

using b200::engine;
using b200::raise;

BinarySequence::BinarySequence(std::vector<int8_t> elements) : elems_(std::move(elements)) {
  // sequence.cpp:20-35
  const size_t n = elems_.size();
  if (n < kMinLength || n > kMaxLength)
    throw ConfigError("sequence length " + std::to_string(n) + " out of supported range [" +
                      std::to_string(kMinLength) + ", " + std::to_string(kMaxLength) + "]");
  for (size_t i = 0; i < n; ++i)
    if (elems_[i] != 1 && elems_[i] != -1)
      throw ConfigError("sequence element at position " + std::to_string(i) + " is " +
                        std::to_string(int(elems_[i])) + "; elements must be +1 or -1");
}

void BinarySequence::flip(uint32_t j) {   // sequence.cpp:37-44
  if (j >= elems_.size())
    throw ConfigError("flip position " + std::to_string(j) + " out of range for length " +
                      std::to_string(elems_.size()));
  elems_[j] = static_cast<int8_t>(-elems_[j]);
}

SidelobeTable SidelobeTable::build(const BinarySequence& s) {   // sequence.cpp:46-60, on the GPU
  SidelobeTable t;
  t.c_.resize(s.length());
  char err[1024] = {0};
  const int rc = psl_build_table(engine(), s.data(), s.length(), t.c_.data(), err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
  t.c_[0] = static_cast<int32_t>(s.length());
  return t;
}

int32_t SidelobeTable::at(uint32_t k) const {   // sequence.cpp:62-68
  if (k >= c_.size())
    throw ConfigError("correlation shift " + std::to_string(k) + " out of range for length " +
                      std::to_string(c_.size()));
  return c_[k];
}

int32_t autocorrelation(const BinarySequence& s, uint32_t k) {   // sequence.cpp:70-82
  const uint32_t L = s.length();
  if (k >= L)
    throw ConfigError("autocorrelation shift " + std::to_string(k) + " outside 0.." +
                      std::to_string(L - 1));
  const int8_t* e = s.data();
  int32_t acc = 0;
  for (uint32_t i = 0; i + k < L; ++i) acc += static_cast<int32_t>(e[i]) * e[i + k];
  return acc;
}

int32_t psl(const SidelobeTable& t) {   // sequence.cpp:84-93
  int32_t peak = 0;
  for (uint32_t k = 1; k < t.length(); ++k) peak = std::max(peak, std::abs(t.data()[k]));
  return peak;
}

double pow_int(double base, uint32_t exp) { return psl_pow_int(base, exp); }   // sequence.cpp:95-105

PowerTable::PowerTable(uint32_t max_abs_value, uint32_t alpha) : alpha_(alpha) {   // :107-115
  if (alpha < 1) throw ConfigError("fitness exponent must be >= 1");
  lut_.resize(static_cast<size_t>(max_abs_value) + 1);
  for (uint32_t a = 0; a <= max_abs_value; ++a) lut_[a] = psl_pow_int(static_cast<double>(a), alpha);
}

double fitness(const SidelobeTable& t, const PowerTable& pow) {   // sequence.cpp:131-141, on the GPU
  double v = 0.0;
  char err[1024] = {0};
  const int rc = psl_fitness(engine(), t.data(), t.length(), pow.data(), pow.size(), pow.alpha(), &v,
                             err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
  return v;
}

double fitness(const SidelobeTable& t, uint32_t alpha) {   // sequence.cpp:117-129
  if (alpha < 1) throw ConfigError("fitness exponent must be >= 1");
  // pow_int(|C_k|, alpha) term by term == the PowerTable entries (sequence.hpp:70-72)
  return fitness(t, PowerTable(static_cast<uint32_t>(std::max(psl(t), 0)), alpha));
}

double merit_factor(const SidelobeTable& t) {   // sequence.cpp:143-152 (exact int64 energy)
  int64_t energy = 0;
  for (uint32_t k = 1; k < t.length(); ++k)
    energy += static_cast<int64_t>(t.data()[k]) * static_cast<int64_t>(t.data()[k]);
  const double num = static_cast<double>(t.length()) * static_cast<double>(t.length());
  return num / (2.0 * static_cast<double>(energy));
}

void flip_deltas(const BinarySequence& s, uint32_t j, std::span<int32_t> out) {   // :154-172, GPU
  const uint32_t L = s.length();
  if (j >= L)
    throw ConfigError("flip position " + std::to_string(j) + " out of range for length " +
                      std::to_string(L));
  if (out.size() != L) throw ConfigError("flip_deltas output span must have length L");
  char err[1024] = {0};
  const int rc = psl_flip_deltas(engine(), s.data(), L, j, out.data(), err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
}

NeighborEval evaluate_neighbor(const BinarySequence& s, const SidelobeTable& t, uint32_t j,
                               uint32_t alpha) {   // sequence.cpp:174-178
  const PowerTable pow(s.length(), alpha);
  return evaluate_neighbor(s, t, j, pow);
}

NeighborEval evaluate_neighbor(const BinarySequence& s, const SidelobeTable& t, uint32_t j,
                               const PowerTable& pow) {   // sequence.cpp:180-196, on the GPU
  const uint32_t L = s.length();
  if (j >= L)
    throw ConfigError("neighbor position " + std::to_string(j) + " out of range for length " +
                      std::to_string(L));
  if (t.length() != L) throw ConfigError("sidelobe table length does not match sequence length");
  if (pow.size() < L + 1) throw ConfigError("power table too small for sequence length");
  double f = 0.0;
  int32_t p = 0;
  char err[1024] = {0};
  const int rc = psl_evaluate_neighbor(engine(), s.data(), t.data(), pow.data(), pow.size(),
                                       pow.alpha(), L, j, &f, &p, err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
  return {f, p};
}

void apply_flip(BinarySequence& s, SidelobeTable& t, uint32_t j) {   // sequence.cpp:198-224, GPU
  const uint32_t L = s.length();
  if (j >= L)
    throw ConfigError("flip position " + std::to_string(j) + " out of range for length " +
                      std::to_string(L));
  if (t.length() != L) throw ConfigError("sidelobe table length does not match sequence length");
  std::vector<int8_t> e(s.data(), s.data() + L);
  char err[1024] = {0};
  const int rc = psl_apply_flip(engine(), e.data(), t.data(), L, j, err, sizeof err);
  if (rc != PSL_OK) raise(rc, err);
  s.flip(j);
}

}  // namespace pslopt
