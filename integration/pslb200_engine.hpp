// pslb200_engine.hpp -- the one engine context shared by the reference-side
// bindings (pslopt_search_b200.cpp, pslopt_sequence_b200.cpp): created on first
// use on device PSLB200_DEVICE (default 0), status codes mapped back to the
// reference's exception classes (proj/include/pslopt/errors.hpp).
#pragma once

#include <cstdlib>
#include <string>

#include "pslb200.h"
#include "pslopt/errors.hpp"

namespace pslopt::b200 {

inline psl_ctx* engine() {
  static psl_ctx* ctx = [] {
    psl_ctx* c = nullptr;
    char err[512] = {0};
    const char* dev = std::getenv("PSLB200_DEVICE");
    if (psl_ctx_create(dev ? std::atoi(dev) : 0, &c, err, sizeof err) != PSL_OK)
      throw Error(std::string("B200 engine unavailable: ") + err);
    return c;
  }();
  return ctx;
}

[[noreturn]] inline void raise(int rc, const char* err) {
  if (rc == PSL_ERR_CONFIG) throw ConfigError(err);
  if (rc == PSL_ERR_OVERFLOW) throw OverflowError(err);
  throw Error(err);
}

}  // namespace pslopt::b200
