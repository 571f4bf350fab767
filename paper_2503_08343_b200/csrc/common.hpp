// Shared host-side types and error plumbing for libgmrf_b200.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace gmrf {

using i32 = int32_t;
using i64 = int64_t;

// Status codes crossing the C-ABI (include/gmrf_b200.h).
enum Status : int {
  kOk = 0,
  kNotSpd = 1,       // NotPositiveDefiniteError (reference core/types.hpp:40-48)
  kDimension = 2,    // DimensionError (types.hpp:21-24)
  kStructural = 3,   // StructuralError (types.hpp:16-19)
  kContract = 4,     // ContractError (types.hpp:27-30)
  kCuda = 5,         // device failure (no reference analogue)
  kNumerical = 6,    // NumericalError (types.hpp:33-36)
};

struct Error : std::runtime_error {
  Status status;
  Error(Status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(Status s, const std::string& m) { throw Error(s, m); }

inline void require(bool c, Status s, const std::string& m) {
  if (!c) fail(s, m);
}

}  // namespace gmrf
