// Shared host-side types and error plumbing for libgmrf_b200.
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
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

// Host setup loops over columns / entries that are independent of one another
// (plan construction): fn(begin, end, thread) on contiguous ranges of [0, n).
// Exceptions thrown by fn are rethrown on the calling thread.
template <typename F>
inline void parallel_ranges(int64_t n, F&& fn, int max_threads = 32) {
  unsigned hw = std::thread::hardware_concurrency();
  int t = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({static_cast<int64_t>(hw ? hw : 1),
                                                                  max_threads, n / 4096 + 1})));
  if (t == 1) {
    fn(static_cast<int64_t>(0), n, 0);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(t);
  for (int i = 0; i < t; ++i)
    th.emplace_back([&, i] {
      try {
        fn(n * i / t, n * (i + 1) / t, i);
      } catch (...) {
        err[i] = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}
inline int parallel_threads(int64_t n, int max_threads = 32) {
  unsigned hw = std::thread::hardware_concurrency();
  return static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>({static_cast<int64_t>(hw ? hw : 1), max_threads, n / 4096 + 1})));
}

}  // namespace gmrf
