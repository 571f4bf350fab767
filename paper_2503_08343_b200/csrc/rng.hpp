// Host random stream with the reference's exact draw sequence (core/rng.hpp:
// 14-47): mt19937_64, uniform = ((x >> 11) + 0.5)·2⁻⁵³, Box-Muller normals
// returning the cosine branch first and caching the sine branch. Samples and
// RBMC variances of this library consume the same z vectors as the reference
// for the same seed (sample_direct(g, rng), gmrf.hpp:182).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

namespace gmrf {

class HostRng {
 public:
  explicit HostRng(uint64_t seed) : eng_(seed) {}
  double uniform() { return (static_cast<double>(eng_() >> 11) + 0.5) * 0x1.0p-53; }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    const double u1 = uniform(), u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare_ = r * std::sin(th);
    spare_ok_ = true;
    return r * std::cos(th);
  }

 private:
  std::mt19937_64 eng_;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

}  // namespace gmrf
