// tangram/rng.hpp -- drop-in for the reference's seeded randomness
// (rng.hpp:27-70): derive_seed (FNV-1a of the component name + splitmix64
// finalizer, via the C ABI's tg_derive_seed) and Rng, std::mt19937_64 with
// the hand-rolled, portable distributions the reference defines (uniform01
// at 53-bit resolution, modulo uniform_int, two-draw Box-Muller).  Host
// code: it seeds the synthetic workload.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <string_view>

#include "tangram_gpu.h"

namespace tangram {

inline std::uint64_t derive_seed(std::uint64_t master, std::string_view component) {
  return tg_derive_seed(master, std::string(component).c_str());
}

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : mt_(seed) {}

  double uniform01() { return std::ldexp(static_cast<double>(mt_() >> 11), -53); }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
    const std::uint64_t n = static_cast<std::uint64_t>(hi - lo) + 1u;
    return lo + static_cast<std::int64_t>(mt_() % n);
  }
  double normal(double mu, double sigma) {
    const double a = 1.0 - uniform01(), b = uniform01();
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    return mu + sigma * std::sqrt(-2.0 * std::log(a)) * std::cos(kTwoPi * b);
  }
  double truncated_normal(double mu, double sigma) { return std::max(0.0, normal(mu, sigma)); }

 private:
  std::mt19937_64 mt_;
};

}  // namespace tangram
