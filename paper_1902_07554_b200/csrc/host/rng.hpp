// Deterministic random streams for input generation (host setup only).
// Same stream semantics as the reference helpers so seeded inputs are
// identical: mt19937_64 engine, 53-bit uniform01, rejection uniform_index,
// Box-Muller gaussian_pair, splitmix64 mix64/derive_seed
// (/root/reference/proj/include/sbdt/random.hpp:15-43, common.hpp:69-78).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <random>

namespace sbdt_host {

using Rng = std::mt19937_64;

inline std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) {
  return mix64(seed ^ mix64(tag));
}

inline double uniform01(Rng& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

inline std::uint64_t uniform_index(Rng& rng, std::uint64_t n) {
  const std::uint64_t mx = std::numeric_limits<std::uint64_t>::max();
  const std::uint64_t limit = mx - mx % n;
  std::uint64_t x;
  do {
    x = rng();
  } while (x >= limit);
  return x % n;
}

inline void gaussian_pair(Rng& rng, double& z0, double& z1) {
  const double u1 = 1.0 - uniform01(rng);
  const double u2 = uniform01(rng);
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * M_PI * u2;
  z0 = r * std::cos(a);
  z1 = r * std::sin(a);
}

// Sequential normal stream: consumes gaussian_pair two values at a time.
struct NormalStream {
  Rng& rng;
  double spare = 0.0;
  bool has_spare = false;
  explicit NormalStream(Rng& r) : rng(r) {}
  double next() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double z0, z1;
    gaussian_pair(rng, z0, z1);
    spare = z1;
    has_spare = true;
    return z0;
  }
};

// Fixed sub-stream tags: one independent stream per role.
enum StreamTag : std::uint64_t {
  kTagPoints = 1,
  kTagSample = 2,
  kTagSampleDt = 3,
  kTagPartitioner = 4,
  kTagPartialDt = 5,
};

}  // namespace sbdt_host
