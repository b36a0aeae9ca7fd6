// Host setup pipeline: everything that PRODUCES the hot path's inputs
// (points, sample, sample labels, partial DTs). None of it is on the GPU
// path; it exists so both the GPU path and the CPU oracle consume identical
// seeded arrays. Operations follow SPEC.md's contracts:
//   generate         -> SPEC.md:538-588 with BASELINE.json config parameters
//   deduplicate      -> geometry.cpp:350-388 (keep first occurrence)
//   draw_sample      -> SPEC.md:315-323 (partial Fisher-Yates, no replacement)
//   build_sample_graph/edge_weight -> SPEC.md:324-341
//   partition        -> SPEC.md:257-266 (multilevel recursive bisection)
//   parts bucketing  -> SPEC.md:307-312 (ascending ids per part)
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "delaunay.hpp"

namespace sbdt_host {

enum class Distribution : int { kUniform = 0, kNormal = 1, kBubbles = 2, kLines = 3 };

// params (optional overrides; nparams may be 0):
//   normal : mean, sigma                       (default 0.5, 0.1)
//   bubbles: count, r_min, r_max, jitter       (default 64, 0.02, 0.1, 0.002)
//   lines  : count, jitter                     (default 1000, 1e-4)
std::vector<double> generate(Distribution kind, int dim, std::size_t n, std::uint64_t seed,
                             const double* params, int nparams);

// Removes exact duplicates keeping first occurrences; returns old->new remap.
std::vector<std::uint32_t> deduplicate(int dim, std::vector<double>& coords);

std::vector<std::uint32_t> draw_sample(std::size_t n, std::size_t m, std::uint64_t seed);

struct SampleGraph {
  std::size_t n = 0;
  std::vector<std::uint32_t> xadj, adj;
  std::vector<std::int32_t> w;
};

enum class WeightFn : int { kConstant = 0, kInverse = 1, kLogarithmic = 2, kLinear = 3 };

SampleGraph build_sample_graph(int dim, const double* coords, const std::uint32_t* sample_ids,
                               std::size_t m, const TriSoA& sample_dt, WeightFn fn);

// Balanced k-way partition of the sample graph; labels in [0,k).
std::vector<std::uint32_t> partition_graph(const SampleGraph& g, std::uint32_t k, double eps,
                                           std::uint64_t seed);

std::uint64_t cut_weight(const SampleGraph& g, const std::vector<std::uint32_t>& labels);

// Partial DTs of all k parts, concatenated: part p owns simplices
// [offsets[p], offsets[p+1]); neighbor ids are local to the part.
struct Partials {
  int dim = 0;
  std::uint32_t k = 0;
  std::vector<std::uint64_t> offsets;  // k+1
  std::vector<std::uint32_t> verts;    // (dim+1) x S, vertex-major
  std::vector<std::uint32_t> nbrs;     // (dim+1) x S
  std::vector<std::int8_t> parity;     // S
  std::size_t total() const { return offsets.empty() ? 0 : offsets.back(); }
};

Partials build_partials(int dim, const double* coords, std::size_t n, const std::uint32_t* labels,
                        std::uint32_t k, std::uint64_t seed, unsigned threads);

}  // namespace sbdt_host
