// Sequential Bowyer-Watson Delaunay triangulation: the host-setup producer
// of the sample DT and of the k partial DTs that the border kernels consume.
//
// Output conventions are the reference's Triangulation<D> conventions
// (/root/reference/proj/include/sbdt/triangulation.hpp:17-68):
//   * vertices ascending, the infinite sentinel 0xFFFFFFFF sorts last;
//   * neighbors[d] shares the facet opposite vertices[d];
//   * parity = exact orient sign of the stored vertex order (0 if infinite);
//   * the conflict rule (in_sphere tie-broken toward "lowest id is outside",
//     infinite simplices = open outer halfspace with the same tie rule) is the
//     reference's (sequential_dt.cpp:130-169, geometry.hpp:158-166), so the
//     canonical form equals the reference's triangulate_seq output.
// Differences (performance only, result-neutral for a unique DT):
//   * insertion order is a seeded BRIO (biased randomized insertion order,
//     rounds sorted along a Morton curve) and the walk starts at the last
//     created simplex, instead of a uniform shuffle + random start;
//   * cavity slots are recycled only after every outside-neighbor index was
//     recorded during the cavity search (no alias of a freed id; cf. the
//     reference's slot-reuse defect at sequential_dt.cpp:265/296).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace sbdt_host {

constexpr std::uint32_t kInf = 0xFFFFFFFFu;
constexpr std::uint32_t kNone = 0xFFFFFFFFu;

struct DegenerateInputError : std::runtime_error {
  explicit DegenerateInputError(const std::string& w) : std::runtime_error(w) {}
};

// Structure-of-arrays triangulation (compacted: every slot alive).
struct TriSoA {
  int dim = 0;
  std::size_t count = 0;
  std::vector<std::uint32_t> verts;  // (dim+1) x count, vertex-major: verts[j*count + s]
  std::vector<std::uint32_t> nbrs;   // (dim+1) x count
  std::vector<std::int8_t> parity;   // count
};

// Triangulates the points `ids` (global ids into the AoS `coords`, dim 2|3).
// `seed` drives the BRIO order and the walk's random facet rotation.
TriSoA triangulate(int dim, const double* coords, const std::uint32_t* ids, std::size_t n,
                   std::uint64_t seed);

}  // namespace sbdt_host
