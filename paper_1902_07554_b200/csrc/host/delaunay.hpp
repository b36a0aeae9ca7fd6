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
// Only those rules fix the result (a unique DT under the tie rule); the
// construction is this repo's own: a seeded BRIO insertion order (rounds
// sorted along a Morton curve), the first cell from the first D+1 affinely
// independent points (exact tests), a deterministic visibility walk from the
// last created cell (linear-scan fallback on degenerate ties), a depth-first
// cavity search with per-cell marks, new cells linked through an
// open-addressing ridge table, and cavity slots recycled only after every
// outside cell's back link was found (cf. the reference's slot-reuse defect,
// SURVEY.md F4). tests/test_host.py pins the canonical forms against the
// reference's compiled triangulate_seq (golden), incl. near-degenerate sets.
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
