// sbdt/border.hpp — drop-in border-geom GridIndex and dc-engine
// `find_border` backed by libsbdt_gpu.so.
//
// As for assign_points, the reference specifies these operations but ships
// no source (border.cpp / dc_engine.cpp, proj/src/CMakeLists.txt:7-8). The
// signatures below are the SPEC's, in the style of the shipped headers;
// partial triangulations are the reference's own Triangulation<D>
// (proj/include/sbdt/triangulation.hpp:162-258) — slots may hold tombstones,
// which are skipped and mapped back, so BorderSet reports original SimplexIds.
//
// Semantics (bit-identical to the CPU oracle):
//   * GridIndex: cell edge c_G (vol(global bbox)/n_total)^(1/D), origin the
//     global bbox lo; a partition's occupied cells are those of its points.
//   * positive(s): the inflated circumsphere (geometry.hpp:179-183) — or,
//     for an infinite simplex, the outer halfspace of its hull facet — reaches
//     an occupied cell of another partition (grid) / another partition's
//     cell-snapped bbox (bbox).
//   * find_border returns the SPEC BFS set: positive simplices connected
//     through positive simplices to hull_simplices() (triangulation.cpp:34-53);
//     BorderSet::positive additionally carries the full-scan flags.
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "sbdt/sample_partition.hpp"
#include "sbdt/triangulation.hpp"

namespace sbdt {

// SPEC.md:403-406
struct IntersectionPolicy {
  enum Kind { Bbox = SBDT_POLICY_BBOX, Grid = SBDT_POLICY_GRID, Exact = SBDT_POLICY_EXACT };
  Kind kind = Grid;
  double c_G = 1.0;
};

// SPEC.md:396-417 (device-side representation: the owner grid; this host
// object carries what the device build needs).
template <int D>
struct GridIndex {
  std::vector<PointId> point_ids;  // the partition's points
  Box<D> global_bbox;
  std::size_t n_total = 0;
  double c_G = 1.0;
  double cell_edge_length = 0.0;
};

template <int D>
GridIndex<D> build_grid_index(const PointSet& points, std::span<const PointId> part, const Box<D>& global_bbox,
                              std::size_t n_total, double c_G) {
  (void)points;
  if (part.empty()) throw std::invalid_argument("build_grid_index: partition must be non-empty");
  GridIndex<D> gi;
  gi.point_ids.assign(part.begin(), part.end());
  gi.global_bbox = global_bbox;
  gi.n_total = n_total;
  gi.c_G = c_G;
  return gi;
}

// SPEC.md:472-476
struct BorderSet {
  std::vector<std::vector<SimplexId>> simplices;  // per partition: border simplex ids (SPEC BFS)
  std::vector<PointId> border_vertex_ids;         // sorted union of their finite vertices
  std::vector<std::vector<SimplexId>> positive;   // per partition: full-scan positive simplex ids
  std::vector<PointId> positive_vertex_ids;
};

template <int D>
BorderSet find_border(std::span<const Triangulation<D>> partials, std::span<const GridIndex<D>> indices,
                      const IntersectionPolicy& policy, TaskPool* pool = nullptr) {
  (void)pool;
  static_assert(D == 2 || D == 3, "D must be 2 or 3");
  const std::uint32_t k = static_cast<std::uint32_t>(partials.size());
  BorderSet out;
  out.simplices.resize(k);
  out.positive.resize(k);
  if (k == 0) return out;
  if (indices.size() != k) throw std::invalid_argument("find_border: one GridIndex per partial triangulation");
  const PointSet& ps = partials[0].points();
  const std::uint64_t n = ps.size();
  std::vector<std::uint32_t> labels(n, 0);
  for (std::uint32_t p = 0; p < k; ++p)
    for (PointId v : indices[p].point_ids) labels[v] = p;
  // Compact the live slots into the vertex-major SoA of the C ABI.
  std::vector<std::uint64_t> offsets(k + 1, 0);
  std::vector<std::vector<SimplexId>> slot_of(k);
  for (std::uint32_t p = 0; p < k; ++p) {
    partials[p].for_each_alive([&](SimplexId id, const Simplex<D>&) { slot_of[p].push_back(id); });
    offsets[p + 1] = offsets[p] + slot_of[p].size();
  }
  const std::uint64_t S = offsets[k];
  std::vector<std::uint32_t> verts((D + 1) * S), nbrs((D + 1) * S);
  std::vector<std::int8_t> parity(S);
  for (std::uint32_t p = 0; p < k; ++p) {
    std::vector<SimplexId> local(partials[p].slot_count(), kNoSimplex);
    for (std::size_t i = 0; i < slot_of[p].size(); ++i) local[slot_of[p][i]] = static_cast<SimplexId>(i);
    for (std::size_t i = 0; i < slot_of[p].size(); ++i) {
      const Simplex<D>& s = partials[p].at(slot_of[p][i]);
      const std::uint64_t row = offsets[p] + i;
      for (int j = 0; j <= D; ++j) {
        verts[std::uint64_t(j) * S + row] = s.vertices[j];
        nbrs[std::uint64_t(j) * S + row] = s.neighbors[j] == kNoSimplex ? kNoSimplex : local[s.neighbors[j]];
      }
      parity[row] = s.parity;
    }
  }
  std::vector<std::uint8_t> positive(S), border(S);
  std::vector<std::uint32_t> vids(n), bvids(n);
  std::uint64_t nv = 0, nb = 0;
  sbdt_gpu_ctx* ctx = gpu_detail::thread_context();
  gpu_detail::check(ctx,
                    sbdt_gpu_find_border(ctx, D, ps.raw().data(), n, labels.data(), k, offsets.data(), verts.data(),
                                         nbrs.data(), parity.data(), static_cast<int>(policy.kind), policy.c_G,
                                         SBDT_BORDER_HULL_BFS, positive.data(), border.data(), vids.data(), &nv,
                                         bvids.data(), &nb, nullptr),
                    "find_border");
  for (std::uint32_t p = 0; p < k; ++p)
    for (std::size_t i = 0; i < slot_of[p].size(); ++i) {
      if (border[offsets[p] + i]) out.simplices[p].push_back(slot_of[p][i]);
      if (positive[offsets[p] + i]) out.positive[p].push_back(slot_of[p][i]);
    }
  out.border_vertex_ids.assign(bvids.begin(), bvids.begin() + nb);
  out.positive_vertex_ids.assign(vids.begin(), vids.begin() + nv);
  return out;
}

}  // namespace sbdt
