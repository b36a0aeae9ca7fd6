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
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <span>
#include <stdexcept>
#include <vector>

#include "sbdt/sample_partition.hpp"
#include "sbdt/task_pool.hpp"
#include "sbdt/triangulation.hpp"

namespace sbdt {

// SPEC.md:403-406
struct IntersectionPolicy {
  enum Kind { Bbox = SBDT_POLICY_BBOX, Grid = SBDT_POLICY_GRID, Exact = SBDT_POLICY_EXACT };
  Kind kind = Grid;
  double c_G = 1.0;
};

namespace gpu_detail {

// Cube root by a fixed Newton iteration on basic IEEE operations: the repo's
// rounding convention for (V/n)^(1/3) (SPEC.md:403 leaves it open), the same
// sequence as the device grid (csrc/gpu/common.cuh) and the oracle.
inline double cbrt_det(double x) {
  if (!(x > 0.0)) return 0.0;
  int e;
  double m = std::frexp(x, &e);
  int r = e % 3;
  if (r < 0) r += 3;
  m = std::ldexp(m, r);
  e -= r;
  double y = 1.0;
  for (int it = 0; it < 8; ++it) y = y - (y * y * y - m) / (3.0 * y * y);
  return std::ldexp(y, e / 3);
}

// find_border's page-locked staging: slots 8.. of the shared thread-local set
inline PinnedSlot& pinned(int which) { return pinned_slot(8 + which); }

// fn(b, e) over [0, n) in fixed chunks: on the caller's TaskPool (the
// reference's, task_pool.hpp:63-80) when it has workers, else inline — the
// conversions are pure data movement, so results never depend on it.
template <class Fn>
void parallel_chunks(TaskPool* pool, std::size_t n, std::size_t grain, Fn&& fn) {
  if (pool && pool->concurrency() > 1 && n > grain) {
    pool->parallel_for(n, grain, [&](std::size_t b, std::size_t e) { fn(b, e); });
  } else {
    for (std::size_t b = 0; b < n; b += grain) fn(b, std::min(n, b + grain));
  }
}

}  // namespace gpu_detail

// SPEC.md:396-417 (device-side representation: the owner grid; this host
// object carries what the device build needs).
template <int D>
struct GridIndex {
  std::vector<PointId> point_ids;  // the partition's points
  Box<D> global_bbox;
  std::size_t n_total = 0;
  double c_G = 1.0;
  double cell_edge_length = 0.0;   // c_G (vol(global_bbox) / n_total)^(1/D)
};

// pre: partition non-empty. global_bbox / n_total are those of
// the top level of the recursion; find_border grids every level
// with them, so a level's partitions are tested on the same cells.
template <int D>
GridIndex<D> build_grid_index(const PointSet& points, std::span<const PointId> part, const Box<D>& global_bbox,
                              std::size_t n_total, double c_G) {
  if (part.empty()) throw std::invalid_argument("build_grid_index: partition must be non-empty");
  if (!(c_G > 0.0)) throw std::invalid_argument("build_grid_index: c_G must be > 0");
  if (n_total < part.size()) throw std::invalid_argument("build_grid_index: n_total below the partition size");
  for (PointId v : part)
    if (v >= points.size()) throw std::invalid_argument("build_grid_index: point id out of range");
  GridIndex<D> gi;
  gi.point_ids.assign(part.begin(), part.end());
  gi.global_bbox = global_bbox;
  gi.n_total = n_total;
  gi.c_G = c_G;
  double vol = 1.0;
  for (int d = 0; d < D; ++d) vol *= global_bbox.hi[d] - global_bbox.lo[d];
  const double per = vol / static_cast<double>(n_total);
  gi.cell_edge_length = c_G * (D == 2 ? std::sqrt(per) : gpu_detail::cbrt_det(per));
  return gi;
}

// SPEC.md:472-476
struct BorderSet {
  std::vector<std::vector<SimplexId>> simplices;  // per partition: border simplex ids (SPEC BFS)
  std::vector<PointId> border_vertex_ids;         // sorted union of their finite vertices
  std::vector<std::vector<SimplexId>> positive;   // per partition: full-scan positive simplex ids
  std::vector<PointId> positive_vertex_ids;
};

// Options beyond the SPEC signature (the SPEC call is find_border(partials,
// indices, policy, pool) with the defaults below).
struct BorderOptions {
  // SPEC BFS from hull_simplices (BorderSet::simplices / border_vertex_ids);
  // false: the full-scan positive set is the border (north_star semantics:
  // BorderSet::simplices = positive, border_vertex_ids = positive_vertex_ids).
  bool hull_bfs = true;
  // The partition labels of every point (e.g. Partitioning::labels), instead
  // of deriving them from the indices' point lists.
  std::span<const PartitionId> labels{};
  // The PointSet's coordinates and `labels` are those of the last
  // assign_points call on this thread, unchanged: reuse their device copies
  // instead of uploading them again (requires `labels`, the very array
  // assign_points returned).
  bool points_resident = false;
};

template <int D>
BorderSet find_border(std::span<const Triangulation<D>> partials, std::span<const GridIndex<D>> indices,
                      const IntersectionPolicy& policy, TaskPool* pool, const BorderOptions& opts) {
  static_assert(D == 2 || D == 3, "D must be 2 or 3");
  using gpu_detail::parallel_chunks;
  const std::uint32_t k = static_cast<std::uint32_t>(partials.size());
  gpu_detail::PhaseTimes& ph = gpu_detail::last_phases();
  const double t0 = gpu_detail::wall_ms();
  BorderSet out;
  out.simplices.resize(k);
  out.positive.resize(k);
  if (k == 0) return out;
  if (indices.size() != k) throw std::invalid_argument("find_border: one GridIndex per partial triangulation");
  const PointSet& ps = partials[0].points();
  const std::uint64_t n = ps.size();
  // every index of a level carries the same top-level grid
  const GridIndex<D>& g0 = indices[0];
  for (const GridIndex<D>& gi : indices) {
    bool same = gi.n_total == g0.n_total && gi.c_G == g0.c_G;
    for (int d = 0; d < D; ++d) same = same && gi.global_bbox.lo[d] == g0.global_bbox.lo[d] &&
                                       gi.global_bbox.hi[d] == g0.global_bbox.hi[d];
    if (!same) throw std::invalid_argument("find_border: indices built with different grids");
  }
  if (g0.c_G != policy.c_G) throw std::invalid_argument("find_border: policy c_G differs from the indices' c_G");
  // labels: the caller's, or from the indices' point lists (points outside
  // this level's indices are SBDT_UNINDEXED)
  const std::uint32_t* labels = nullptr;
  if (!opts.labels.empty()) {
    if (opts.labels.size() != n) throw std::invalid_argument("find_border: one label per point");
    labels = opts.labels.data();
  } else {
    if (opts.points_resident) throw std::invalid_argument("find_border: points_resident needs the labels array");
    std::uint32_t* lab = gpu_detail::pinned(0).get<std::uint32_t>(n);
    parallel_chunks(pool, n, 1u << 20, [&](std::size_t b, std::size_t e) {
      std::fill(lab + b, lab + e, SBDT_UNINDEXED);
    });
    parallel_chunks(pool, k, 1, [&](std::size_t b, std::size_t e) {
      for (std::size_t p = b; p < e; ++p)
        for (PointId v : indices[p].point_ids) lab[v] = static_cast<std::uint32_t>(p);
    });
    labels = lab;
  }
  // live slots -> the vertex-major SoA rows of the C ABI, in page-locked
  // staging; compact partials (no tombstones) map slot i to row i directly
  std::vector<std::uint64_t> offsets(k + 1, 0);
  std::vector<char> compact(k);
  for (std::uint32_t p = 0; p < k; ++p) {
    compact[p] = partials[p].alive_count() == partials[p].slot_count();
    offsets[p + 1] = offsets[p] + partials[p].alive_count();
  }
  const std::uint64_t S = offsets[k];
  std::uint32_t* verts = gpu_detail::pinned(1).get<std::uint32_t>((D + 1) * S);
  std::uint32_t* nbrs = gpu_detail::pinned(2).get<std::uint32_t>((D + 1) * S);
  std::int8_t* parity = gpu_detail::pinned(3).get<std::int8_t>(S);
  std::vector<std::vector<SimplexId>> slot_of(k);  // non-compact partials only
  parallel_chunks(pool, k, 1, [&](std::size_t b, std::size_t e) {
    for (std::size_t p = b; p < e; ++p) {
      if (compact[p]) continue;
      const Triangulation<D>& t = partials[p];
      std::vector<SimplexId> local(t.slot_count(), kNoSimplex);
      t.for_each_alive([&](SimplexId id, const Simplex<D>&) {
        local[id] = static_cast<SimplexId>(slot_of[p].size());
        slot_of[p].push_back(id);
      });
      for (std::size_t i = 0; i < slot_of[p].size(); ++i) {
        const Simplex<D>& s = t.at(slot_of[p][i]);
        const std::uint64_t row = offsets[p] + i;
        for (int j = 0; j <= D; ++j) {
          verts[std::uint64_t(j) * S + row] = s.vertices[j];
          nbrs[std::uint64_t(j) * S + row] = s.neighbors[j] == kNoSimplex ? kNoSimplex : local[s.neighbors[j]];
        }
        parity[row] = s.parity;
      }
    }
  });
  // The compact partials' rows are converted chunk by chunk from inside the
  // call (sbdt_gpu_set_fill): the C ABI asks for rows [r0, r1) right before
  // it uploads them, so this conversion overlaps the previous chunk's
  // transfer (the non-compact partials were converted above).
  constexpr std::size_t kRowGrain = 1u << 15;
  const bool exact = policy.kind == IntersectionPolicy::Exact;
  auto convert = [&](std::uint64_t r0, std::uint64_t r1) {
    parallel_chunks(pool, r1 - r0, kRowGrain, [&](std::size_t b0, std::size_t e0) {
      const std::size_t b = r0 + b0, e = r0 + e0;
      std::uint32_t p =
          static_cast<std::uint32_t>(std::upper_bound(offsets.begin(), offsets.end(), b) - offsets.begin()) - 1;
      for (std::size_t row = b; row < e;) {
        while (offsets[p + 1] <= row) ++p;
        const std::size_t end = std::min<std::size_t>(e, offsets[p + 1]);
        if (compact[p]) {
          // only what the device reads: all vertex rows; the neighbour rows
          // for the BFS, else only row D (the hull rows' owner, read in place
          // from this page-locked buffer); parity for the exact policy
          const Simplex<D>* raw = partials[p].raw_simplices().data() + (row - offsets[p]);
          for (std::size_t r = row; r < end; ++r)
            for (int j = 0; j <= D; ++j) verts[std::uint64_t(j) * S + r] = raw[r - row].vertices[j];
          for (int j = opts.hull_bfs ? 0 : D; j <= D; ++j)
            for (std::size_t r = row; r < end; ++r) nbrs[std::uint64_t(j) * S + r] = raw[r - row].neighbors[j];
          if (exact)
            for (std::size_t r = row; r < end; ++r) parity[r] = raw[r - row].parity;
        }
        row = end;
      }
    });
  };
  struct FillState {
    decltype(convert)* fn;
    static int call(void* user, int what, std::uint64_t r0, std::uint64_t r1) {
      if (what != SBDT_FILL_ROWS) return 0;
      try {
        (*static_cast<FillState*>(user)->fn)(r0, r1);
        return 0;
      } catch (...) {
        return 1;
      }
    }
  } fill_state{&convert};
  std::uint8_t* positive = gpu_detail::pinned(4).get<std::uint8_t>(S);
  std::uint8_t* border = opts.hull_bfs ? gpu_detail::pinned(5).get<std::uint8_t>(S) : nullptr;
  std::uint32_t* vids = gpu_detail::pinned(6).get<std::uint32_t>(n);
  std::uint32_t* bvids = opts.hull_bfs ? gpu_detail::pinned(7).get<std::uint32_t>(n) : nullptr;
  std::uint64_t nv = 0, nb = 0;
  double gbb[2 * D];
  for (int d = 0; d < D; ++d) gbb[d] = g0.global_bbox.lo[d], gbb[D + d] = g0.global_bbox.hi[d];
  const std::uint32_t flags = (opts.hull_bfs ? SBDT_BORDER_HULL_BFS : 0u) |
                              (opts.points_resident ? SBDT_BORDER_RESIDENT_POINTS : 0u);
  // points_resident: the device keeps the points and labels of the last
  // assign_points call, which handed the C ABI its page-locked copies
  const double* coords_arg = ps.raw().data();
  const std::uint32_t* labels_arg = labels;
  if (opts.points_resident) {
    const gpu_detail::ResidentRecord& rr = gpu_detail::resident();
    if (rr.coords != ps.raw().data() || rr.n != n || rr.labels != opts.labels.data())
      throw std::invalid_argument("find_border: points_resident needs the points and labels of the last assign_points");
    coords_arg = rr.staged_coords;
    labels_arg = rr.staged_labels;
  }
  sbdt_gpu_ctx* ctx = gpu_detail::thread_context();
  const double t1 = gpu_detail::wall_ms();
  struct FillGuard {
    sbdt_gpu_ctx* c;
    ~FillGuard() { sbdt_gpu_set_fill(c, nullptr, nullptr); }
  } fill_guard{ctx};
  sbdt_gpu_set_fill(ctx, &FillState::call, &fill_state);
  gpu_detail::check(ctx,
                    sbdt_gpu_find_border(ctx, D, coords_arg, n, labels_arg, k, offsets.data(), verts, nbrs, parity,
                                         static_cast<int>(policy.kind), policy.c_G, flags, positive, border, vids, &nv,
                                         bvids, opts.hull_bfs ? &nb : nullptr, nullptr, gbb, g0.n_total),
                    "find_border");
  const double t2 = gpu_detail::wall_ms();
  // flags -> per-partition simplex ids (original slot ids): count, size, fill,
  // skipping 8 zero flags at a time
  auto collect = [&](const std::uint8_t* flags, std::uint64_t base, std::uint64_t cnt, std::size_t p,
                     std::vector<SimplexId>& dst) {
    std::uint64_t c = 0;
    for (std::uint64_t i = 0; i < cnt; ++i) c += flags[base + i] != 0;
    dst.resize(c);
    std::uint64_t w = 0, i = 0;
    for (; i < cnt && (base + i) % 8 != 0; ++i)
      if (flags[base + i]) dst[w++] = compact[p] ? static_cast<SimplexId>(i) : slot_of[p][i];
    for (; i + 8 <= cnt; i += 8) {
      std::uint64_t word;
      std::memcpy(&word, flags + base + i, 8);
      if (!word) continue;
      for (std::uint64_t t = i; t < i + 8; ++t)
        if (flags[base + t]) dst[w++] = compact[p] ? static_cast<SimplexId>(t) : slot_of[p][t];
    }
    for (; i < cnt; ++i)
      if (flags[base + i]) dst[w++] = compact[p] ? static_cast<SimplexId>(i) : slot_of[p][i];
  };
  parallel_chunks(pool, k, 1, [&](std::size_t b, std::size_t e) {
    for (std::size_t p = b; p < e; ++p) {
      const std::uint64_t cnt = offsets[p + 1] - offsets[p];
      collect(positive, offsets[p], cnt, p, out.positive[p]);
      // without the BFS the full-scan positive set is the border
      if (border) collect(border, offsets[p], cnt, p, out.simplices[p]);
      else out.simplices[p] = out.positive[p];
    }
  });
  out.positive_vertex_ids.assign(vids, vids + nv);
  out.border_vertex_ids.assign(opts.hull_bfs ? bvids : vids, opts.hull_bfs ? bvids + nb : vids + nv);
  ph.prepare_ms = t1 - t0, ph.device_ms = t2 - t1, ph.finish_ms = gpu_detail::wall_ms() - t2;
  return out;
}

// The SPEC signature: SPEC BFS semantics, labels from the indices.
template <int D>
BorderSet find_border(std::span<const Triangulation<D>> partials, std::span<const GridIndex<D>> indices,
                      const IntersectionPolicy& policy, TaskPool* pool = nullptr) {
  return find_border<D>(partials, indices, policy, pool, BorderOptions{});
}

}  // namespace sbdt
