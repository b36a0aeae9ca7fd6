// TEST INFRASTRUCTURE (oracle) — CPU restatement of the hot path:
//   assign_points      SPEC.md:342-350,371,382 (nearest sample, ties -> lowest
//                      sample PointId; kd-tree accelerator + brute-force ground truth)
//   GridIndex          SPEC.md:396-417 (occupied cells, per-cell point lists,
//                      AABB tree by recursive median split along the longest axis)
//   intersects_*       SPEC.md:418-443 (+ infinite-simplex rule :451)
//   find_border        SPEC.md:488-496 + PAPER.md:152-165 (BFS from hull_simplices,
//                      triangulation.cpp:34-53) and the north_star full scan.
// Templated on a primitive policy: OwnPrims (oracle/prims.hpp, restated) or
// RefPrims (oracle/ref/ref_glue.cpp, the reference's compiled geometry.cpp).
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <functional>
#include <numeric>
#include <thread>
#include <vector>

#include "prims.hpp"

namespace sbdt_oracle {

constexpr std::uint32_t kInf = 0xFFFFFFFFu;

enum PolicyKind : int { kBbox = 0, kGrid = 1, kExact = 2 };

// Optional external pool (oracle/ref/ref_glue.cpp installs the reference's own
// sbdt::TaskPool, task_pool.hpp:63-80, for the timed "reference" CPU arm).
// Chunking is by `grain` either way, so results are identical.
using ParallelRunner = void (*)(std::size_t n, std::size_t grain,
                                const std::function<void(std::size_t, std::size_t)>& fn);
inline ParallelRunner g_runner = nullptr;

inline void parallel_for(std::size_t n, std::size_t grain, unsigned threads,
                         const std::function<void(std::size_t, std::size_t)>& fn) {
  if (g_runner && threads > 1) {
    g_runner(n, grain, fn);
    return;
  }
  if (threads <= 1 || n <= grain) {
    for (std::size_t b = 0; b < n; b += grain) fn(b, std::min(n, b + grain));
    return;
  }
  std::atomic<std::size_t> next{0};
  auto worker = [&] {
    for (;;) {
      const std::size_t b = next.fetch_add(grain);
      if (b >= n) return;
      fn(b, std::min(n, b + grain));
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < threads; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
}

// ---------------------------------------------------------------------------
// assign_points
// ---------------------------------------------------------------------------
template <int D, class Prims>
void assign_brute(const double* xyz, std::size_t n, const std::uint32_t* sample_ids, std::size_t m,
                  const std::uint32_t* sample_labels, std::uint32_t* labels, unsigned threads) {
  parallel_for(n, 4096, threads, [&](std::size_t b, std::size_t e) {
    for (std::size_t i = b; i < e; ++i) {
      const double* p = xyz + i * D;
      double best = INFINITY;
      std::uint32_t best_id = kInf, best_label = 0;
      for (std::size_t s = 0; s < m; ++s) {
        const double d2 = Prims::sqdist(p, xyz + std::size_t(sample_ids[s]) * D);
        if (d2 < best || (d2 == best && sample_ids[s] < best_id)) {
          best = d2;
          best_id = sample_ids[s];
          best_label = sample_labels[s];
        }
      }
      labels[i] = best_label;
    }
  });
}

// kd-tree over the sample (the reference's nanoflann accelerator).
// Pruning is conservative so the result equals the brute-force argmin exactly.
template <int D, class Prims>
class SampleKdTree {
 public:
  SampleKdTree(const double* xyz, const std::uint32_t* sample_ids, std::size_t m,
               const std::uint32_t* sample_labels)
      : xyz_(xyz), ids_(sample_ids, sample_ids + m), labels_(sample_labels, sample_labels + m) {
    idx_.resize(m);
    std::iota(idx_.begin(), idx_.end(), 0u);
    if (m) build(0, static_cast<std::uint32_t>(m));
  }

  std::uint32_t nearest_label(const double* p) const {
    double best = INFINITY;
    std::uint32_t best_id = kInf, best_label = 0;
    if (nodes_.empty()) return 0;
    std::uint32_t stack[128];
    int top = 0;
    stack[top++] = 0;
    while (top) {
      const Node& nd = nodes_[stack[--top]];
      if (nd.split_dim < 0) {
        for (std::uint32_t i = nd.begin; i < nd.end; ++i) {
          const std::uint32_t s = idx_[i];
          const double d2 = Prims::sqdist(p, xyz_ + std::size_t(ids_[s]) * D);
          if (d2 < best || (d2 == best && ids_[s] < best_id)) {
            best = d2;
            best_id = ids_[s];
            best_label = labels_[s];
          }
        }
        continue;
      }
      const double diff = p[nd.split_dim] - nd.split;
      const std::uint32_t near = diff < 0 ? nd.left : nd.right;
      const std::uint32_t far = diff < 0 ? nd.right : nd.left;
      // far side visited unless provably farther (relative margin >> rounding)
      if (!(diff * diff > best * (1.0 + 1e-9))) stack[top++] = far;
      stack[top++] = near;
    }
    return best_label;
  }

 private:
  struct Node {
    int split_dim;  // -1 leaf
    double split;
    std::uint32_t left, right, begin, end;
  };
  double coord(std::uint32_t s, int d) const { return xyz_[std::size_t(ids_[s]) * D + d]; }
  std::uint32_t build(std::uint32_t b, std::uint32_t e) {
    const std::uint32_t id = static_cast<std::uint32_t>(nodes_.size());
    nodes_.push_back(Node{-1, 0.0, 0, 0, b, e});
    if (e - b <= 8) return id;
    double lo[D], hi[D];
    for (int d = 0; d < D; ++d) lo[d] = hi[d] = coord(idx_[b], d);
    for (std::uint32_t i = b; i < e; ++i)
      for (int d = 0; d < D; ++d) {
        lo[d] = std::min(lo[d], coord(idx_[i], d));
        hi[d] = std::max(hi[d], coord(idx_[i], d));
      }
    int sd = 0;
    for (int d = 1; d < D; ++d)
      if (hi[d] - lo[d] > hi[sd] - lo[sd]) sd = d;
    const std::uint32_t mid = b + (e - b) / 2;
    std::nth_element(idx_.begin() + b, idx_.begin() + mid, idx_.begin() + e,
                     [&](std::uint32_t x, std::uint32_t y) { return coord(x, sd) < coord(y, sd); });
    const double split = coord(idx_[mid], sd);
    // points with coord < split are left of mid, >= right (nth_element guarantee)
    const std::uint32_t l = build(b, mid);
    const std::uint32_t r = build(mid, e);
    nodes_[id].split_dim = sd;
    nodes_[id].split = split;
    nodes_[id].left = l;
    nodes_[id].right = r;
    return id;
  }
  const double* xyz_;
  std::vector<std::uint32_t> ids_, labels_, idx_;
  std::vector<Node> nodes_;
};

template <int D, class Prims>
void assign_kdtree(const double* xyz, std::size_t n, const std::uint32_t* sample_ids, std::size_t m,
                   const std::uint32_t* sample_labels, std::uint32_t* labels, unsigned threads) {
  SampleKdTree<D, Prims> tree(xyz, sample_ids, m, sample_labels);
  parallel_for(n, 4096, threads, [&](std::size_t b, std::size_t e) {
    for (std::size_t i = b; i < e; ++i) labels[i] = tree.nearest_label(xyz + i * D);
  });
}

// ---------------------------------------------------------------------------
// Grid parameters + GridIndex
// ---------------------------------------------------------------------------
template <int D>
struct GridParams {
  double lo[D], hi[D];
  double edge;
  std::int64_t dims[D];
};

// Cube root by a fixed Newton iteration on basic IEEE operations only: the
// repo's convention for the (V/n)^(1/D) rounding, which SPEC.md:403 leaves
// open. The GPU evaluates the identical sequence (csrc/gpu/common.cuh), so
// both sides get the same cell edge bit for bit.
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

// edge = c_G * (vol(global bbox) / n_total)^(1/D)  (SPEC.md:403 / :410 / :450
// convention), origin = global bbox lo, from a given global bbox and n_total
// (recursion levels keep the top level's, build_grid_index post).
template <int D>
GridParams<D> grid_from_bbox(const double* lo, const double* hi, std::size_t n_total, double c_G) {
  GridParams<D> g;
  for (int d = 0; d < D; ++d) g.lo[d] = lo[d], g.hi[d] = hi[d];
  double vol = 1.0;
  for (int d = 0; d < D; ++d) vol *= (g.hi[d] - g.lo[d]);
  const double per = vol / static_cast<double>(n_total);
  g.edge = c_G * (D == 2 ? std::sqrt(per) : cbrt_det(per));
  for (int d = 0; d < D; ++d) g.dims[d] = static_cast<std::int64_t>(std::floor((g.hi[d] - g.lo[d]) / g.edge)) + 1;
  return g;
}

// ... from the bbox of all n points and n_total.
template <int D>
GridParams<D> grid_from_bbox_of(const double* xyz, std::size_t n, std::size_t n_total, double c_G) {
  double lo[D], hi[D];
  for (int d = 0; d < D; ++d) {
    lo[d] = INFINITY;
    hi[d] = -INFINITY;
  }
  for (std::size_t i = 0; i < n; ++i)
    for (int d = 0; d < D; ++d) {
      lo[d] = std::min(lo[d], xyz[i * D + d]);
      hi[d] = std::max(hi[d], xyz[i * D + d]);
    }
  return grid_from_bbox<D>(lo, hi, n_total, c_G);
}

// ... from the bbox of all n points and n.
template <int D>
GridParams<D> grid_params(const double* xyz, std::size_t n, double c_G) {
  double lo[D], hi[D];
  for (int d = 0; d < D; ++d) {
    lo[d] = INFINITY;
    hi[d] = -INFINITY;
  }
  for (std::size_t i = 0; i < n; ++i)
    for (int d = 0; d < D; ++d) {
      lo[d] = std::min(lo[d], xyz[i * D + d]);
      hi[d] = std::max(hi[d], xyz[i * D + d]);
    }
  return grid_from_bbox<D>(lo, hi, n, c_G);
}

// cell = floor((p - lo) / edge), clamped to the grid (SURVEY.md §7 grid decision).
template <int D>
inline std::int64_t cell_coord(const GridParams<D>& g, double x, int d) {
  const double f = std::floor((x - g.lo[d]) / g.edge);
  if (!(f >= 0.0)) return 0;
  if (f >= static_cast<double>(g.dims[d] - 1)) return g.dims[d] - 1;
  return static_cast<std::int64_t>(f);
}
template <int D>
inline Box<D> cell_box(const GridParams<D>& g, const std::int64_t* c) {
  Box<D> b;
  for (int d = 0; d < D; ++d) {
    b.lo[d] = g.lo[d] + static_cast<double>(c[d]) * g.edge;
    b.hi[d] = g.lo[d] + static_cast<double>(c[d] + 1) * g.edge;
  }
  return b;
}

template <int D>
struct GridIndex {
  std::vector<std::int64_t> cells;             // occupied cells, linear ids ascending
  std::vector<std::uint32_t> cell_start;       // CSR into points
  std::vector<std::uint32_t> points;           // point ids per cell
  std::vector<Box<D>> cell_boxes;
  struct Node {
    Box<D> box;
    std::int32_t left = -1, right = -1, leaf = -1;  // leaf = cell index
  };
  std::vector<Node> nodes;  // nodes[0] = root
  Box<D> root_box;          // partition point bbox (diagnostic)
  bool empty() const { return cells.empty(); }
  // Root box of the bbox policy (intersects_bbox): the AABB-tree
  // root, i.e. the partition bbox snapped to its occupied cells. SPEC.md
  // requires both "root_box equals the partition's bounding box" and "every
  // node box contains its leaf boxes"; only the snapped box satisfies the
  // second, and it is what makes the policy chain exact <= grid <= bbox
  // (acceptance criterion 7) hold without exceptions.
  const Box<D>& bbox_policy_box() const { return nodes[0].box; }
};

template <int D>
inline std::int64_t linear_cell(const GridParams<D>& g, const std::int64_t* c) {
  std::int64_t id = c[D - 1];
  for (int d = D - 2; d >= 0; --d) id = id * g.dims[d] + c[d];
  return id;
}
template <int D>
inline void unlinear_cell(const GridParams<D>& g, std::int64_t id, std::int64_t* c) {
  for (int d = 0; d < D; ++d) {
    c[d] = id % g.dims[d];
    id /= g.dims[d];
  }
}

template <int D>
GridIndex<D> build_grid_index(const GridParams<D>& g, const double* xyz, const std::uint32_t* part,
                              std::size_t np) {
  GridIndex<D> gi;
  std::vector<std::pair<std::int64_t, std::uint32_t>> keyed(np);
  for (int d = 0; d < D; ++d) {
    gi.root_box.lo[d] = INFINITY;
    gi.root_box.hi[d] = -INFINITY;
  }
  for (std::size_t i = 0; i < np; ++i) {
    const double* p = xyz + std::size_t(part[i]) * D;
    std::int64_t c[D];
    for (int d = 0; d < D; ++d) {
      c[d] = cell_coord<D>(g, p[d], d);
      gi.root_box.lo[d] = std::min(gi.root_box.lo[d], p[d]);
      gi.root_box.hi[d] = std::max(gi.root_box.hi[d], p[d]);
    }
    keyed[i] = {linear_cell<D>(g, c), part[i]};
  }
  std::sort(keyed.begin(), keyed.end());
  for (std::size_t i = 0; i < np; ++i) {
    if (i == 0 || keyed[i].first != keyed[i - 1].first) {
      gi.cells.push_back(keyed[i].first);
      gi.cell_start.push_back(static_cast<std::uint32_t>(i));
    }
    gi.points.push_back(keyed[i].second);
  }
  gi.cell_start.push_back(static_cast<std::uint32_t>(np));
  gi.cell_boxes.resize(gi.cells.size());
  for (std::size_t c = 0; c < gi.cells.size(); ++c) {
    std::int64_t cc[D];
    unlinear_cell<D>(g, gi.cells[c], cc);
    gi.cell_boxes[c] = cell_box<D>(g, cc);
  }
  // AABB tree: recursive median split of occupied cells along the longest axis.
  if (!gi.cells.empty()) {
    std::vector<std::int32_t> order(gi.cells.size());
    std::iota(order.begin(), order.end(), 0);
    std::function<std::int32_t(std::size_t, std::size_t)> build = [&](std::size_t b, std::size_t e) {
      const std::int32_t id = static_cast<std::int32_t>(gi.nodes.size());
      gi.nodes.emplace_back();
      Box<D> bx = gi.cell_boxes[order[b]];
      for (std::size_t i = b + 1; i < e; ++i)
        for (int d = 0; d < D; ++d) {
          bx.lo[d] = std::min(bx.lo[d], gi.cell_boxes[order[i]].lo[d]);
          bx.hi[d] = std::max(bx.hi[d], gi.cell_boxes[order[i]].hi[d]);
        }
      gi.nodes[id].box = bx;
      if (e - b == 1) {
        gi.nodes[id].leaf = order[b];
        return id;
      }
      int sd = 0;
      for (int d = 1; d < D; ++d)
        if (bx.hi[d] - bx.lo[d] > bx.hi[sd] - bx.lo[sd]) sd = d;
      const std::size_t mid = b + (e - b) / 2;
      std::nth_element(order.begin() + b, order.begin() + mid, order.begin() + e,
                       [&](std::int32_t x, std::int32_t y) {
                         return gi.cell_boxes[x].lo[sd] < gi.cell_boxes[y].lo[sd] ||
                                (gi.cell_boxes[x].lo[sd] == gi.cell_boxes[y].lo[sd] && x < y);
                       });
      const std::int32_t l = build(b, mid);
      const std::int32_t r = build(mid, e);
      gi.nodes[id].left = l;
      gi.nodes[id].right = r;
      return id;
    };
    build(0, gi.cells.size());
  }
  return gi;
}

// AABB descent: calls leaf_fn(cell) for every occupied leaf cell whose box
// passes `test`; stops early when leaf_fn returns true. Node boxes are exact
// unions of their leaf boxes, and both tests are monotone under box
// containment, so the descent equals a linear scan over occupied cells.
template <int D, class Test, class LeafFn>
bool descend(const GridIndex<D>& gi, const Test& test, const LeafFn& leaf_fn) {
  if (gi.nodes.empty()) return false;
  std::vector<std::int32_t> stack;
  stack.push_back(0);
  while (!stack.empty()) {
    const auto& nd = gi.nodes[stack.back()];
    stack.pop_back();
    if (!test(nd.box)) continue;
    if (nd.leaf >= 0) {
      if (leaf_fn(nd.leaf)) return true;
      continue;
    }
    stack.push_back(nd.right);
    stack.push_back(nd.left);
  }
  return false;
}

// ---------------------------------------------------------------------------
// find_border
// ---------------------------------------------------------------------------
struct PartialsView {
  std::uint32_t k;
  const std::uint64_t* offsets;  // k+1
  const std::uint32_t* verts;    // (D+1) x S vertex-major
  const std::uint32_t* nbrs;     // (D+1) x S, local to the part
  const std::int8_t* parity;
  std::uint64_t S;
};

struct BorderResult {
  std::vector<std::uint8_t> positive;  // full scan (north_star semantics)
  std::vector<std::uint8_t> border;    // hull-seeded BFS (SPEC find_border semantics)
  std::vector<std::uint32_t> vertices_positive;  // sorted unique finite vertices of positive
  std::vector<std::uint32_t> vertices_border;    // sorted unique finite vertices of border
};

template <int D, class Prims>
class BorderOracle {
 public:
  // grid_bbox (lo[D], hi[D]) / n_total: the top level's grid at a recursion
  // level (nullptr / 0: the bbox and count of all n points); points labelled
  // kInf belong to no index of this level.
  BorderOracle(const double* xyz, std::size_t n, const std::uint32_t* labels, const PartialsView& pv,
               int policy, double c_G, unsigned threads, const double* grid_bbox = nullptr, std::size_t n_total = 0)
      : xyz_(xyz), n_(n), pv_(pv), policy_(policy), threads_(threads) {
    g_ = grid_bbox ? grid_from_bbox<D>(grid_bbox, grid_bbox + D, n_total ? n_total : n, c_G)
                   : (n_total ? grid_from_bbox_of<D>(xyz, n, n_total, c_G) : grid_params<D>(xyz, n, c_G));
    std::vector<std::vector<std::uint32_t>> parts(pv.k);
    for (std::size_t i = 0; i < n; ++i)
      if (labels[i] != kInf) parts[labels[i]].push_back(static_cast<std::uint32_t>(i));
    idx_.resize(pv.k);
    parallel_for(pv.k, 1, threads, [&](std::size_t b, std::size_t e) {
      for (std::size_t p = b; p < e; ++p) idx_[p] = build_grid_index<D>(g_, xyz, parts[p].data(), parts[p].size());
    });
  }

  const GridParams<D>& params() const { return g_; }
  const GridIndex<D>& index(std::uint32_t p) const { return idx_[p]; }

  const double* P(std::uint32_t v) const { return xyz_ + std::size_t(v) * D; }
  std::uint32_t vert(std::uint64_t s, int j) const { return pv_.verts[std::uint64_t(j) * pv_.S + s]; }
  std::uint32_t nbr(std::uint64_t s, int j) const { return pv_.nbrs[std::uint64_t(j) * pv_.S + s]; }

  // Positive test of simplex s (global row) of part i against every j != i.
  bool positive(std::uint64_t s, std::uint32_t i) const {
    const bool infinite = vert(s, D) == kInf;
    if (!infinite) {
      const double* p[D + 1];
      for (int j = 0; j <= D; ++j) p[j] = P(vert(s, j));
      const Sphere<D> sph = Prims::sphere(p);
      const int par = pv_.parity[s];
      for (std::uint32_t j = 0; j < pv_.k; ++j) {
        if (j == i || idx_[j].empty()) continue;
        if (policy_ == kBbox) {
          if (Prims::box_sphere(idx_[j].bbox_policy_box(), sph)) return true;
          continue;
        }
        auto test = [&](const Box<D>& b) { return Prims::box_sphere(b, sph); };
        if (policy_ == kGrid) {
          if (descend<D>(idx_[j], test, [](std::int32_t) { return true; })) return true;
        } else {
          const GridIndex<D>& gi = idx_[j];
          if (descend<D>(gi, test, [&](std::int32_t c) {
                for (std::uint32_t t = gi.cell_start[c]; t < gi.cell_start[c + 1]; ++t)
                  if (Prims::in_sphere_or(p, par, P(gi.points[t])) > 0) return true;
                return false;
              }))
            return true;
        }
      }
      return false;
    }
    // infinite simplex: outer halfspace of the hull facet
    const double* facet[D];
    for (int j = 0; j < D; ++j) facet[j] = P(vert(s, j));
    const std::uint64_t owner = pv_.offsets[i] + nbr(s, D);
    std::uint32_t inner = kInf;
    for (int a = 0; a <= D; ++a) {
      const std::uint32_t v = vert(owner, a);
      bool on = false;
      for (int f = 0; f < D; ++f) on |= (vert(s, f) == v);
      if (!on) {
        inner = v;
        break;
      }
    }
    const double* ip = P(inner);
    for (std::uint32_t j = 0; j < pv_.k; ++j) {
      if (j == i || idx_[j].empty()) continue;
      if (policy_ == kBbox) {
        if (Prims::halfspace_box(facet, ip, idx_[j].bbox_policy_box())) return true;
        continue;
      }
      auto test = [&](const Box<D>& b) { return Prims::halfspace_box(facet, ip, b); };
      if (policy_ == kGrid) {
        if (descend<D>(idx_[j], test, [](std::int32_t) { return true; })) return true;
      } else {
        const GridIndex<D>& gi = idx_[j];
        const double* pts[D + 1];
        for (int a = 0; a < D; ++a) pts[a] = facet[a];
        pts[D] = ip;
        const int inner_sign = Prims::orient_pts(pts);
        if (descend<D>(gi, test, [&](std::int32_t c) {
              for (std::uint32_t t = gi.cell_start[c]; t < gi.cell_start[c + 1]; ++t) {
                pts[D] = P(gi.points[t]);
                const int o = Prims::orient_pts(pts);
                if (o != 0 && o != inner_sign) return true;
              }
              return false;
            }))
          return true;
      }
    }
    return false;
  }

  // Full scan + BFS over parts [p0, p1) (all parts by default).
  BorderResult run(std::uint32_t p0, std::uint32_t p1, bool with_bfs = true) const {
    BorderResult r;
    r.positive.assign(pv_.S, 0);
    r.border.assign(pv_.S, 0);
    parallel_for(p1 - p0, 1, threads_, [&](std::size_t b, std::size_t e) {
      for (std::size_t q = b; q < e; ++q) {
        const std::uint32_t i = static_cast<std::uint32_t>(p0 + q);
        for (std::uint64_t s = pv_.offsets[i]; s < pv_.offsets[i + 1]; ++s) r.positive[s] = positive(s, i) ? 1 : 0;
        if (with_bfs) bfs(i, r.positive, r.border);
      }
    });
    r.vertices_positive = collect(r.positive, p0, p1);
    r.vertices_border = collect(r.border, p0, p1);
    return r;
  }

  // SPEC find_border BFS (Alg. 1): seeds = hull_simplices (triangulation.cpp:34-53);
  // a dequeued positive simplex joins the border and enqueues unmarked neighbors.
  void bfs(std::uint32_t i, const std::vector<std::uint8_t>& positive, std::vector<std::uint8_t>& border) const {
    const std::uint64_t off = pv_.offsets[i], cnt = pv_.offsets[i + 1] - off;
    std::vector<std::uint8_t> mark(cnt, 0);
    std::vector<std::uint32_t> queue;
    for (std::uint64_t l = 0; l < cnt; ++l) {
      const std::uint64_t s = off + l;
      bool hull = vert(s, D) == kInf;
      if (!hull)
        for (int d = 0; d <= D && !hull; ++d) hull = vert(off + nbr(s, d), D) == kInf;
      if (hull) {
        mark[l] = 1;
        queue.push_back(static_cast<std::uint32_t>(l));
      }
    }
    for (std::size_t h = 0; h < queue.size(); ++h) {
      const std::uint32_t l = queue[h];
      if (!positive[off + l]) continue;
      border[off + l] = 1;
      for (int d = 0; d <= D; ++d) {
        const std::uint32_t nb = nbr(off + l, d);
        if (!mark[nb]) {
          mark[nb] = 1;
          queue.push_back(nb);
        }
      }
    }
  }

  std::vector<std::uint32_t> collect(const std::vector<std::uint8_t>& flags, std::uint32_t p0,
                                     std::uint32_t p1) const {
    std::vector<std::uint8_t> mark(n_, 0);
    for (std::uint64_t s = pv_.offsets[p0]; s < pv_.offsets[p1]; ++s) {
      if (!flags[s]) continue;
      for (int j = 0; j <= D; ++j) {
        const std::uint32_t v = vert(s, j);
        if (v != kInf) mark[v] = 1;
      }
    }
    std::vector<std::uint32_t> out;
    for (std::size_t v = 0; v < n_; ++v)
      if (mark[v]) out.push_back(static_cast<std::uint32_t>(v));
    return out;
  }

  // Circumsphere (inflated) of a finite simplex, for the 1e-12 centre/radius check.
  Sphere<D> sphere_of(std::uint64_t s) const {
    const double* p[D + 1];
    for (int j = 0; j <= D; ++j) p[j] = P(vert(s, j));
    return Prims::sphere(p);
  }

 private:
  const double* xyz_;
  std::size_t n_;
  PartialsView pv_;
  int policy_;
  unsigned threads_;
  GridParams<D> g_;
  std::vector<GridIndex<D>> idx_;
};

}  // namespace sbdt_oracle
