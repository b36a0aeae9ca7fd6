// TEST INFRASTRUCTURE — C ABI of the CPU oracle (liboracle.so), for tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
// This library is the CHECKER: the product path never loads it.
#include <chrono>
#include <cstdio>
#include <type_traits>
#include <cstring>
#include <exception>

#include "merge.hpp"
#include "path.hpp"

using namespace sbdt_oracle;

namespace {
template <int D>
void export_border(const BorderOracle<D, OwnPrims<D>>& bo, const BorderResult& r, std::uint8_t* positive_out,
                   std::uint8_t* border_out, std::uint32_t* vpos_out, std::uint64_t* n_vpos,
                   std::uint32_t* vbfs_out, std::uint64_t* n_vbfs, double* spheres_out, std::uint64_t S,
                   const std::uint32_t* verts) {
  if (positive_out) std::memcpy(positive_out, r.positive.data(), S);
  if (border_out) std::memcpy(border_out, r.border.data(), S);
  if (n_vpos) *n_vpos = r.vertices_positive.size();
  if (n_vbfs) *n_vbfs = r.vertices_border.size();
  if (vpos_out) std::memcpy(vpos_out, r.vertices_positive.data(), r.vertices_positive.size() * 4);
  if (vbfs_out) std::memcpy(vbfs_out, r.vertices_border.data(), r.vertices_border.size() * 4);
  if (spheres_out) {
    for (std::uint64_t s = 0; s < S; ++s) {
      double* o = spheres_out + s * (D + 1);
      if (verts[std::uint64_t(D) * S + s] == kInf) {
        for (int d = 0; d <= D; ++d) o[d] = 0.0;
        continue;
      }
      const auto sp = bo.sphere_of(s);
      for (int d = 0; d < D; ++d) o[d] = sp.center[d];
      o[D] = sp.radius_squared;
    }
  }
}
}  // namespace

extern "C" {

const char* oracle_version() { return "sbdt-oracle 1 (restatement of SPEC.md assign_points/find_border)"; }

int oracle_assign_brute(int dim, const double* xyz, std::uint64_t n, const std::uint32_t* sample_ids,
                        std::uint64_t m, const std::uint32_t* sample_labels, std::uint32_t* labels, int threads) {
  if (dim == 2) assign_brute<2, OwnPrims<2>>(xyz, n, sample_ids, m, sample_labels, labels, threads);
  else if (dim == 3) assign_brute<3, OwnPrims<3>>(xyz, n, sample_ids, m, sample_labels, labels, threads);
  else return 1;
  return 0;
}

int oracle_assign_kdtree(int dim, const double* xyz, std::uint64_t n, const std::uint32_t* sample_ids,
                         std::uint64_t m, const std::uint32_t* sample_labels, std::uint32_t* labels,
                         int threads) {
  if (dim == 2) assign_kdtree<2, OwnPrims<2>>(xyz, n, sample_ids, m, sample_labels, labels, threads);
  else if (dim == 3) assign_kdtree<3, OwnPrims<3>>(xyz, n, sample_ids, m, sample_labels, labels, threads);
  else return 1;
  return 0;
}

// Assign only the points [begin, end) of xyz (bounded CPU-baseline sample);
// the kd-tree is built over the full sample.
int oracle_assign_kdtree_range(int dim, const double* xyz, std::uint64_t begin, std::uint64_t end,
                               const std::uint32_t* sample_ids, std::uint64_t m,
                               const std::uint32_t* sample_labels, std::uint32_t* labels, int threads) {
  if (dim == 2) {
    SampleKdTree<2, OwnPrims<2>> tree(xyz, sample_ids, m, sample_labels);
    parallel_for(end - begin, 4096, threads, [&](std::size_t b, std::size_t e) {
      for (std::size_t i = b; i < e; ++i) labels[i] = tree.nearest_label(xyz + (begin + i) * 2);
    });
  } else if (dim == 3) {
    SampleKdTree<3, OwnPrims<3>> tree(xyz, sample_ids, m, sample_labels);
    parallel_for(end - begin, 4096, threads, [&](std::size_t b, std::size_t e) {
      for (std::size_t i = b; i < e; ++i) labels[i] = tree.nearest_label(xyz + (begin + i) * 3);
    });
  } else {
    return 1;
  }
  return 0;
}

int oracle_grid_params(int dim, const double* xyz, std::uint64_t n, double c_G, double* lo, double* hi,
                       double* edge, std::int64_t* dims) {
  if (dim == 2) {
    auto g = grid_params<2>(xyz, n, c_G);
    for (int d = 0; d < 2; ++d) lo[d] = g.lo[d], hi[d] = g.hi[d], dims[d] = g.dims[d];
    *edge = g.edge;
  } else if (dim == 3) {
    auto g = grid_params<3>(xyz, n, c_G);
    for (int d = 0; d < 3; ++d) lo[d] = g.lo[d], hi[d] = g.hi[d], dims[d] = g.dims[d];
    *edge = g.edge;
  } else {
    return 1;
  }
  return 0;
}

// find_border over parts [p0, p1) (p1 = 0 means all parts).
int oracle_find_border(int dim, const double* xyz, std::uint64_t n, const std::uint32_t* labels, std::uint32_t k,
                       const std::uint64_t* offsets, const std::uint32_t* verts, const std::uint32_t* nbrs,
                       const std::int8_t* parity, int policy, double c_G, int threads, std::uint32_t p0,
                       std::uint32_t p1, std::uint8_t* positive_out, std::uint8_t* border_out,
                       std::uint32_t* vpos_out, std::uint64_t* n_vpos, std::uint32_t* vbfs_out,
                       std::uint64_t* n_vbfs, double* spheres_out, double* times_out, const double* grid_bbox,
                       std::uint64_t n_total, char* err, int errlen) {
  try {
    PartialsView pv{k, offsets, verts, nbrs, parity, offsets[k]};
    if (p1 == 0) p1 = k;
    auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    auto go = [&](auto tag) {
      constexpr int D = decltype(tag)::value;
      const double t0 = now();
      BorderOracle<D, OwnPrims<D>> bo(xyz, n, labels, pv, policy, c_G, threads, grid_bbox, n_total);
      const double t1 = now();
      auto r = bo.run(p0, p1);
      const double t2 = now();
      // times_out: [index build (per-part GridIndex), full scan + BFS + vertex sets]
      if (times_out) times_out[0] = t1 - t0, times_out[1] = t2 - t1;
      export_border<D>(bo, r, positive_out, border_out, vpos_out, n_vpos, vbfs_out, n_vbfs, spheres_out, pv.S, verts);
    };
    if (dim == 2) go(std::integral_constant<int, 2>{});
    else if (dim == 3) go(std::integral_constant<int, 3>{});
    else return 1;
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen > 0) std::snprintf(err, errlen, "%s", e.what());
    return 2;
  }
}

// Split timing of the oracle (bench cpu_baseline): index build vs find_border
// over parts [p0,p1); returns seconds via out params.
int oracle_time_border(int dim, const double* xyz, std::uint64_t n, const std::uint32_t* labels, std::uint32_t k,
                       const std::uint64_t* offsets, const std::uint32_t* verts, const std::uint32_t* nbrs,
                       const std::int8_t* parity, int policy, double c_G, int threads, std::uint32_t p0,
                       std::uint32_t p1, int reps, double* t_build, double* t_border, std::uint64_t* n_border_vertices) {
  PartialsView pv{k, offsets, verts, nbrs, parity, offsets[k]};
  auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  auto go = [&](auto tag) {
    constexpr int D = decltype(tag)::value;
    const double t0 = now();
    BorderOracle<D, OwnPrims<D>> bo(xyz, n, labels, pv, policy, c_G, threads);
    const double t1 = now();
    *t_build = t1 - t0;
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
      const double a = now();
      auto res = bo.run(p0, p1);
      const double b = now();
      best = std::min(best, b - a);
      *n_border_vertices = res.vertices_border.size();
    }
    *t_border = best;
  };
  if (dim == 2) go(std::integral_constant<int, 2>{});
  else if (dim == 3) go(std::integral_constant<int, 3>{});
  else return 1;
  return 0;
}

// Primitive entry points (pinned against oracle/_ref and golden vectors).
int oracle_orient(int dim, const double* pts) {
  const double* p[4] = {pts, pts + dim, pts + 2 * dim, pts + 3 * dim};
  return dim == 2 ? orient<2>(p) : orient<3>(p);
}
int oracle_in_sphere(int dim, const double* pts, const double* q) {
  if (dim == 2) return in_sphere2(pts, pts + 2, pts + 4, q);
  return in_sphere3(pts, pts + 3, pts + 6, pts + 9, q);
}
// Batches in the layout of sbdt_gpu_predicates (see ref_orient_batch).
void oracle_orient_batch(int dim, const double* pts, std::uint64_t count, std::int8_t* out) {
  const std::uint64_t per = std::uint64_t(dim + 1) * dim;
  for (std::uint64_t i = 0; i < count; ++i) out[i] = static_cast<std::int8_t>(oracle_orient(dim, pts + i * per));
}
void oracle_in_sphere_batch(int dim, const double* pts, std::uint64_t count, std::int8_t* out) {
  const std::uint64_t per = std::uint64_t(dim + 2) * dim;
  for (std::uint64_t i = 0; i < count; ++i) {
    const double* b = pts + i * per;
    out[i] = static_cast<std::int8_t>(oracle_in_sphere(dim, b, b + std::uint64_t(dim + 1) * dim));
  }
}

int oracle_circumsphere(int dim, const double* pts, double* out) {
  try {
    const double* p[4] = {pts, pts + dim, pts + 2 * dim, pts + 3 * dim};
    if (dim == 2) {
      auto s = circumsphere<2>(p);
      out[0] = s.center[0], out[1] = s.center[1], out[2] = s.radius_squared;
    } else {
      auto s = circumsphere<3>(p);
      out[0] = s.center[0], out[1] = s.center[1], out[2] = s.center[2], out[3] = s.radius_squared;
    }
    return 0;
  } catch (const DegenerateSimplex&) {
    return 1;
  }
}
int oracle_box_sphere(int dim, const double* lo, const double* hi, const double* center, double r2) {
  if (dim == 2) {
    Box<2> b{{lo[0], lo[1]}, {hi[0], hi[1]}};
    return box_sphere_overlap<2>(b, Sphere<2>{{center[0], center[1]}, r2});
  }
  Box<3> b{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
  return box_sphere_overlap<3>(b, Sphere<3>{{center[0], center[1], center[2]}, r2});
}
int oracle_halfspace_box(int dim, const double* facet, const double* inner, const double* lo, const double* hi) {
  if (dim == 2) {
    const double* f[2] = {facet, facet + 2};
    return halfspace_box_overlap<2>(f, inner, Box<2>{{lo[0], lo[1]}, {hi[0], hi[1]}});
  }
  const double* f[3] = {facet, facet + 3, facet + 6};
  return halfspace_box_overlap<3>(f, inner, Box<3>{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
}

// merge + update_neighbors (oracle/merge.hpp). Returns a handle (nullptr on
// error, message in err); rows / export / free below.
void* oracle_merge(int dim, std::uint32_t k, const std::uint64_t* offsets, const std::uint32_t* verts,
                   const std::uint32_t* nbrs, const std::int8_t* parity, const std::uint8_t* border,
                   const std::uint32_t* tb_verts, const std::uint32_t* tb_nbrs, const std::int8_t* tb_parity,
                   std::uint64_t SB, const std::uint32_t* labels, int hull, char* err, int errlen) {
  try {
    MergeOut r = dim == 2 ? merge_oracle<2>(k, offsets, verts, nbrs, parity, border, tb_verts, tb_nbrs, tb_parity,
                                            SB, labels, hull != 0)
                          : merge_oracle<3>(k, offsets, verts, nbrs, parity, border, tb_verts, tb_nbrs, tb_parity,
                                            SB, labels, hull != 0);
    if (!r.error.empty()) {
      if (err && errlen > 0) std::snprintf(err, errlen, "%s", r.error.c_str());
      return nullptr;
    }
    return new MergeOut(std::move(r));
  } catch (const std::exception& e) {
    if (err && errlen > 0) std::snprintf(err, errlen, "%s", e.what());
    return nullptr;
  }
}
std::uint64_t oracle_merge_rows(void* h) { return static_cast<MergeOut*>(h)->rows; }
void oracle_merge_export(void* h, std::uint32_t* verts, std::uint32_t* nbrs, std::int8_t* parity,
                         std::uint64_t* offsets) {
  const MergeOut* r = static_cast<MergeOut*>(h);
  std::memcpy(verts, r->verts.data(), r->verts.size() * 4);
  std::memcpy(nbrs, r->nbrs.data(), r->nbrs.size() * 4);
  std::memcpy(parity, r->parity.data(), r->parity.size());
  std::memcpy(offsets, r->offsets.data(), r->offsets.size() * 8);
}
void oracle_merge_free(void* h) { delete static_cast<MergeOut*>(h); }

}  // extern "C"
