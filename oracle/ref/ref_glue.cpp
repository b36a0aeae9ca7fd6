// TEST INFRASTRUCTURE — extern "C" glue over the REFERENCE's own compiled
// primitives (/root/reference/proj/src/{geometry,triangulation}.cpp and the
// F4-patched sequential_dt.cpp, compiled by path; see oracle/Makefile).
// Used only to pin the oracle's restatement (oracle/prims.hpp, path.hpp) and
// the host DT builder, and to generate tests/golden/ fixtures.
#include <algorithm>
#include <chrono>
#include <functional>
#include <array>
#include <cstring>
#include <numeric>
#include <vector>

#include "sbdt/geometry.hpp"
#include "sbdt/sequential_dt.hpp"
#include "sbdt/task_pool.hpp"
#include "sbdt/triangulation.hpp"
#include "../path.hpp"

namespace {

template <int D>
std::array<sbdt::Vec<D>, D + 1> to_arr(const double* const* p, int count) {
  std::array<sbdt::Vec<D>, D + 1> a{};
  for (int i = 0; i < count; ++i)
    for (int d = 0; d < D; ++d) a[i][d] = p[i][d];
  return a;
}
template <int D>
sbdt::Box<D> to_box(const sbdt_oracle::Box<D>& b) {
  sbdt::Box<D> r;
  for (int d = 0; d < D; ++d) r.lo[d] = b.lo[d], r.hi[d] = b.hi[d];
  return r;
}
template <int D>
sbdt::Sphere<D> to_sphere(const sbdt_oracle::Sphere<D>& s) {
  sbdt::Sphere<D> r;
  for (int d = 0; d < D; ++d) r.center[d] = s.center[d];
  r.radius_squared = s.radius_squared;
  return r;
}

// The path templates instantiated with the reference's primitives.
template <int D>
struct RefPrims {
  static sbdt_oracle::Sphere<D> sphere(const double* const* p) {
    const auto s = sbdt::inflated<D>(sbdt::circumsphere<D>(to_arr<D>(p, D + 1)));
    sbdt_oracle::Sphere<D> r;
    for (int d = 0; d < D; ++d) r.center[d] = s.center[d];
    r.radius_squared = s.radius_squared;
    return r;
  }
  static bool box_sphere(const sbdt_oracle::Box<D>& b, const sbdt_oracle::Sphere<D>& s) {
    return sbdt::box_sphere_overlap<D>(to_box<D>(b), to_sphere<D>(s));
  }
  static bool halfspace_box(const double* const* f, const double* inner, const sbdt_oracle::Box<D>& b) {
    std::array<sbdt::Vec<D>, D> facet;
    for (int i = 0; i < D; ++i)
      for (int d = 0; d < D; ++d) facet[i][d] = f[i][d];
    sbdt::Vec<D> in;
    for (int d = 0; d < D; ++d) in[d] = inner[d];
    return sbdt::halfspace_box_overlap<D>(facet, in, to_box<D>(b));
  }
  static int orient_pts(const double* const* p) { return sbdt::orient<D>(to_arr<D>(p, D + 1)); }
  static int in_sphere_or(const double* const* p, int parity, const double* q) {
    sbdt::Vec<D> qq;
    for (int d = 0; d < D; ++d) qq[d] = q[d];
    return sbdt::in_sphere_oriented<D>(to_arr<D>(p, D + 1), parity, qq);
  }
  static double sqdist(const double* a, const double* b) {
    sbdt::Vec<D> x, y;
    for (int d = 0; d < D; ++d) x[d] = a[d], y[d] = b[d];
    return sbdt::squared_distance<D>(x, y);
  }
};

struct RefTri {
  int dim;
  std::vector<std::uint32_t> verts, nbrs;  // vertex-major, compacted
  std::vector<std::int8_t> parity;
  std::uint64_t count = 0;
};

template <int D>
RefTri run_ref_dt(const double* xyz, std::uint64_t n_points, const std::uint32_t* ids, std::uint64_t n,
                  std::uint64_t seed) {
  sbdt::PointSet ps(D);
  for (std::uint64_t i = 0; i < n_points; ++i) ps.add(xyz + i * D);
  std::vector<sbdt::PointId> v(ids, ids + n);
  auto t = sbdt::triangulate_seq<D>(ps, v, seed);
  t.compact();
  RefTri r;
  r.dim = D;
  const auto& raw = t.raw_simplices();
  r.count = raw.size();
  r.verts.resize((D + 1) * r.count);
  r.nbrs.resize((D + 1) * r.count);
  r.parity.resize(r.count);
  for (std::uint64_t s = 0; s < r.count; ++s) {
    for (int j = 0; j <= D; ++j) {
      r.verts[j * r.count + s] = raw[s].vertices[j];
      r.nbrs[j * r.count + s] = raw[s].neighbors[j];
    }
    r.parity[s] = raw[s].parity;
  }
  return r;
}

// The reference's own work pool (task_pool.hpp:63-80) behind path.hpp's
// parallel_for: fixed-grain chunks, so the outputs equal the oracle's.
sbdt::TaskPool* g_pool = nullptr;
void pool_runner(std::size_t n, std::size_t grain, const std::function<void(std::size_t, std::size_t)>& fn) {
  g_pool->parallel_for(n, grain, fn);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <int D>
void time_step(const double* xyz, std::uint64_t n, const std::uint32_t* sample_ids, std::uint64_t m,
               const std::uint32_t* sample_labels, std::uint64_t n_assign, const std::uint32_t* labels,
               const sbdt_oracle::PartialsView& pv, int policy, double c_G, unsigned threads, std::uint32_t p0,
               std::uint32_t p1, std::uint32_t* labels_out, std::uint8_t* positive_out, double* times,
               std::uint64_t* n_vb) {
  const double t0 = now_s();
  sbdt_oracle::SampleKdTree<D, RefPrims<D>> tree(xyz, sample_ids, m, sample_labels);
  sbdt_oracle::parallel_for(n_assign, 4096, threads, [&](std::size_t b, std::size_t e) {
    for (std::size_t i = b; i < e; ++i) labels_out[i] = tree.nearest_label(xyz + i * D);
  });
  const double t1 = now_s();
  sbdt_oracle::BorderOracle<D, RefPrims<D>> bo(xyz, n, labels, pv, policy, c_G, threads);
  const double t2 = now_s();
  auto r = bo.run(p0, p1);
  const double t3 = now_s();
  times[0] = t1 - t0, times[1] = t2 - t1, times[2] = t3 - t2;
  *n_vb = r.vertices_border.size();
  if (positive_out) std::memcpy(positive_out + pv.offsets[p0], r.positive.data() + pv.offsets[p0],
                                pv.offsets[p1] - pv.offsets[p0]);
}

}  // namespace

extern "C" {

// One timed CPU step of the path on the REFERENCE's primitives (geometry.cpp,
// compiled by path) and the reference's TaskPool(threads) (threads <= 1: the
// inline determinism baseline, task_pool.hpp:20-21): kd-tree assign_points
// over points [0, n_assign) -> labels_out, then find_border
// (per-part GridIndex build + full scan + BFS) over
// parts [p0, p1) with the given labels. times: [assign, index build, border].
int ref_time_step(int dim, const double* xyz, std::uint64_t n, const std::uint32_t* sample_ids, std::uint64_t m,
                  const std::uint32_t* sample_labels, std::uint64_t n_assign, const std::uint32_t* labels,
                  std::uint32_t k, const std::uint64_t* offsets, const std::uint32_t* verts,
                  const std::uint32_t* nbrs, const std::int8_t* parity, int policy, double c_G, unsigned threads,
                  std::uint32_t p0, std::uint32_t p1, std::uint32_t* labels_out, std::uint8_t* positive_out,
                  double* times, std::uint64_t* n_vb) {
  try {
    sbdt_oracle::PartialsView pv{k, offsets, verts, nbrs, parity, offsets[k]};
    if (p1 == 0 || p1 > k) p1 = k;
    sbdt::TaskPool pool(threads);
    g_pool = &pool;
    sbdt_oracle::g_runner = threads > 1 ? pool_runner : nullptr;
    if (dim == 2)
      time_step<2>(xyz, n, sample_ids, m, sample_labels, n_assign, labels, pv, policy, c_G, threads, p0, p1,
                   labels_out, positive_out, times, n_vb);
    else
      time_step<3>(xyz, n, sample_ids, m, sample_labels, n_assign, labels, pv, policy, c_G, threads, p0, p1,
                   labels_out, positive_out, times, n_vb);
    sbdt_oracle::g_runner = nullptr;
    g_pool = nullptr;
    return 0;
  } catch (...) {
    sbdt_oracle::g_runner = nullptr;
    g_pool = nullptr;
    return 1;
  }
}

int ref_orient(int dim, const double* pts) {
  if (dim == 2) return sbdt::orient2({pts[0], pts[1]}, {pts[2], pts[3]}, {pts[4], pts[5]});
  return sbdt::orient3({pts[0], pts[1], pts[2]}, {pts[3], pts[4], pts[5]}, {pts[6], pts[7], pts[8]},
                       {pts[9], pts[10], pts[11]});
}
int ref_in_sphere(int dim, const double* p, const double* q) {
  if (dim == 2) return sbdt::in_sphere2({p[0], p[1]}, {p[2], p[3]}, {p[4], p[5]}, {q[0], q[1]});
  return sbdt::in_sphere3({p[0], p[1], p[2]}, {p[3], p[4], p[5]}, {p[6], p[7], p[8]}, {p[9], p[10], p[11]},
                          {q[0], q[1], q[2]});
}
// Batches in the layout of sbdt_gpu_predicates: per case (dim+1) points for
// orient, (dim+1) simplex points then q for in_sphere.
void ref_orient_batch(int dim, const double* pts, std::uint64_t count, std::int8_t* out) {
  const std::uint64_t per = std::uint64_t(dim + 1) * dim;
  for (std::uint64_t i = 0; i < count; ++i) out[i] = static_cast<std::int8_t>(ref_orient(dim, pts + i * per));
}
void ref_in_sphere_batch(int dim, const double* pts, std::uint64_t count, std::int8_t* out) {
  const std::uint64_t per = std::uint64_t(dim + 2) * dim;
  for (std::uint64_t i = 0; i < count; ++i) {
    const double* b = pts + i * per;
    out[i] = static_cast<std::int8_t>(ref_in_sphere(dim, b, b + std::uint64_t(dim + 1) * dim));
  }
}

int ref_circumsphere(int dim, const double* pts, double* out) {
  try {
    if (dim == 2) {
      auto s = sbdt::circumsphere<2>({sbdt::Vec<2>{pts[0], pts[1]}, sbdt::Vec<2>{pts[2], pts[3]},
                                      sbdt::Vec<2>{pts[4], pts[5]}});
      out[0] = s.center[0], out[1] = s.center[1], out[2] = s.radius_squared;
    } else {
      auto s = sbdt::circumsphere<3>({sbdt::Vec<3>{pts[0], pts[1], pts[2]}, sbdt::Vec<3>{pts[3], pts[4], pts[5]},
                                      sbdt::Vec<3>{pts[6], pts[7], pts[8]}, sbdt::Vec<3>{pts[9], pts[10], pts[11]}});
      out[0] = s.center[0], out[1] = s.center[1], out[2] = s.center[2], out[3] = s.radius_squared;
    }
    return 0;
  } catch (const sbdt::DegenerateSimplex&) {
    return 1;
  }
}
double ref_inflate(double r2) {
  sbdt::Sphere<2> s{{0, 0}, r2};
  return sbdt::inflated<2>(s).radius_squared;
}
int ref_box_sphere(int dim, const double* lo, const double* hi, const double* c, double r2) {
  if (dim == 2)
    return sbdt::box_sphere_overlap<2>(sbdt::Box<2>{{lo[0], lo[1]}, {hi[0], hi[1]}}, sbdt::Sphere<2>{{c[0], c[1]}, r2});
  return sbdt::box_sphere_overlap<3>(sbdt::Box<3>{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}},
                                     sbdt::Sphere<3>{{c[0], c[1], c[2]}, r2});
}
int ref_halfspace_box(int dim, const double* f, const double* inner, const double* lo, const double* hi) {
  if (dim == 2)
    return sbdt::halfspace_box_overlap<2>({sbdt::Vec<2>{f[0], f[1]}, sbdt::Vec<2>{f[2], f[3]}}, {inner[0], inner[1]},
                                          sbdt::Box<2>{{lo[0], lo[1]}, {hi[0], hi[1]}});
  return sbdt::halfspace_box_overlap<3>(
      {sbdt::Vec<3>{f[0], f[1], f[2]}, sbdt::Vec<3>{f[3], f[4], f[5]}, sbdt::Vec<3>{f[6], f[7], f[8]}},
      {inner[0], inner[1], inner[2]}, sbdt::Box<3>{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
}

void* ref_triangulate(int dim, const double* xyz, std::uint64_t n_points, const std::uint32_t* ids, std::uint64_t n,
                      std::uint64_t seed) {
  try {
    if (dim == 2) return new RefTri(run_ref_dt<2>(xyz, n_points, ids, n, seed));
    return new RefTri(run_ref_dt<3>(xyz, n_points, ids, n, seed));
  } catch (...) {
    return nullptr;
  }
}
std::uint64_t ref_tri_count(void* h) { return static_cast<RefTri*>(h)->count; }
void ref_tri_export(void* h, std::uint32_t* verts, std::uint32_t* nbrs, std::int8_t* parity) {
  auto* t = static_cast<RefTri*>(h);
  if (verts) std::memcpy(verts, t->verts.data(), t->verts.size() * 4);
  if (nbrs) std::memcpy(nbrs, t->nbrs.data(), t->nbrs.size() * 4);
  if (parity) std::memcpy(parity, t->parity.data(), t->parity.size());
}
void ref_tri_free(void* h) { delete static_cast<RefTri*>(h); }

int ref_assign_brute(int dim, const double* xyz, std::uint64_t n, const std::uint32_t* sample_ids, std::uint64_t m,
                     const std::uint32_t* sample_labels, std::uint32_t* labels) {
  if (dim == 2) sbdt_oracle::assign_brute<2, RefPrims<2>>(xyz, n, sample_ids, m, sample_labels, labels, 8);
  else sbdt_oracle::assign_brute<3, RefPrims<3>>(xyz, n, sample_ids, m, sample_labels, labels, 8);
  return 0;
}

int ref_find_border(int dim, const double* xyz, std::uint64_t n, const std::uint32_t* labels, std::uint32_t k,
                    const std::uint64_t* offsets, const std::uint32_t* verts, const std::uint32_t* nbrs,
                    const std::int8_t* parity, int policy, double c_G, std::uint8_t* positive_out,
                    std::uint8_t* border_out, std::uint32_t* vpos, std::uint64_t* n_vpos, std::uint32_t* vbfs,
                    std::uint64_t* n_vbfs) {
  sbdt_oracle::PartialsView pv{k, offsets, verts, nbrs, parity, offsets[k]};
  auto go = [&](auto bo) {
    auto r = bo.run(0, k);
    std::memcpy(positive_out, r.positive.data(), pv.S);
    std::memcpy(border_out, r.border.data(), pv.S);
    *n_vpos = r.vertices_positive.size();
    *n_vbfs = r.vertices_border.size();
    if (vpos) std::memcpy(vpos, r.vertices_positive.data(), r.vertices_positive.size() * 4);
    if (vbfs) std::memcpy(vbfs, r.vertices_border.data(), r.vertices_border.size() * 4);
  };
  if (dim == 2) go(sbdt_oracle::BorderOracle<2, RefPrims<2>>(xyz, n, labels, pv, policy, c_G, 8));
  else go(sbdt_oracle::BorderOracle<3, RefPrims<3>>(xyz, n, labels, pv, policy, c_G, 8));
  return 0;
}

}  // extern "C"
