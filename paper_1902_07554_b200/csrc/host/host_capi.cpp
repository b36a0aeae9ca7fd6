// C ABI of the host setup library (libsbdt_host.so), consumed by the
// Python driver (bench.py, tests) through ctypes. Setup only: nothing here
// is on the measured GPU path.
#include <cstdio>
#include <cstring>
#include <exception>

#include <vector>

#include "../common/predicates.hpp"
#include "rng.hpp"
#include "setup.hpp"

using namespace sbdt_host;

namespace {
void set_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) std::snprintf(err, errlen, "%s", msg);
}
}  // namespace

extern "C" {

// The shared predicates (csrc/common/predicates.hpp: binary64 filter, then
// expansion arithmetic or scaled big integers), host build, in the layout of
// sbdt_gpu_predicates: op 0 orient ((dim+1) points per case), op 1 in_sphere
// ((dim+1) simplex points then q). The same source the kernels compile; the
// tests pin it against the reference's compiled geometry.cpp on CPU.
int sbdt_host_predicates(int op, int dim, const double* pts, std::uint64_t count, std::int8_t* out) {
  if ((op != 0 && op != 1) || (dim != 2 && dim != 3)) return 1;
  std::vector<double> buf(op == 1 ? (dim == 3 ? sbdt_pred::kInSphere3Scratch : sbdt_pred::kInSphere2Scratch) : 1);
  for (std::uint64_t i = 0; i < count; ++i) {
    int r;
    if (op == 0) {
      const double* b = pts + i * (dim + 1) * dim;
      r = dim == 2 ? sbdt_pred::orient2(b, b + 2, b + 4) : sbdt_pred::orient3(b, b + 3, b + 6, b + 9);
    } else {
      const double* b = pts + i * (dim + 2) * dim;
      if (dim == 2) {
        r = sbdt_pred::in_sphere2_filtered(b, b + 2, b + 4, b + 6);
        if (r == 2) r = sbdt_pred::in_sphere2_exact_buf(b, b + 2, b + 4, b + 6, buf.data());
      } else {
        r = sbdt_pred::in_sphere3_filtered(b, b + 3, b + 6, b + 9, b + 12);
        if (r == 2) r = sbdt_pred::in_sphere3_exact_buf(b, b + 3, b + 6, b + 9, b + 12, buf.data());
      }
    }
    out[i] = static_cast<std::int8_t>(r);
  }
  return 0;
}

std::uint64_t sbdt_host_generate(int kind, int dim, std::uint64_t n, std::uint64_t seed,
                                 const double* params, int nparams, double* out) {
  try {
    auto v = generate(static_cast<Distribution>(kind), dim, n, seed, params, nparams);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return n;
  } catch (...) {
    return 0;
  }
}

std::uint64_t sbdt_host_deduplicate(int dim, double* coords, std::uint64_t n, std::uint32_t* remap) {
  std::vector<double> v(coords, coords + n * dim);
  auto r = deduplicate(dim, v);
  std::memcpy(coords, v.data(), v.size() * sizeof(double));
  if (remap) std::memcpy(remap, r.data(), r.size() * sizeof(std::uint32_t));
  return v.size() / dim;
}

int sbdt_host_draw_sample(std::uint64_t n, std::uint64_t m, std::uint64_t seed, std::uint32_t* out) {
  try {
    auto s = draw_sample(n, m, seed);
    std::memcpy(out, s.data(), s.size() * sizeof(std::uint32_t));
    return 0;
  } catch (...) {
    return 1;
  }
}

void* sbdt_host_triangulate(int dim, const double* coords, const std::uint32_t* ids, std::uint64_t n,
                            std::uint64_t seed, char* err, int errlen) {
  try {
    return new TriSoA(triangulate(dim, coords, ids, n, seed));
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}
std::uint64_t sbdt_host_tri_count(void* h) { return static_cast<TriSoA*>(h)->count; }
void sbdt_host_tri_export(void* h, std::uint32_t* verts, std::uint32_t* nbrs, std::int8_t* parity) {
  auto* t = static_cast<TriSoA*>(h);
  if (verts) std::memcpy(verts, t->verts.data(), t->verts.size() * 4);
  if (nbrs) std::memcpy(nbrs, t->nbrs.data(), t->nbrs.size() * 4);
  if (parity) std::memcpy(parity, t->parity.data(), t->parity.size());
}
void sbdt_host_tri_free(void* h) { delete static_cast<TriSoA*>(h); }

int sbdt_host_partition_sample(int dim, const double* coords, const std::uint32_t* sample_ids,
                               std::uint64_t m, std::uint32_t k, double eps, int weight_fn,
                               std::uint64_t seed, std::uint32_t* labels_out, std::uint64_t* cut_out,
                               char* err, int errlen) {
  try {
    TriSoA dt = triangulate(dim, coords, sample_ids, m, derive_seed(seed, kTagSampleDt));
    SampleGraph g = build_sample_graph(dim, coords, sample_ids, m, dt, static_cast<WeightFn>(weight_fn));
    auto labels = partition_graph(g, k, eps, seed);
    std::memcpy(labels_out, labels.data(), m * 4);
    if (cut_out) *cut_out = cut_weight(g, labels);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 1;
  }
}

// Graph-level API (tests of the partitioner contract).
int sbdt_host_partition_csr(std::uint64_t n, const std::uint32_t* xadj, const std::uint32_t* adj,
                            const std::int32_t* w, std::uint32_t k, double eps, std::uint64_t seed,
                            std::uint32_t* labels_out, std::uint64_t* cut_out, char* err, int errlen) {
  try {
    SampleGraph g;
    g.n = n;
    g.xadj.assign(xadj, xadj + n + 1);
    g.adj.assign(adj, adj + xadj[n]);
    g.w.assign(w, w + xadj[n]);
    auto labels = partition_graph(g, k, eps, seed);
    std::memcpy(labels_out, labels.data(), n * 4);
    if (cut_out) *cut_out = cut_weight(g, labels);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 1;
  }
}

void* sbdt_host_build_partials(int dim, const double* coords, std::uint64_t n, const std::uint32_t* labels,
                               std::uint32_t k, std::uint64_t seed, int threads, char* err, int errlen) {
  try {
    return new Partials(build_partials(dim, coords, n, labels, k, seed, threads < 0 ? 0 : threads));
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}
std::uint64_t sbdt_host_partials_total(void* h) { return static_cast<Partials*>(h)->total(); }
void sbdt_host_partials_export(void* h, std::uint64_t* offsets, std::uint32_t* verts, std::uint32_t* nbrs,
                               std::int8_t* parity) {
  auto* p = static_cast<Partials*>(h);
  if (offsets) std::memcpy(offsets, p->offsets.data(), p->offsets.size() * 8);
  if (verts) std::memcpy(verts, p->verts.data(), p->verts.size() * 4);
  if (nbrs) std::memcpy(nbrs, p->nbrs.data(), p->nbrs.size() * 4);
  if (parity) std::memcpy(parity, p->parity.data(), p->parity.size());
}
void sbdt_host_partials_free(void* h) { delete static_cast<Partials*>(h); }

}  // extern "C"
