// K4-K9 — border-simplex detection (
// PAPER.md Alg. 1 border block, §3.2 primitives) on sm_100a.
//
// K4  owner grid: one uint16 code per cell of the global uniform grid
//     (SPEC.md:396-417 GridIndex, all partitions at once): EMPTY, a single
//     owning partition p, or MULTI. A pyramid of coarser levels (64 children
//     per block: 4x4x4 in 3D, 8x8 in 2D) stores the same code per block.
//     "some occupied cell of partition j != i overlaps X" is then
//     "some cell with code not in {EMPTY, i} overlaps X" — the SPEC's
//     exists-j loop without iterating j.
// K5  finite simplices: circumsphere in binary64 with the reference's exact
//     operation order (geometry.cpp:298-327 / :279-296), inflated
//     (geometry.hpp:179-183), then a pyramid descent with box_sphere_overlap
//     (geometry.hpp:187-201). Pruning is exact: block boxes are exact unions of
//     their cells' boxes and the test is monotone under containment in
//     binary64, so the result equals a linear scan over occupied cells.
// K6  infinite simplices: halfspace_box_overlap (geometry.cpp:329-345) with
//     exact orientation (filtered + expansion arithmetic), same descent.
// K9  border vertices: positive simplices flag their finite vertices; a
//     two-pass ballot/prefix-sum compaction emits the sorted, deduplicated
//     border-vertex ids.
#include <cuda_runtime.h>

#include "common.cuh"
#include "context.cuh"
#include "scan.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {

constexpr int kBThreads = 256;

template <int D>
struct OwnerGrid {
  Grid<D> g;
  double inv_edge;
  double margin;
  int levels;  // number of levels incl. leaf level 0; top level has one block
  int shift;   // log2 of per-axis fanout
  int ldims[kMaxLevels][D];
  unsigned long long loff[kMaxLevels + 1];
};

template <int D>
constexpr int fan_shift() {
  return D == 3 ? 2 : 3;  // 64 children per block
}

template <int D>
__device__ __forceinline__ unsigned long long lin(const int* dims, const int* c) {
  unsigned long long id = static_cast<unsigned>(c[D - 1]);
#pragma unroll
  for (int d = D - 2; d >= 0; --d) id = id * static_cast<unsigned>(dims[d]) + static_cast<unsigned>(c[d]);
  return id;
}

// Packed descent entries: level | coordinates (3D: 20/20/19 bits, 2D: 29/29).
template <int D>
__device__ __forceinline__ unsigned long long pack(int L, const int* c) {
  if constexpr (D == 3)
    return (static_cast<unsigned long long>(L) << 59) | (static_cast<unsigned long long>(c[2]) << 40) |
           (static_cast<unsigned long long>(c[1]) << 20) | static_cast<unsigned long long>(c[0]);
  else
    return (static_cast<unsigned long long>(L) << 58) | (static_cast<unsigned long long>(c[1]) << 29) |
           static_cast<unsigned long long>(c[0]);
}
template <int D>
__device__ __forceinline__ int unpack(unsigned long long e, int* c) {
  if constexpr (D == 3) {
    c[0] = static_cast<int>(e & 0xFFFFFu);
    c[1] = static_cast<int>((e >> 20) & 0xFFFFFu);
    c[2] = static_cast<int>((e >> 40) & 0x7FFFFu);
    return static_cast<int>(e >> 59);
  } else {
    c[0] = static_cast<int>(e & 0x1FFFFFFFu);
    c[1] = static_cast<int>((e >> 29) & 0x1FFFFFFFu);
    return static_cast<int>(e >> 58);
  }
}

__global__ void k_bbox_points_init(unsigned long long* bbox, int dim) {
  if (threadIdx.x < static_cast<unsigned>(dim)) {
    bbox[threadIdx.x] = 0xFFFFFFFFFFFFFFFFULL;
    bbox[dim + threadIdx.x] = 0ULL;
  }
}

template <int D>
__global__ void k_bbox_points(const double* __restrict__ xyz, std::uint64_t n, unsigned long long* bbox) {
  double lo[D], hi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) lo[d] = INFINITY, hi[d] = -INFINITY;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x)
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double v = xyz[i * D + d];
      lo[d] = fmin(lo[d], v);
      hi[d] = fmax(hi[d], v);
    }
  __shared__ unsigned long long s_lo[D], s_hi[D];
  if (threadIdx.x < D) s_lo[threadIdx.x] = 0xFFFFFFFFFFFFFFFFULL, s_hi[threadIdx.x] = 0ULL;
  __syncthreads();
#pragma unroll
  for (int d = 0; d < D; ++d) {
    atomicMin(&s_lo[d], dbl_to_ordered(lo[d]));
    atomicMax(&s_hi[d], dbl_to_ordered(hi[d]));
  }
  __syncthreads();
  if (threadIdx.x < D) {
    atomicMin(&bbox[threadIdx.x], s_lo[threadIdx.x]);
    atomicMax(&bbox[D + threadIdx.x], s_hi[threadIdx.x]);
  }
}

// Grid parameters from the global bbox: edge = c_G (V/n)^(1/D) (SPEC.md:403 /
// build_grid_index post), origin = bbox lo, dims = floor(ext/edge)+1.
template <int D>
__global__ void k_owner_params(const unsigned long long* bbox, std::uint64_t n, double c_G,
                               unsigned long long cap, OwnerGrid<D>* og, unsigned* status) {
  double lo[D], hi[D], vol = 1.0, ext_max = 0.0, mag = 0.0;
  for (int d = 0; d < D; ++d) {
    lo[d] = ordered_to_dbl(bbox[d]);
    hi[d] = ordered_to_dbl(bbox[D + d]);
    vol *= (hi[d] - lo[d]);
    ext_max = fmax(ext_max, hi[d] - lo[d]);
    mag = fmax(mag, fmax(fabs(lo[d]), fabs(hi[d])));
  }
  const double per = vol / static_cast<double>(n);
  const double e = c_G * ((D == 2) ? sqrt(per) : cbrt_det(per));
  unsigned long long cells = 1;
  bool bad = !(e > 0.0);
  const double axis_cap = D == 3 ? 500000.0 : 500000000.0;  // packed-coordinate range
  for (int d = 0; d < D; ++d) {
    og->g.lo[d] = lo[d];
    const double f = bad ? 0.0 : floor((hi[d] - lo[d]) / e);
    if (!(f < axis_cap)) bad = true;
    og->g.dims[d] = bad ? 1 : static_cast<long long>(f) + 1;
    cells *= static_cast<unsigned long long>(og->g.dims[d]);
  }
  if (bad || cells > cap) {
    atomicOr(status, kStGridCap);
    for (int d = 0; d < D; ++d) og->g.dims[d] = 1;
  }
  og->g.edge = bad ? 1.0 : e;
  og->inv_edge = 1.0 / og->g.edge;
  og->margin = 1e-9 * (mag + ext_max + og->g.edge);
  const int sh = fan_shift<D>();
  og->shift = sh;
  int L = 0;
  unsigned long long off = 0;
  for (;;) {
    bool top = true;
    unsigned long long cnt = 1;
    for (int d = 0; d < D; ++d) {
      og->ldims[L][d] = static_cast<int>(((og->g.dims[d] - 1) >> (L * sh)) + 1);
      cnt *= static_cast<unsigned long long>(og->ldims[L][d]);
      top = top && og->ldims[L][d] == 1;
    }
    og->loff[L] = off;
    off += cnt;
    ++L;
    if (top || L == kMaxLevels) break;
  }
  og->loff[L] = off;
  og->levels = L;
}

// Mark leaf cells with their owner; optionally the per-partition point bbox.
template <int D>
__global__ void k_owner_mark(const double* __restrict__ xyz, const std::uint32_t* __restrict__ labels,
                             std::uint64_t n, const OwnerGrid<D>* __restrict__ ogp, std::uint16_t* __restrict__ owner,
                             unsigned long long* __restrict__ pbbox, std::uint32_t k) {
  __shared__ Grid<D> g;
  __shared__ int dims[D];
  extern __shared__ unsigned long long s_pb[];  // [k][2D] when pbbox != nullptr
  if (threadIdx.x == 0) {
    g = ogp->g;
    for (int d = 0; d < D; ++d) dims[d] = ogp->ldims[0][d];
  }
  if (pbbox)
    for (std::uint32_t j = threadIdx.x; j < k * 2 * D; j += blockDim.x)
      s_pb[j] = ((j % (2 * D)) < D) ? 0xFFFFFFFFFFFFFFFFULL : 0ULL;
  __syncthreads();
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    double x[D];
    int c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      x[d] = xyz[i * D + d];
      c[d] = static_cast<int>(cell_coord<D>(g, x[d], d));
    }
    const std::uint32_t lab = labels[i];
    std::uint16_t* slot = owner + lin<D>(dims, c);
    unsigned short old = *slot;
    while (old != lab && old != kOwnerMulti) {
      const unsigned short nv = (old == kOwnerEmpty) ? static_cast<unsigned short>(lab) : kOwnerMulti;
      const unsigned short prev = atomicCAS(reinterpret_cast<unsigned short*>(slot), old, nv);
      if (prev == old) break;
      old = prev;
    }
    if (pbbox) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        atomicMin(&s_pb[lab * 2 * D + d], dbl_to_ordered(x[d]));
        atomicMax(&s_pb[lab * 2 * D + D + d], dbl_to_ordered(x[d]));
      }
    }
  }
  if (pbbox) {
    __syncthreads();
    for (std::uint32_t j = threadIdx.x; j < k * 2 * D; j += blockDim.x) {
      if ((j % (2 * D)) < D) atomicMin(&pbbox[j], s_pb[j]);
      else atomicMax(&pbbox[j], s_pb[j]);
    }
  }
}

__global__ void k_pbbox_init(unsigned long long* pbbox, std::uint32_t count, int dim) {
  for (std::uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x)
    pbbox[j] = ((j % (2 * dim)) < static_cast<std::uint32_t>(dim)) ? 0xFFFFFFFFFFFFFFFFULL : 0ULL;
}

__device__ __forceinline__ std::uint16_t combine(std::uint16_t a, std::uint16_t b) {
  if (a == kOwnerEmpty) return b;
  if (b == kOwnerEmpty) return a;
  return a == b ? a : kOwnerMulti;
}

template <int D>
__device__ __forceinline__ void build_block(const OwnerGrid<D>& og, std::uint16_t* owner, int L, unsigned long long id) {
  const int F = 1 << og.shift;
  int c[D];
  {
    unsigned long long rem = id;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      c[d] = static_cast<int>(rem % static_cast<unsigned>(og.ldims[L][d]));
      rem /= static_cast<unsigned>(og.ldims[L][d]);
    }
  }
  std::uint16_t code = kOwnerEmpty;
  int ch[D];
  const int* cd = og.ldims[L - 1];
  if constexpr (D == 3) {
    for (ch[2] = c[2] * F; ch[2] < min((c[2] + 1) * F, cd[2]); ++ch[2])
      for (ch[1] = c[1] * F; ch[1] < min((c[1] + 1) * F, cd[1]); ++ch[1])
        for (ch[0] = c[0] * F; ch[0] < min((c[0] + 1) * F, cd[0]); ++ch[0])
          code = combine(code, owner[og.loff[L - 1] + lin<D>(cd, ch)]);
  } else {
    for (ch[1] = c[1] * F; ch[1] < min((c[1] + 1) * F, cd[1]); ++ch[1])
      for (ch[0] = c[0] * F; ch[0] < min((c[0] + 1) * F, cd[0]); ++ch[0])
        code = combine(code, owner[og.loff[L - 1] + lin<D>(cd, ch)]);
  }
  owner[og.loff[L] + id] = code;
}

template <int D>
__global__ void k_owner_level(const OwnerGrid<D>* __restrict__ ogp, std::uint16_t* __restrict__ owner, int L) {
  __shared__ OwnerGrid<D> og;
  if (threadIdx.x == 0) og = *ogp;
  __syncthreads();
  if (L >= og.levels) return;
  const unsigned long long cnt = og.loff[L + 1] - og.loff[L];
  for (unsigned long long id = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; id < cnt;
       id += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
    build_block<D>(og, owner, L, id);
}

template <int D>
__global__ void k_owner_levels_tail(const OwnerGrid<D>* __restrict__ ogp, std::uint16_t* __restrict__ owner, int L0) {
  __shared__ OwnerGrid<D> og;
  if (threadIdx.x == 0) og = *ogp;
  __syncthreads();
  for (int L = L0; L < og.levels; ++L) {
    const unsigned long long cnt = og.loff[L + 1] - og.loff[L];
    for (unsigned long long id = threadIdx.x; id < cnt; id += blockDim.x) build_block<D>(og, owner, L, id);
    __syncthreads();
  }
}

// ---- descent helpers -----------------------------------------------------------
template <int D>
__device__ __forceinline__ void block_box(const OwnerGrid<D>& og, int L, const int* c, double* blo, double* bhi) {
  const int s = L * og.shift;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const long long first = static_cast<long long>(c[d]) << s;
    long long last1 = static_cast<long long>(c[d] + 1) << s;
    if (last1 > og.g.dims[d]) last1 = og.g.dims[d];
    blo[d] = cell_lo<D>(og.g, first, d);
    bhi[d] = cell_lo<D>(og.g, last1, d);
  }
}

// Depth-first pyramid descent with one cursor frame per level (depth bounded
// by the number of levels, no overflow). Visits the blocks of level L0 in the
// leaf range [a,b] (restricted) or the single top block; a block whose code
// is EMPTY or `self` is pruned; test(blo, bhi) returns 0 (reject), 1
// (descend) or 2 (accept: every sub-box passes, so a foreign occupied leaf
// inside passes). A leaf that passes is a hit.
template <int D, class Test>
__device__ bool descend(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner, std::uint32_t self, int L0,
                        const int* a, const int* b, bool restrict_range, const Test& test) {
  struct Frame {
    int lo[D], hi[D], cur[D];
    int level;
  };
  Frame fr[kMaxLevels + 1];
  int depth = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    fr[0].lo[d] = restrict_range ? (a[d] >> (L0 * og.shift)) : 0;
    fr[0].hi[d] = restrict_range ? (b[d] >> (L0 * og.shift)) : og.ldims[L0][d] - 1;
    fr[0].cur[d] = fr[0].lo[d];
  }
  fr[0].level = L0;
  while (depth > 0) {
    Frame& f = fr[depth - 1];
    if (f.cur[D - 1] > f.hi[D - 1]) {
      --depth;
      continue;
    }
    int cc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cc[d] = f.cur[d];
    // odometer advance
    ++f.cur[0];
#pragma unroll
    for (int d = 0; d < D - 1; ++d)
      if (f.cur[d] > f.hi[d]) {
        f.cur[d] = f.lo[d];
        ++f.cur[d + 1];
      }
    const int lv = f.level;
    const std::uint16_t code = owner[og.loff[lv] + lin<D>(og.ldims[lv], cc)];
    if (code == kOwnerEmpty || code == self) continue;
    double blo[D], bhi[D];
    block_box<D>(og, lv, cc, blo, bhi);
    const int r = test(blo, bhi);
    if (r == 0) continue;
    if (lv == 0 || r == 2) return true;
    const int cl = lv - 1;
    const int csh = cl * og.shift;
    Frame& g = fr[depth];
    bool empty = false;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      int lo = cc[d] << og.shift;
      int hi = min(((cc[d] + 1) << og.shift) - 1, og.ldims[cl][d] - 1);
      if (restrict_range) {
        lo = max(lo, a[d] >> csh);
        hi = min(hi, b[d] >> csh);
      }
      g.lo[d] = lo;
      g.hi[d] = hi;
      g.cur[d] = lo;
      empty = empty || lo > hi;
    }
    g.level = cl;
    if (!empty) ++depth;
  }
  return false;
}

// true iff some cell with owner code not in {EMPTY, self} overlaps the sphere.
template <int D>
__device__ bool sphere_hits_foreign(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner,
                                    const double* c, double r2, std::uint32_t self) {
  if (isnan(r2)) return false;
  bool fin = isfinite(r2);
#pragma unroll
  for (int d = 0; d < D; ++d) fin = fin && isfinite(c[d]);
  int a[D], b[D];
  if (fin) {
    // Conservative leaf range: the margin (1e-9 relative) dominates the
    // rounding of this multiply-by-inverse binning.
    const double r = sqrt(r2) * (1.0 + 1e-9) + og.margin;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double fa = floor((c[d] - r - og.g.lo[d]) * og.inv_edge);
      const double fb = floor((c[d] + r - og.g.lo[d]) * og.inv_edge);
      const double top = static_cast<double>(og.ldims[0][d] - 1);
      if (fb < 0.0 || fa > top) return false;
      a[d] = fa < 0.0 ? 0 : static_cast<int>(fa);
      b[d] = fb > top ? og.ldims[0][d] - 1 : static_cast<int>(fb);
    }
  } else {
#pragma unroll
    for (int d = 0; d < D; ++d) a[d] = 0, b[d] = og.ldims[0][d] - 1;
  }
  int L = 0;
  for (; L < og.levels - 1; ++L) {
    bool ok = true;
#pragma unroll
    for (int d = 0; d < D; ++d) ok = ok && ((b[d] >> (L * og.shift)) - (a[d] >> (L * og.shift)) <= 1);
    if (ok) break;
  }
  // Fast path: start blocks (<= 2 per axis) all EMPTY or own partition.
  {
    int s0[D], n0[D];
    bool any = false;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      s0[d] = a[d] >> (L * og.shift);
      n0[d] = (b[d] >> (L * og.shift)) - s0[d] + 1;
    }
    const int total = D == 3 ? n0[0] * n0[1] * n0[2] : n0[0] * n0[1];
    for (int t = 0; t < total && !any; ++t) {
      int cc[D], rem = t;  // every n0 is 1 or 2 at the start level
#pragma unroll
      for (int d = 0; d < D; ++d) {
        cc[d] = s0[d] + (rem & (n0[d] - 1));
        rem >>= (n0[d] - 1);
      }
      const std::uint16_t code = owner[og.loff[L] + lin<D>(og.ldims[L], cc)];
      any = !(code == kOwnerEmpty || code == self);
    }
    if (!any) return false;
  }
  return descend<D>(og, owner, self, L, a, b, true, [&](const double* blo, const double* bhi) {
    if (!box_sphere<D>(blo, bhi, c, r2)) return 0;
    return box_inside_sphere<D>(blo, bhi, c, r2) ? 2 : 1;
  });
}

// Halfspace variant: test = some box corner strictly on the outer side of
// the facet plane (exact orient), full = every corner strictly outside.
template <int D>
__device__ int corners_outside(const double* const* facet, int inner_sign, const double* blo, const double* bhi) {
  const double* pts[D + 1];
#pragma unroll
  for (int i = 0; i < D; ++i) pts[i] = facet[i];
  double corner[D];
  pts[D] = corner;
  int outside = 0;
  for (unsigned cm = 0; cm < (1u << D); ++cm) {
#pragma unroll
    for (int d = 0; d < D; ++d) corner[d] = (cm & (1u << d)) ? bhi[d] : blo[d];
    const int s = orient_dev<D>(pts);
    if (s != 0 && s != inner_sign) ++outside;
  }
  return outside;
}

template <int D>
__device__ bool halfspace_hits_foreign(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner,
                                       const double* const* facet, int inner_sign, std::uint32_t self) {
  return descend<D>(og, owner, self, og.levels - 1, nullptr, nullptr, false,
                    [&](const double* blo, const double* bhi) {
                      const int out = corners_outside<D>(facet, inner_sign, blo, bhi);
                      if (out == 0) return 0;
                      return out == (1 << D) ? 2 : 1;
                    });
}

// circumsphere (geometry.cpp:279-327) + inflated (geometry.hpp:179-183)
template <int D>
__device__ __forceinline__ void circumsphere_inflated(const double (*p)[D], double* center, double* r2) {
  if constexpr (D == 2) {
    const double ux = p[1][0] - p[0][0], uy = p[1][1] - p[0][1];
    const double vx = p[2][0] - p[0][0], vy = p[2][1] - p[0][1];
    const double bu = 0.5 * (ux * ux + uy * uy);
    const double bv = 0.5 * (vx * vx + vy * vy);
    const double det = ux * vy - uy * vx;
    const double cx = (bu * vy - bv * uy) / det;
    const double cy = (ux * bv - vx * bu) / det;
    center[0] = p[0][0] + cx;
    center[1] = p[0][1] + cy;
    *r2 = (cx * cx + cy * cy) * (1.0 + 1e-10);
  } else {
    double m[3][3], rhs[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double n2 = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        m[i][d] = p[i + 1][d] - p[0][d];
        n2 += m[i][d] * m[i][d];
      }
      rhs[i] = 0.5 * n2;
    }
    const double m00 = m[0][0], m01 = m[0][1], m02 = m[0][2];
    const double m10 = m[1][0], m11 = m[1][1], m12 = m[1][2];
    const double m20 = m[2][0], m21 = m[2][1], m22 = m[2][2];
    // det3x3 exactly as geometry.cpp:310-314, for m and the three Cramer matrices
    const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) + m02 * (m10 * m21 - m11 * m20);
    const double r0 = rhs[0], r1 = rhs[1], r2_ = rhs[2];
    const double d0 = r0 * (m11 * m22 - m12 * m21) - m01 * (r1 * m22 - m12 * r2_) + m02 * (r1 * m21 - m11 * r2_);
    const double d1 = m00 * (r1 * m22 - m12 * r2_) - r0 * (m10 * m22 - m12 * m20) + m02 * (m10 * r2_ - r1 * m20);
    const double d2 = m00 * (m11 * r2_ - r1 * m21) - m01 * (m10 * r2_ - r1 * m20) + r0 * (m10 * m21 - m11 * m20);
    const double rel0 = d0 / det, rel1 = d1 / det, rel2 = d2 / det;
    center[0] = p[0][0] + rel0;
    center[1] = p[0][1] + rel1;
    center[2] = p[0][2] + rel2;
    *r2 = (rel0 * rel0 + rel1 * rel1 + rel2 * rel2) * (1.0 + 1e-10);
  }
}

__device__ __forceinline__ std::uint32_t part_of(const std::uint64_t* offs, std::uint32_t k, std::uint64_t s) {
  std::uint32_t lo = 0, hi = k;  // offs[lo] <= s < offs[hi]
  while (hi - lo > 1) {
    const std::uint32_t mid = (lo + hi) >> 1;
    if (offs[mid] <= s) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct BorderArgs {
  const double* xyz;
  std::uint64_t n;
  std::uint32_t k;
  const std::uint64_t* offsets;
  const std::uint32_t* verts;
  const std::uint32_t* nbrs;
  const std::int8_t* parity;
  std::uint64_t S;
  int policy;
  const std::uint16_t* owner;
  const unsigned long long* pbbox;  // [k][2D] ordered (bbox policy)
  std::uint8_t* positive;
  std::uint8_t* vflags;
  double* spheres;  // optional (D+1) per simplex
  std::uint32_t* inf_queue;
  unsigned* inf_count;
  unsigned* status;
};

// bbox-policy root box of partition j: its point bbox snapped to the occupied
// cells (= the AABB-tree root, oracle GridIndex::bbox_policy_box). Cell
// binning is monotone, so the extreme cells are the cells of the extreme points.
template <int D>
__device__ __forceinline__ bool bbox_policy_box(const OwnerGrid<D>& og, const unsigned long long* pbbox,
                                                std::uint32_t j, double* blo, double* bhi) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double pl = ordered_to_dbl(pbbox[j * 2 * D + d]);
    const double ph = ordered_to_dbl(pbbox[j * 2 * D + D + d]);
    if (!(pl <= ph)) return false;  // empty partition
    blo[d] = cell_lo<D>(og.g, cell_coord<D>(og.g, pl, d), d);
    bhi[d] = cell_lo<D>(og.g, cell_coord<D>(og.g, ph, d) + 1, d);
  }
  return true;
}

template <int D>
__device__ __forceinline__ bool bbox_policy_sphere(const OwnerGrid<D>& og, const BorderArgs& a, std::uint32_t self,
                                                   const double* c, double r2) {
  for (std::uint32_t j = 0; j < a.k; ++j) {
    if (j == self) continue;
    double blo[D], bhi[D];
    if (bbox_policy_box<D>(og, a.pbbox, j, blo, bhi) && box_sphere<D>(blo, bhi, c, r2)) return true;
  }
  return false;
}

template <int D>
__global__ void __launch_bounds__(kBThreads) k_border_finite(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp) {
  __shared__ OwnerGrid<D> og;
  extern __shared__ std::uint64_t s_off[];
  if (threadIdx.x == 0) og = *ogp;
  for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off[j] = a.offsets[j];
  __syncthreads();
  for (std::uint64_t s = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < a.S;
       s += std::uint64_t(gridDim.x) * blockDim.x) {
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = __ldcs(a.verts + std::uint64_t(j) * a.S + s);
    if (v[D] == kInfVertex) {
      const unsigned slot = atomicAdd(a.inf_count, 1u);
      a.inf_queue[slot] = static_cast<std::uint32_t>(s);
      continue;
    }
    if (a.parity[s] == 0) atomicOr(a.status, kStDegenerate);
    const std::uint32_t self = part_of(s_off, a.k, s);
    double p[D + 1][D];
#pragma unroll
    for (int j = 0; j <= D; ++j)
#pragma unroll
      for (int d = 0; d < D; ++d) p[j][d] = a.xyz[std::size_t(v[j]) * D + d];
    double c[D], r2;
    circumsphere_inflated<D>(p, c, &r2);
    if (a.spheres) {
#pragma unroll
      for (int d = 0; d < D; ++d) a.spheres[s * (D + 1) + d] = c[d];
      a.spheres[s * (D + 1) + D] = r2;
    }
    const bool pos = (a.policy == SBDT_POLICY_BBOX) ? bbox_policy_sphere<D>(og, a, self, c, r2)
                                                    : sphere_hits_foreign<D>(og, a.owner, c, r2, self);
    __stcs(a.positive + s, static_cast<std::uint8_t>(pos ? 1 : 0));
    if (pos)
#pragma unroll
      for (int j = 0; j <= D; ++j) a.vflags[v[j]] = 1;
  }
}

template <int D>
__global__ void __launch_bounds__(128) k_border_infinite(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp) {
  __shared__ OwnerGrid<D> og;
  extern __shared__ std::uint64_t s_off[];
  if (threadIdx.x == 0) og = *ogp;
  for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off[j] = a.offsets[j];
  __syncthreads();
  const unsigned count = *a.inf_count;
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x) {
    const std::uint64_t s = a.inf_queue[q];
    const std::uint32_t self = part_of(s_off, a.k, s);
    std::uint32_t fv[D];
#pragma unroll
    for (int j = 0; j < D; ++j) fv[j] = a.verts[std::uint64_t(j) * a.S + s];
    const std::uint64_t owner_row = s_off[self] + a.nbrs[std::uint64_t(D) * a.S + s];
    std::uint32_t inner = kInfVertex;
    for (int j = 0; j <= D; ++j) {
      const std::uint32_t w = a.verts[std::uint64_t(j) * a.S + owner_row];
      bool on = false;
#pragma unroll
      for (int f = 0; f < D; ++f) on = on || (fv[f] == w);
      if (!on) {
        inner = w;
        break;
      }
    }
    const double* facet[D];
#pragma unroll
    for (int j = 0; j < D; ++j) facet[j] = a.xyz + std::size_t(fv[j]) * D;
    const double* pts[D + 1];
#pragma unroll
    for (int j = 0; j < D; ++j) pts[j] = facet[j];
    pts[D] = a.xyz + std::size_t(inner) * D;
    const int inner_sign = orient_dev<D>(pts);
    bool pos = false;
    if (a.policy == SBDT_POLICY_BBOX) {
      for (std::uint32_t j = 0; j < a.k && !pos; ++j) {
        if (j == self) continue;
        double blo[D], bhi[D];
        if (bbox_policy_box<D>(og, a.pbbox, j, blo, bhi) && corners_outside<D>(facet, inner_sign, blo, bhi) > 0)
          pos = true;
      }
    } else {
      pos = halfspace_hits_foreign<D>(og, a.owner, facet, inner_sign, self);
    }
    a.positive[s] = pos ? 1 : 0;
    if (a.spheres)
#pragma unroll
      for (int d = 0; d <= D; ++d) a.spheres[s * (D + 1) + d] = 0.0;
    if (pos)
#pragma unroll
      for (int j = 0; j < D; ++j) a.vflags[fv[j]] = 1;
  }
}

// ---- K9: flag compaction (two passes, ballot + block prefix sums) -------------
constexpr int kCompactThreads = 256;
constexpr int kCompactPerThread = 32;
constexpr int kCompactTile = kCompactThreads * kCompactPerThread;

__global__ void k_compact_count(const std::uint8_t* __restrict__ flags, std::uint64_t n,
                                std::uint32_t* __restrict__ block_counts) {
  const std::uint64_t first = std::uint64_t(blockIdx.x) * kCompactTile + std::uint64_t(threadIdx.x) * kCompactPerThread;
  std::uint32_t cnt = 0;
  if (first + kCompactPerThread <= n) {
    const uint4* p = reinterpret_cast<const uint4*>(flags + first);
    const uint4 a = p[0], b = p[1];
    const unsigned w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) cnt += __popc(w[i] & 0x01010101u);
  } else {
    for (std::uint64_t i = first; i < n && i < first + kCompactPerThread; ++i) cnt += flags[i] != 0;
  }
  std::uint32_t total;
  block_exclusive_scan<kCompactThreads>(cnt, &total);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = total;
}

__global__ void k_compact_write(const std::uint8_t* __restrict__ flags, std::uint64_t n,
                                const std::uint32_t* __restrict__ block_offsets, std::uint32_t* __restrict__ out) {
  const std::uint64_t first = std::uint64_t(blockIdx.x) * kCompactTile + std::uint64_t(threadIdx.x) * kCompactPerThread;
  unsigned w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (first + kCompactPerThread <= n) {
    const uint4* p = reinterpret_cast<const uint4*>(flags + first);
    const uint4 a = p[0], b = p[1];
    w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w, w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
  } else {
    for (std::uint64_t i = first; i < n && i < first + kCompactPerThread; ++i)
      if (flags[i]) w[(i - first) >> 2] |= 1u << (8 * ((i - first) & 3));
  }
  std::uint32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) cnt += __popc(w[i] & 0x01010101u);
  std::uint32_t pos = block_exclusive_scan<kCompactThreads>(cnt, nullptr) + block_offsets[blockIdx.x];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if ((w[i] >> (8 * b)) & 0xFFu) out[pos++] = static_cast<std::uint32_t>(first + 4 * i + b);
}

__global__ void k_u32_to_u64(const std::uint32_t* in, std::uint64_t* out) { *out = *in; }

// ---------------------------------------------------------------------------
int compact_flags(sbdt_gpu_ctx* ctx, const std::uint8_t* d_flags, std::uint64_t n, std::uint32_t* d_out,
                  std::uint64_t* d_count) {
  cudaStream_t st = ctx->stream;
  const std::uint64_t blocks = (n + kCompactTile - 1) / kCompactTile;
  SBDT_WS(bc, std::uint32_t, "compact.bc", blocks + 2);
  SBDT_WS(tot, std::uint32_t, "compact.tot", 1);
  if (blocks == 0) {
    SBDT_CUDA_TRY(cudaMemsetAsync(d_count, 0, 8, st));
    return kOk;
  }
  k_compact_count<<<static_cast<unsigned>(blocks), kCompactThreads, 0, st>>>(d_flags, n, bc);
  k_scan_single<<<1, kScanThreads, 0, st>>>(bc, blocks, tot);
  k_compact_write<<<static_cast<unsigned>(blocks), kCompactThreads, 0, st>>>(d_flags, n, bc, d_out);
  k_u32_to_u64<<<1, 1, 0, st>>>(tot, d_count);
  ctx->launches += 4;
  return kOk;
}

template <int D>
int border_impl(sbdt_gpu_ctx* ctx, const sbdt_border_args* in) {
  cudaStream_t st = ctx->stream;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const double cg = in->c_G > 0 ? in->c_G : 1.0;
  double scale = 1.0;
  for (int d = 0; d < D; ++d) scale /= cg;
  const unsigned long long cap = static_cast<unsigned long long>(4.0 * double(in->n) * scale) + 4096;
  const unsigned long long owner_len = cap * 8 / 7 + 64 * kMaxLevels + 64;
  SBDT_WS(og, OwnerGrid<D>, "border.og", 1);
  SBDT_WS(owner, std::uint16_t, "border.owner", owner_len);
  SBDT_WS(bbox, unsigned long long, "border.bbox", 2 * D);
  SBDT_WS(infq, std::uint32_t, "border.infq", in->S / 2 + 1024);
  SBDT_WS(infc, unsigned, "border.infc", 1);
  unsigned long long* pbbox = nullptr;
  if (in->policy == SBDT_POLICY_BBOX) {
    SBDT_WS(pb, unsigned long long, "border.pbbox", std::uint64_t(in->k) * 2 * D);
    pbbox = pb;
  }

  StageTimer tgrid(ctx, "border.grid");
  const unsigned long long* bb = reinterpret_cast<const unsigned long long*>(in->d_bbox_ordered);
  if (!bb) {
    k_bbox_points_init<<<1, 32, 0, st>>>(bbox, D);
    const std::uint64_t want = (in->n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 8 ? want : std::uint64_t(sms) * 8);
    k_bbox_points<D><<<blocks > 0 ? blocks : 1, 256, 0, st>>>(in->d_xyz, in->n, bbox);
    ctx->launches += 2;
    bb = bbox;
  }
  k_owner_params<D><<<1, 1, 0, st>>>(bb, in->n, cg, cap, og, ctx->d_status);
  SBDT_CUDA_TRY(cudaMemsetAsync(owner, 0xFF, sizeof(std::uint16_t) * owner_len, st));
  if (pbbox) {
    k_pbbox_init<<<(in->k * 2 * D + 255) / 256, 256, 0, st>>>(pbbox, in->k * 2 * D, D);
    ctx->launches += 1;
  }
  {
    const std::uint64_t want = (in->n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 16 ? want : std::uint64_t(sms) * 16);
    const std::size_t sh = pbbox ? sizeof(unsigned long long) * in->k * 2 * D : 0;
    k_owner_mark<D><<<blocks > 0 ? blocks : 1, 256, sh, st>>>(in->d_xyz, in->d_labels, in->n, og, owner, pbbox, in->k);
  }
  k_owner_level<D><<<sms * 8, 256, 0, st>>>(og, owner, 1);
  k_owner_level<D><<<sms * 2, 256, 0, st>>>(og, owner, 2);
  k_owner_levels_tail<D><<<1, 1024, 0, st>>>(og, owner, 3);
  ctx->launches += 6;

  SBDT_CUDA_TRY(cudaMemsetAsync(in->d_vertex_flags, 0, in->n, st));
  SBDT_CUDA_TRY(cudaMemsetAsync(infc, 0, sizeof(unsigned), st));
  tgrid.end();
  BorderArgs a;
  a.xyz = in->d_xyz;
  a.n = in->n;
  a.k = in->k;
  a.offsets = in->d_offsets;
  a.verts = in->d_verts;
  a.nbrs = in->d_nbrs;
  a.parity = in->d_parity;
  a.S = in->S;
  a.policy = in->policy;
  a.owner = owner;
  a.pbbox = pbbox;
  a.positive = in->d_positive;
  a.vflags = in->d_vertex_flags;
  a.spheres = in->d_spheres;
  a.inf_queue = infq;
  a.inf_count = infc;
  a.status = ctx->d_status;
  const std::size_t offs_sh = sizeof(std::uint64_t) * (in->k + 1);
  {
    const std::uint64_t want = (in->S + kBThreads - 1) / kBThreads;
    const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 32 ? want : std::uint64_t(sms) * 32);
    {
      StageTimer t(ctx, "border.finite");
      if (blocks > 0) k_border_finite<D><<<blocks, kBThreads, offs_sh, st>>>(a, og);
    }
    {
      StageTimer t(ctx, "border.infinite");
      k_border_infinite<D><<<sms * 2, 128, offs_sh, st>>>(a, og);
    }
    ctx->launches += 2;
  }
  StageTimer tc(ctx, "border.compact");
  int rc = compact_flags(ctx, in->d_vertex_flags, in->n, in->d_vertex_ids, in->d_vertex_count);
  if (rc != kOk) return rc;
  SBDT_CUDA_TRY(cudaGetLastError());
  return kOk;
}

template int border_impl<2>(sbdt_gpu_ctx*, const sbdt_border_args*);
template int border_impl<3>(sbdt_gpu_ctx*, const sbdt_border_args*);

}  // namespace sbdt_gpu
