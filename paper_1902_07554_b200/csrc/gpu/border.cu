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
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"
#include "context.cuh"
#include "owner_grid.cuh"
#include "../common/plane_filter.hpp"
#include "scan.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {

constexpr int kBThreads = 256;
#ifndef PF_THREADS
#define PF_THREADS 256
#define PF_CTAS 4
#endif
constexpr int kPfThreads = PF_THREADS;  // prefilter CTA size / CTAs per SM (launch bound)
constexpr std::uint32_t kSmemOffsMax = 1024;  // part offsets staged in shared memory up to this many (k + 1)

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

// The grid's bbox given by the caller (recursion levels), as ordered keys.
struct GridBox {
  double lo[3], hi[3];
};
template <int D>
__global__ void k_set_bbox(GridBox gb, unsigned long long* bbox) {
#pragma unroll
  for (int d = 0; d < D; ++d) {
    bbox[d] = dbl_to_ordered(gb.lo[d]);
    bbox[D + d] = dbl_to_ordered(gb.hi[d]);
  }
}

__global__ void k_pbbox_init(unsigned long long* pbbox, std::uint32_t count, int dim) {
  for (std::uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x)
    pbbox[j] = ((j % (2 * dim)) < static_cast<std::uint32_t>(dim)) ? 0xFFFFFFFFFFFFFFFFULL : 0ULL;
}

// Exact orientation of the simplex (predicates.hpp: filter + expansion
// arithmetic); 0 = degenerate, which the reference's circumsphere rejects
// with DegenerateSimplex (geometry.cpp:279-297).
template <int D>
__device__ __forceinline__ int orientation_exact(const double (*p)[D], unsigned long long* escalations = nullptr) {
  const double* q[D + 1];
#pragma unroll
  for (int j = 0; j <= D; ++j) q[j] = p[j];
  return orient_dev<D>(q, escalations);
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

// MUFU approximations used only inside bounds that carry >= 1e-5 relative
// slack (PTX: rcp.approx.f32 within 1 ulp, sqrt.approx.f32 within ~2^-22).
// .ftz: one MUFU, no denormal fixup sequence. A subnormal input reads as 0:
// enclosing_sphere_f32 then fails its L > 1e-24 (1e-18) range check (edge
// lengths) or sees a non-finite centre (det), and its r, e arguments are
// >= 0.25 in 3-D (integer edges, P0e); only reciprocals of |det| <= 1e24
// (checked through L) are taken, far from a subnormal result.
__device__ __forceinline__ float sqrt_apx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_apx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// floor(x) for |x| < 2^22: x + 1.5 * 2^23 rounded toward -inf lands in
// [2^23, 2^24) where the float's bits are 0x4B400000 + floor(x).
__device__ __forceinline__ int floor_small(float x) { return __float_as_int(__fadd_rd(x, 12582912.f)) - 0x4B400000; }

template <int D>
struct Sphere32 {
  float P0[D];   // offset of vertex 0 from the grid origin
  float rel[D];  // centre - P0
  float r;       // |rel| (binary32, sqrt.approx)
  float e;       // bound on |centre - binary64 centre| (norm)
};

// Binary32 circumcentre with a rigorous error bound, for the prefilter only.
// Inputs: the edge vectors A[j] = P_{j+1} - P0 rounded to binary32 (at most
// two relative roundings per component), a bound eta on each component's
// absolute error from the coordinate encoding, P0 and per-axis bounds P0e on
// |P0 - (x0 - lo)|. With a, b, c the edges the centre relative to P0 is
//   rel = (|a|^2 (b x c) + |b|^2 (c x a) + |c|^2 (a x b)) / (2 a.(b x c)).
// Error budget:
//  - arithmetic incl. the input roundings (each term a product of at most 16
//    rounded factors): numerators within g NB and det within g DB of their
//    values at the encoded inputs, g = 2e-6 > gamma_16, with the absolute-value
//    sums bounded by Cauchy-Schwarz: NB = |a||b||c| (|a|+|b|+|c|),
//    DB = sqrt(3) |a||b||c|;
//  - encoding: with eta2 = sqrt(3) eta and M >= every edge length,
//    |dn| <= 6 M^2 (2 M eta2 + eta2^2) and |ddet| <= 3 M^2 eta2 + M eta2^2.
// With EN, ED the two totals and |det'| > 4 ED,
//   |rel_i' - rel_i| <= (EN / 2 + |rel_i'| ED) / (|det'| - ED) + 1.5e-6 |rel_i'|
// (the last term: rcp.approx and the product), plus P0e_i for the centre's
// offset. The binary64 Cramer evaluation of circumsphere_inflated() is ~1e-9
// of that bound from the exact centre (unit roundoff 2^-53), absorbed by the
// 1e-6 slacks. The 2-D form is the same with a x b
// (|dn| <= 2 (3 M^2 eta2 + M eta2^2), |ddet| <= 2 M eta2 + eta2^2).
// false when the bound cannot be established (ill-conditioned, non-finite,
// binary32 under/overflow range).
template <int D>
__device__ __forceinline__ bool enclosing_sphere_f32(const float (*A)[D], float eta, const float* P0e,
                                                     Sphere32<D>& sp) {
  // Fused multiply-adds (explicit: the file is built with -fmad=false for the
  // binary64 reference expressions) round once where a separate product and
  // sum round twice, so every term carries at most as many roundings as the
  // gamma_16 budget above counts, with the same absolute-value sums.
  constexpr float g = 2e-6f;
  const float eta2 = 1.7321f * eta * 1.0001f;
  float err[D];
  float* rel = sp.rel;
  if constexpr (D == 2) {
    const float ax = A[0][0], ay = A[0][1], bx = A[1][0], by = A[1][1];
    const float aa = fmaf(ax, ax, ay * ay), bb = fmaf(bx, bx, by * by);
    const float det = fmaf(ax, by, -(ay * bx));
    const float la = sqrt_apx(aa) * 1.00001f, lb = sqrt_apx(bb) * 1.00001f;
    const float L = la * lb;
    const float M = fmaf(fmaxf(la, lb), 1.0001f, eta2);
    const float EN = fmaf(g * L * 1.0001f, la + lb, 2.f * M * eta2 * fmaf(3.f, M, eta2));
    const float ED = fmaf(g * 1.0001f, L, eta2 * fmaf(2.f, M, eta2));
    if (!(L > 1e-18f) || !(L < 1e18f) || !(fabsf(det) > 4.f * ED)) return false;
    const float inv2d = 0.5f * rcp_apx(det);
    rel[0] = fmaf(aa, by, -(bb * ay)) * inv2d;
    rel[1] = fmaf(bb, ax, -(aa * bx)) * inv2d;
    const float rden = 1.0002f * rcp_apx(fabsf(det) - ED);
    const float hEN = 0.5f * EN;
#pragma unroll
    for (int d = 0; d < 2; ++d)
      err[d] = fmaf(fmaf(fabsf(rel[d]), ED, hEN), rden, fmaf(1.5e-6f, fabsf(rel[d]), P0e[d]));
  } else {
    const float* a = A[0];
    const float* b = A[1];
    const float* q = A[2];
    const float aa = fmaf(a[0], a[0], fmaf(a[1], a[1], a[2] * a[2]));
    const float bb = fmaf(b[0], b[0], fmaf(b[1], b[1], b[2] * b[2]));
    const float qq = fmaf(q[0], q[0], fmaf(q[1], q[1], q[2] * q[2]));
    const float x0 = fmaf(b[1], q[2], -(b[2] * q[1])), x1 = fmaf(b[2], q[0], -(b[0] * q[2])),
                x2 = fmaf(b[0], q[1], -(b[1] * q[0]));
    const float y0 = fmaf(q[1], a[2], -(q[2] * a[1])), y1 = fmaf(q[2], a[0], -(q[0] * a[2])),
                y2 = fmaf(q[0], a[1], -(q[1] * a[0]));
    const float z0 = fmaf(a[1], b[2], -(a[2] * b[1])), z1 = fmaf(a[2], b[0], -(a[0] * b[2])),
                z2 = fmaf(a[0], b[1], -(a[1] * b[0]));
    const float det = fmaf(a[0], x0, fmaf(a[1], x1, a[2] * x2));
    const float la = sqrt_apx(aa) * 1.00001f, lb = sqrt_apx(bb) * 1.00001f, lq = sqrt_apx(qq) * 1.00001f;
    const float L = la * lb * lq;
    const float M = fmaf(fmaxf(la, fmaxf(lb, lq)), 1.0001f, eta2);
    const float M2 = M * M;
    const float EN = fmaf(g * L * 1.0001f, la + lb + lq, 6.f * M2 * eta2 * fmaf(2.f, M, eta2));
    const float ED = fmaf(g * 1.7321f * 1.0001f, L, M * eta2 * fmaf(3.f, M, eta2));
    if (!(L > 1e-24f) || !(L < 1e24f) || !(fabsf(det) > 4.f * ED)) return false;
    const float inv2d = 0.5f * rcp_apx(det);
    rel[0] = fmaf(aa, x0, fmaf(bb, y0, qq * z0)) * inv2d;
    rel[1] = fmaf(aa, x1, fmaf(bb, y1, qq * z1)) * inv2d;
    rel[2] = fmaf(aa, x2, fmaf(bb, y2, qq * z2)) * inv2d;
    const float rden = 1.0002f * rcp_apx(fabsf(det) - ED);
    const float hEN = 0.5f * EN;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      err[d] = fmaf(fmaf(fabsf(rel[d]), ED, hEN), rden, fmaf(1.5e-6f, fabsf(rel[d]), P0e[d]));
  }
  float rr = rel[0] * rel[0], ee = err[0] * err[0];
#pragma unroll
  for (int d = 1; d < D; ++d) {
    rr = fmaf(rel[d], rel[d], rr);
    ee = fmaf(err[d], err[d], ee);
  }
  if (!isfinite(rr) || !isfinite(ee)) return false;  // also catches non-finite rel / err
  sp.r = sqrt_apx(rr);
  sp.e = sqrt_apx(ee) * 1.0001f;
  return true;
}

// Decodes the packed prefilter coordinates (k_owner_mark) of one row into the
// edge vectors, P0 and the encoding error bounds of enclosing_sphere_f32, in
// the row's coordinate UNIT (prefilter_decide scales by it):
//   3-D: unit = qh, 21-bit fixed point q with |q - (x - lo) / qh| <= 0.5001:
//        edges are exact integer differences, eta = 1.0003 (two encodings);
//        P0 = q0 exactly: P0e = 0.50011;
//   2-D: unit = 1, binary32 offsets with |P - (x - lo)| <= u |P|: edges one
//        rounding, eta = 2u max|P|, P0e = u |P0|.
template <int D>
__device__ __forceinline__ void gather_row(const std::uint64_t* __restrict__ xq, const std::uint32_t* v, std::uint64_t n,
                                           std::uint64_t* w) {
#pragma unroll
  for (int j = 0; j <= D; ++j) w[j] = __ldg(xq + (v[j] < n ? v[j] : n));  // xq[n] exists (infinite / padding rows)
}

template <int D>
__device__ __forceinline__ void decode_row(const std::uint64_t* w, float (*A)[D], float* P0, float* P0e, float* eta) {
  constexpr float u = 5.9604645e-8f;
  if constexpr (D == 3) {
    int q[4][3];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int d = 0; d < 3; ++d) q[j][d] = static_cast<int>((w[j] >> (21 * d)) & 0x1FFFFFu);
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int d = 0; d < 3; ++d)
        // |dq| < 2^21: exact in binary32 via the 1.5 * 2^23 bias
        A[j][d] = __int_as_float(0x4B400000 + (q[j + 1][d] - q[0][d])) - 12582912.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      P0[d] = __int_as_float(0x4B000000 | q[0][d]) - 8388608.f;  // exact
      P0e[d] = 0.50011f;
    }
    *eta = 1.0003f;
  } else {
    float P[3][2];
    float pm = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      P[j][0] = __uint_as_float(static_cast<unsigned>(w[j]));
      P[j][1] = __uint_as_float(static_cast<unsigned>(w[j] >> 32));
      pm = fmaxf(pm, fmaxf(fabsf(P[j][0]), fabsf(P[j][1])));
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int d = 0; d < 2; ++d) A[j][d] = P[j + 1][d] - P[0][d];
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      P0[d] = P[0][d];
      P0e[d] = 6e-8f * fabsf(P0[d]);
    }
    *eta = 2.0001f * u * pm;
  }
}

constexpr int kFlatSpan = 7;  // widest per-axis cell range of the flattened exact scan

// Leaf-cell range of the (inflated binary64) sphere, as og_sphere_hits_foreign
// computes it: 0 = no cell reachable (negative), 1 = spans <= kFlatSpan
// (flattened cell scan), 2 = spans <= 16, 3 = wider or non-finite (2 and 3:
// pyramid descent in k_border_wide).
template <int D>
__device__ __forceinline__ int leaf_range(const OwnerGrid<D>& og, const double* c, double r2, int* lo, int* span) {
  if (isnan(r2)) return 0;
  bool fin = isfinite(r2);
#pragma unroll
  for (int d = 0; d < D; ++d) fin = fin && isfinite(c[d]);
  if (!fin) return 3;
  const double r = sqrt(r2) * (1.0 + 1e-9) + og.margin;
  int mode = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double fa = floor((c[d] - r - og.g.lo[d]) * og.inv_edge);
    const double fb = floor((c[d] + r - og.g.lo[d]) * og.inv_edge);
    const double top = static_cast<double>(og.ldims[0][d] - 1);
    if (fb < 0.0 || fa > top) return 0;
    lo[d] = fa < 0.0 ? 0 : static_cast<int>(fa);
    const int hi = fb > top ? og.ldims[0][d] - 1 : static_cast<int>(fb);
    span[d] = hi - lo[d] + 1;
    if (span[d] > kFlatSpan) mode = max(mode, 2);
    if (span[d] > 16) mode = 3;
  }
  if (mode == 2 && og.levels < 3) mode = 3;
  return mode;
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

// The part offsets of a kernel: staged in shared memory when k + 1 <=
// kSmemOffsMax, else read in place (an explicit, warp-uniform branch keeps
// the common case on shared-memory loads rather than generic ones).
struct PartOffs {
  const std::uint64_t* sh;
  const std::uint64_t* gl;
  bool small;
  __device__ __forceinline__ std::uint64_t operator[](std::uint32_t j) const { return small ? sh[j] : __ldg(gl + j); }
  __device__ __forceinline__ std::uint32_t part(std::uint32_t k, std::uint64_t s) const {
    return small ? part_of(sh, k, s) : part_of(gl, k, s);
  }
};

// part_of for a warp of consecutive rows: one binary search by lane 0, the
// lanes outside that part (warps straddling a part boundary) search alone.
// Must be called by the full warp.
__device__ __forceinline__ std::uint32_t part_of_warp(const std::uint64_t* offs, std::uint32_t k, std::uint64_t s) {
  std::uint32_t p0 = 0;
  if ((threadIdx.x & 31u) == 0) p0 = part_of(offs, k, s);
  p0 = __shfl_sync(0xffffffffu, p0, 0);
  if (s >= offs[p0] && s < offs[p0 + 1]) return p0;
  return part_of(offs, k, s);
}

struct BorderArgs {
  const double* xyz;
  const std::uint64_t* xq;    // packed prefilter coordinates by PointId (k_owner_mark)
  std::uint64_t n;
  std::uint32_t k;
  const std::uint64_t* offsets;
  const std::uint32_t* verts;
  const std::uint32_t* nbrs;
  const std::int8_t* parity;
  std::uint64_t S;
  int policy;
  const std::uint16_t* owner;
  const std::uint64_t* field;  // window field + foreign mask per cell (k_field_tiles), linear over ldims[0]
  const unsigned long long* pbbox;  // [k][2D] ordered (bbox policy)
  std::uint8_t* positive;
  std::uint8_t* vflags;
  double* spheres;  // optional (D+1) per simplex
  std::uint32_t* inf_queue;
  unsigned* inf_count;
  unsigned* status;
  unsigned long long* counters;  // census (optional), see sbdt_gpu_border_stats
  // exact policy
  int exact;
  const std::uint32_t* cell_start;  // per level-0 cell: first slot in cell_pts (k_cell_*)
  const void* cell_pts;             // CellPt<D>[n]
  std::uint32_t* esc;               // undecided filtered in_sphere tests: (row, cell-point slot)
  unsigned* esc_count;
  unsigned esc_cap;
  // rows with an undecided pair that did not fit the queue: decided again,
  // whole, by k_border_redo (bit per row + list)
  unsigned* redo_bits;
  std::uint32_t* redo_rows;
  unsigned* redo_count;
  // exact policy, hull rows: the hull vertex set of all partials (sorted ids)
  const std::uint32_t* labels;
  const std::uint32_t* hull_ids;
  const unsigned long long* hull_count;
  const unsigned* hull_valid;  // 1: every partition with points has simplex rows (the set is complete)
};

// Exact policy, one leaf cell: is some point of another part strictly inside
// the circumsphere of p (in_sphere_oriented, geometry.hpp:144-151)? The
// filtered predicate decides almost always; undecided pairs are queued for
// k_border_escalate (expansion arithmetic) and count as "not inside" here.
template <int D>
__device__ bool cell_points_inside(const BorderArgs& a, unsigned long long idx, const double (*p)[D], int parity,
                                   std::uint32_t self, std::uint64_t s) {
  const CellPt<D>* pts = static_cast<const CellPt<D>*>(a.cell_pts);
  const double* A = parity != 1 ? p[1] : p[0];
  const double* B = parity != 1 ? p[0] : p[1];
  for (std::uint32_t t = a.cell_start[idx], e = a.cell_start[idx + 1]; t < e; ++t) {
    const CellPt<D> q = pts[t];
    if (q.label == self) continue;
    int r;
    if constexpr (D == 3) r = sbdt_pred::in_sphere3_filtered(A, B, p[2], p[3], q.x);
    else r = sbdt_pred::in_sphere2_filtered(A, B, p[2], q.x);
    if (r == 1) return true;
    if (r == 2) {
      const unsigned slot = atomicAdd(a.esc_count, 1u);
      if (slot < a.esc_cap) {
        a.esc[2ull * slot] = static_cast<std::uint32_t>(s);
        a.esc[2ull * slot + 1] = t;
      } else {  // the queue is full: the whole row is decided again after the escalation
        const unsigned bit = 1u << (s & 31u);
        if (!(atomicOr(&a.redo_bits[s >> 5], bit) & bit)) a.redo_rows[atomicAdd(a.redo_count, 1u)] = static_cast<std::uint32_t>(s);
      }
    }
  }
  return false;
}

// Exact policy, hull row: is some point of another part of this leaf cell
// strictly on the outer side of the facet (orient != 0, != inner side)?
template <int D>
__device__ bool cell_points_outside(const BorderArgs& a, unsigned long long idx, const double* const* facet,
                                    int inner_sign, std::uint32_t self) {
  const CellPt<D>* pts = static_cast<const CellPt<D>*>(a.cell_pts);
  const double* q4[D + 1];
#pragma unroll
  for (int j = 0; j < D; ++j) q4[j] = facet[j];
  for (std::uint32_t t = a.cell_start[idx], e = a.cell_start[idx + 1]; t < e; ++t) {
    const CellPt<D> q = pts[t];
    if (q.label == self) continue;
    q4[D] = q.x;
    const int o = orient_dev<D>(q4, a.counters ? a.counters + kCtrOrientExact : nullptr);
    if (o != 0 && o != inner_sign) return true;
  }
  return false;
}

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
  extern __shared__ std::uint64_t s_off_sh[];
  if (threadIdx.x == 0) og = *ogp;
  if (a.k + 1 <= kSmemOffsMax)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  // part offsets in shared memory, or read in place for very large k
  const PartOffs s_off{s_off_sh, a.offsets, a.k + 1 <= kSmemOffsMax};
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
    const std::uint32_t self = s_off.part(a.k, s);
    double p[D + 1][D];
#pragma unroll
    for (int j = 0; j <= D; ++j)
#pragma unroll
      for (int d = 0; d < D; ++d) p[j][d] = a.xyz[std::size_t(v[j]) * D + d];
    if (orientation_exact<D>(p) == 0) atomicOr(a.status, kStDegenerate);
    double c[D], r2;
    circumsphere_inflated<D>(p, c, &r2);
    if (a.spheres) {
#pragma unroll
      for (int d = 0; d < D; ++d) a.spheres[s * (D + 1) + d] = c[d];
      a.spheres[s * (D + 1) + D] = r2;
    }
    const bool pos = (a.policy == SBDT_POLICY_BBOX) ? bbox_policy_sphere<D>(og, a, self, c, r2)
                                                    : og_sphere_hits_foreign<D>(og, a.owner, c, r2, self);
    __stcs(a.positive + s, static_cast<std::uint8_t>(pos ? 1 : 0));
    if (pos)
#pragma unroll
      for (int j = 0; j <= D; ++j) a.vflags[v[j]] = 1;
  }
}

// Grid policy, two kernels joined by a global candidate queue:
//   A  k_border_prefilter, one thread per row: binary32 enclosing sphere with
//      an a-posteriori error bound, then
//        - negative if its cell range sits in one window (cell, 3^D or 5^D
//          neighbourhood) whose combined code is EMPTY or self;
//        - positive if the conservative INNER ball reaches the cell of its
//          centre and that cell holds another part;
//        - otherwise the row is appended to the candidate queue.
//      Rows that reference kInfiniteVertex go to the halfspace queue.
//   C  k_border_exact, warps pull 32 candidates at a time: the reference's
//      binary64 circumsphere (exact operation order), then the cells of its
//      range are tested as one flattened (candidate, cell) stream over the
//      32 lanes (no per-candidate serial loop, no CTA barriers); wide ranges
//      use the two-level cooperative scan, huge ones the pyramid descent.
// A only concludes for spheres that contain / are contained in the exact
// binary64 sphere, so the flags equal the exact test's.
constexpr int kExactWarps = 4;
// candidate-queue reach value of a row whose binary32 sphere failed: the
// exact stage checks its exact orientation (DegenerateSimplex, geometry.cpp:281)
constexpr float kReachCheckOrient = -2.f;
constexpr unsigned kQChunk = 64;              // candidate-queue slots claimed per warp at a time
constexpr std::uint32_t kNoRow = 0xFFFFFFFFu;  // unused (hole) candidate-queue slot

template <int D>
__device__ __forceinline__ void load_simplex(const BorderArgs& a, const std::uint32_t* v, double (*p)[D]) {
#pragma unroll
  for (int j = 0; j <= D; ++j)
#pragma unroll
    for (int d = 0; d < D; ++d) p[j][d] = __ldg(a.xyz + std::size_t(v[j]) * D + d);
}

// Per-launch constants of the prefilter's decision (registers, not the
// shared OwnerGrid: the hot loop reads them every row).
template <int D>
struct PfConst {
  const std::uint64_t* field;  // window field + foreign mask (k_field_tiles), linear over ldims[0]
  int ctop[D];                 // kFloorBias + ldims[0][d] - 1
  unsigned dim0, dim1;         // ldims[0][0], ldims[0][1] (linear index)
  float inv_e, margin_c, lo_mag;
  bool pos_ok;                 // positive proofs allowed (cell boxes within binary32 reach)
  bool contain;                // exact policy: a proof needs a foreign cell INSIDE the inner ball (its points
                               // then lie strictly inside the circumsphere), not only overlapping it
};

// candidate record's outer-ball slot: the foreign mask does not apply (the
// centre cell's field code is not the row's part, or the centre is outside
// the grid); -1: it applies for positive proofs only (range wider than 3^D)
constexpr float kRoutNoMask = -2.f;
// prefilter's half-width of the conservative cell range around its centre
// cell, unknown (range beyond binary32 floor reach): such rows and those
// with need > kFlatHalf go straight to the wide queue
constexpr int kNeedUnknown = 1 << 20;
constexpr int kFlatHalf = 3;      // need <= 3: every axis spans <= 7 cells (the flattened scan)
constexpr int kWideHeavyNeed = 8;  // need > 8: spans > 17 cells, the pyramid rows (queued first)

// floor_small(x) + kFloorBias: the bits of x + 1.5 * 2^23 rounded down
constexpr int kFloorBias = 0x4B400000;

// Prefilter decision for one finite row from its binary32 sphere:
// 0 negative, 1 positive, 2 exact stage. One field word (k_field_tiles) at
// the cell cc of the sphere's centre (clamped into the grid):
//   negative: the conservative cell range of the enclosing ball (binary32
//     cell units with explicit slack, a superset of the exact stage's leaf
//     range, clipped to the grid) lies in the (2h+1)^D window around cc for
//     some h < hs whose non-empty cells are all owned by `self`;
//   positive: the INNER ball (inside the binary64 sphere, checked in
//     binary64) reaches the cell of its centre, which holds another part.
// For an undecided row (2) the cell-unit centre U and the inner ball's reach
// are stored in out_U / out_reach (reach < 0: no positive proof possible) for
// the exact stage's neighbour test (octant_proof).
template <int D>
__device__ __forceinline__ int prefilter_decide(const PfConst<D>& pc, const Sphere32<D>& sp, std::uint32_t self,
                                                const std::uint64_t f64, float* out_U, float* out_reach,
                                                float* out_rout, std::uint32_t* out_mask, int* out_need,
                                                float* out_rp) {
  // (straight-line: every test is evaluated and the outcome selected at the
  // end; the row's field word f64 = field[cc] was loaded by prefilter_fast_negative)
  // R >= radius of the inflated binary64 sphere + distance between centres
  float slack = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) slack = fmaxf(slack, fabsf(sp.P0[d]) + fabsf(sp.rel[d]));
  slack = (slack + pc.lo_mag) * 1e-15f;
  const float R = fmaf(fmaf(sp.r, 1.000004f, 2.01f * sp.e), 1.000001f, slack);
  const float Rc = fmaf(R * pc.inv_e, 1.000001f, pc.margin_c);
  float Uc[D], um = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    Uc[d] = (sp.P0[d] + sp.rel[d]) * pc.inv_e;
    um = fmaxf(um, fabsf(Uc[d]));
  }
  // rounding of Uc (three roundings of |Uc|) and of Uc -/+ Rp: below 4e-7 (|Uc| + Rc)
  const float sl = fmaf(4e-7f, um + Rc, 1e-6f);
  const float Rp = Rc + sl;
  const bool ok = um + Rp < 4194304.f;  // within floor_small's range (false for NaN)
  int need = 0, cb[D];
  bool inside = ok;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float u = ok ? Uc[d] : 0.f;
    const int a = max(__float_as_int(__fadd_rd(u - Rp, 12582912.f)), kFloorBias);
    const int b = min(__float_as_int(__fadd_rd(u + Rp, 12582912.f)), pc.ctop[d]);
    const int c0 = __float_as_int(__fadd_rd(u, 12582912.f));
    const int cc = min(max(c0, kFloorBias), pc.ctop[d]);
    inside = inside && c0 == cc;
    need = max(need, max(cc - a, b - cc));
    cb[d] = cc - kFloorBias;
  }
  const std::uint32_t fw = static_cast<std::uint32_t>(f64);
  const std::uint32_t code = fw & 0xFFFFu;
  const int hs = static_cast<int>(fw >> 24);
  *out_mask = static_cast<std::uint32_t>(f64 >> 32);
  *out_need = ok ? need : kNeedUnknown;
  const bool neg = ok && code == self && need < hs;
  // Positive proof, in binary32 cell units: cc = floor(Uc) holds Uc, the
  // real centre lies within sqrt(D) sl of Uc, and the cell box in cell units
  // is [cc, cc + 1] up to the binary64 rounding of cell_lo (< 1e-7 cells
  // while (|lo| / edge + dims) < 2^26, checked by the caller through pos_ok).
  // If the inner ball, shrunk by the exact stage's margin, still reaches that
  // box, the binary64 box test on the binary64 sphere accepts it. The same
  // holds for every other cell whose box is within the remaining reach of Uc
  // (the foreign-mask test and the binary32 cell scan).
  const float rin_c = ((sp.r * 0.999996f - 2.01f * sp.e * 1.000001f) * 0.999999f - slack) * pc.inv_e * 0.999998f;
  const float reach = rin_c - pc.margin_c - 1.7321f * sl - 2e-7f;
  const bool can_pos = inside && pc.pos_ok && reach > 0.f;
  // The window of radius hs (1 <= hs <= H) around cc is MULTI: it holds an
  // occupied cell of another part. Grid policy: if the inner ball reaches
  // even the nearest point of the window's farthest cell (per axis
  // hs - 1 + max(f, 1 - f)), it overlaps that cell. Exact policy: the inner
  // ball must contain the whole window (far corners: hs + max(f, 1 - f)), so
  // that cell's points lie strictly inside the circumsphere; likewise the
  // centre cell (far corner: max(f, 1 - f)).
  float dd = 0.f, dc = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float f = Uc[d] - static_cast<float>(cb[d]);  // exact when inside: cb = floor(Uc)
    const float mf = fmaxf(f, 1.f - f);
    const float m = mf + static_cast<float>(pc.contain ? hs : hs - 1);
    dd = fmaf(m, m, dd);
    dc = fmaf(mf, mf, dc);
  }
  const float reach2 = reach * reach;
  const bool pos_centre = !(fw & kFieldEmptyBit) && code != self &&  // non-empty, another part or MULTI
                          (!pc.contain || dc * 1.000002f + 1e-6f < reach2);
  const bool pos_window = hs >= 1 && hs <= field_h<D>() && dd * 1.000002f + 1e-6f < reach2;
  const bool pos = !neg && can_pos && (pos_centre || pos_window);
  // the record for the neighbour proofs and the cell scans (centre inside the grid)
#pragma unroll
  for (int d = 0; d < D; ++d) out_U[d] = Uc[d];
  *out_rp = inside ? Rp : -1.f;
  *out_rout = (inside && code == self) ? (need <= 1 ? Rp : -1.f) : kRoutNoMask;
  *out_reach = can_pos ? reach : -1.f;
  return neg ? 0 : (pos ? 1 : 2);
}

// The prefilter's pass over EVERY row: only the negative proof of
// prefilter_decide, with an upper bound of its `need` that costs one floor
// instead of two per axis; loads the field word *out_f64 = field[cc]. A row it
// does not prove negative is deferred to the warp's batch, where
// prefilter_decide runs in full on the recorded sphere (so the outcome of
// every row is the one prefilter_decide gives: this pass only accepts rows
// that prefilter_decide would also call negative).
//   With the centre inside the grid (cc = floor(u), f = u - cc exact) and
//   d = 6e-8 (|u| + Rp) >= the rounding of u -/+ Rp:
//     floor(fl(u + Rp)) - cc <= floor(f + Rp + d),
//     cc - floor(fl(u - Rp))  = ceil(Rp - f + d) <= floor(Rp + (1 - f) + d),
//   and clipping the range to the grid only shrinks it, so
//     need <= floor(Rp + max_d max(f_d, 1 - f_d) + d) =: need_u
//   (evaluated with 3e-7 (um + Rp) + 1e-6 for d and the roundings of the sum).
template <int D>
__device__ __forceinline__ bool prefilter_fast_negative(const PfConst<D>& pc, const Sphere32<D>& sp,
                                                        std::uint32_t self, std::uint64_t* out_f64) {
  // (the same expressions as prefilter_decide up to Rp and cc)
  float slack = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) slack = fmaxf(slack, fabsf(sp.P0[d]) + fabsf(sp.rel[d]));
  slack = (slack + pc.lo_mag) * 1e-15f;
  const float R = fmaf(fmaf(sp.r, 1.000004f, 2.01f * sp.e), 1.000001f, slack);
  const float Rc = fmaf(R * pc.inv_e, 1.000001f, pc.margin_c);
  float Uc[D], um = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    Uc[d] = (sp.P0[d] + sp.rel[d]) * pc.inv_e;
    um = fmaxf(um, fabsf(Uc[d]));
  }
  const float sl = fmaf(4e-7f, um + Rc, 1e-6f);
  const float Rp = Rc + sl;
  const bool ok = um + Rp < 4194304.f;  // within floor_small's range (false for NaN)
  int cb[D];
  bool inside = ok;
  float mfm = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float u = ok ? Uc[d] : 0.f;
    const int c0 = __float_as_int(__fadd_rd(u, 12582912.f));
    const int cc = min(max(c0, kFloorBias), pc.ctop[d]);
    inside = inside && c0 == cc;
    cb[d] = cc - kFloorBias;
    // (cc carries the bits of 1.5 * 2^23 + cb: cb as a float without an I2F)
    const float f = u - (__int_as_float(cc) - 12582912.f);  // exact when inside
    mfm = fmaxf(mfm, fmaxf(f, 1.f - f));
  }
  unsigned long long li;
  if constexpr (D == 3)
    li = static_cast<unsigned long long>(static_cast<unsigned>(cb[1]) + pc.dim1 * static_cast<unsigned>(cb[2])) * pc.dim0 +
         static_cast<unsigned>(cb[0]);
  else
    li = static_cast<unsigned long long>(static_cast<unsigned>(cb[1])) * pc.dim0 + static_cast<unsigned>(cb[0]);
  const std::uint64_t f64 = __ldg(pc.field + li);
  *out_f64 = f64;
  const std::uint32_t fw = static_cast<std::uint32_t>(f64);
  // (hs <= H + 1: any bound >= 8 reads as "too wide")
  const int need_u = floor_small(fminf(fmaf(um + Rp, 3e-7f, mfm + Rp) + 1e-6f, 8.f));
  return inside && (fw & 0xFFFFu) == self && need_u < static_cast<int>(fw >> 24);
}

// The neighbours of the centre cell c0 = floor(U) on the near side of U in
// each axis (the 2^D - 1 cells of the octant U lies in; the far ones are at
// least half a cell further): positive if one holds another part and its box
// is within `reach` (cell units, all error slack already subtracted, see
// prefilter_decide) of U.
template <int D>
__device__ __forceinline__ bool octant_proof(const OwnerGrid<D>& og, const BorderArgs& a, const float* U, float reach,
                                             std::uint32_t self) {
  if (!(reach > 0.f)) return false;
  const float reach2 = reach * reach;
  int c0[D], side[D];
  float gap[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    c0[d] = floor_small(U[d]);  // U lies in the grid (checked when reach was recorded)
    const float f = U[d] - static_cast<float>(c0[d]);
    side[d] = f < 0.5f ? -1 : 1;
    gap[d] = f < 0.5f ? f : 1.f - f;
  }
  // all the neighbours' field words are loaded before any is tested (one
  // memory latency instead of up to 2^D - 1 in a row)
  std::uint32_t fw[(1 << D) - 1];
#pragma unroll
  for (int k = 1; k < (1 << D); ++k) {
    int cn[D];
    float d2 = 0.f;
    bool ok = true;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const bool move = (k >> d) & 1;
      cn[d] = c0[d] + (move ? side[d] : 0);
      ok = ok && cn[d] >= 0 && cn[d] < og.ldims[0][d];
      d2 += move ? gap[d] * gap[d] : 0.f;
    }
    unsigned long long li = static_cast<unsigned>(cn[D - 1]);
#pragma unroll
    for (int d = D - 2; d >= 0; --d) li = li * static_cast<unsigned>(og.ldims[0][d]) + static_cast<unsigned>(cn[d]);
    fw[k - 1] = (ok && d2 * 1.000002f + 1e-12f < reach2) ? static_cast<std::uint32_t>(__ldg(a.field + li)) : kFieldEmptyBit;
  }
  bool hit = false;
#pragma unroll
  for (int k = 0; k < (1 << D) - 1; ++k) hit = hit || (!(fw[k] & kFieldEmptyBit) && (fw[k] & 0xFFFFu) != self);
  return hit;
}

// The centre cell's foreign mask m (k_field_tiles; the row's part is the
// cell's field code, checked by the prefilter): 1 if the inner ball (reach,
// all error slack already subtracted) reaches the box of a foreign
// neighbour (exact policy: contains it, so that its points lie strictly
// inside the circumsphere), 0 if the outer ball (rout > 0: radius in cell units with every
// slack, its cell range inside the 3^D window) stays strictly away from all
// of them, -1 undecided. Box distances in cell units from U, whose cell is
// c0 = floor(U): per axis the gap to the neighbour at offset -1, 0, +1 is
// f, 0, 1 - f (f = U - c0).
template <int D>
__device__ __forceinline__ int exact_mask_test(const std::uint32_t m, const float* U, float reach, float rout,
                                               bool contain) {
  // per axis, for the neighbour offsets -1, 0, +1: the squared box gap to U
  // (f, 0, 1 - f) and, for the exact policy's containment proof, the squared
  // far-corner distance (1 + f, max(f, 1 - f), 2 - f)
  float g[D][3], h[D][3];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float f = U[d] - static_cast<float>(floor_small(U[d]));  // exact
    g[d][0] = f * f;
    g[d][1] = 0.f;
    g[d][2] = (1.f - f) * (1.f - f);
    const float mf = fmaxf(f, 1.f - f);
    h[d][0] = (1.f + f) * (1.f + f);
    h[d][1] = mf * mf;
    h[d][2] = (2.f - f) * (2.f - f);
  }
  if (!m) return rout > 0.f ? 0 : -1;
  // smallest squared box gap (mn) and, under the exact policy only
  // (`contain` is uniform over the launch), far-corner distance (mx) over
  // the foreign neighbours
  auto smallest = [&](const float (*t)[3]) {
    float r = INFINITY;
    if constexpr (D == 3) {
#pragma unroll
      for (int o2 = 0; o2 < 3; ++o2)
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1) {
          const float s12 = t[1][o1] + t[2][o2];
#pragma unroll
          for (int o0 = 0; o0 < 3; ++o0)
            if ((m >> (o0 + 3 * o1 + 9 * o2)) & 1u) r = fminf(r, t[0][o0] + s12);
        }
    } else {
#pragma unroll
      for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
        for (int o0 = 0; o0 < 3; ++o0)
          if ((m >> (o0 + 3 * o1)) & 1u) r = fminf(r, t[0][o0] + t[1][o1]);
    }
    return r;
  };
  const float mn = smallest(g);
  float mx = INFINITY;
  if (contain) mx = smallest(h);
  // (a few binary32 roundings of the squared distances, far inside the margins)
  const float prove = contain ? mx : mn;
  if (reach > 0.f && prove * 1.000002f + 1e-12f < reach * reach) return 1;
  if (rout > 0.f && mn * 0.99999f - 1e-6f > rout * rout) return 0;
  return -1;
}

// Rows are claimed by warps in chunks of kPfChunk from a launch-wide cursor
// (instead of a static grid-stride split): every warp works on the same
// sliding window of rows, so the packed-coordinate lines and field words of
// the 1-2 partitions in flight stay in L2 instead of spreading over the rows
// of warps that drifted apart, and a lane's consecutive rows are 32 apart
// (vertices shared by neighbouring rows hit in L1).
#ifndef PF_ITERS
#define PF_ITERS 8
#endif
constexpr unsigned kPfIters = PF_ITERS;
constexpr unsigned kPfBatch = 64;  // per-warp batch of undecided rows (< 32 waiting + 32 arriving)
template <int D>
constexpr int kPfBatchWords = 3 * D + 7;
constexpr unsigned kPfChunk = 32 * kPfIters;

template <int D, bool BIGK>
__global__ void __launch_bounds__(kPfThreads, PF_CTAS) k_border_prefilter(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp,
                                                                std::uint32_t* __restrict__ cand, std::uint64_t cap,
                                                                unsigned* __restrict__ ncand, std::uint64_t row_begin,
                                                                std::uint64_t row_end,
                                                                unsigned long long* __restrict__ cursor,
                                                                std::uint32_t* __restrict__ wq, std::uint64_t wcap,
                                                                unsigned* __restrict__ nwide,
                                                                unsigned* __restrict__ nwlight,
                                                                std::uint32_t* __restrict__ sq, std::uint64_t scap,
                                                                unsigned* __restrict__ nsq) {
  __shared__ OwnerGrid<D> og;
  extern __shared__ std::uint64_t s_off_sh[];
  if (threadIdx.x == 0) og = *ogp;
  if constexpr (!BIGK)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  // part offsets in shared memory, or read in place for very large k (BIGK)
  const std::uint64_t* s_off = BIGK ? a.offsets : s_off_sh;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  // rows [row_begin, row_end); every warp iterates over its own claimed
  // chunks (no CTA barrier: the batch flushes make warps uneven), with one
  // chunk of lookahead for the id prefetch
  __shared__ std::uint32_t s_bat[kPfThreads / 32][kPfBatchWords<D>][kPfBatch];
  __shared__ std::uint32_t s_ids[kPfThreads / 32][D + 1][32];  // the next row's vertex ids, per lane
  unsigned long long claim = 0;
  if (lane == 0) claim = atomicAdd(cursor, 2ull * kPfChunk);
  claim = __shfl_sync(0xffffffffu, claim, 0);
  const std::uint64_t base = row_begin + claim;
  const std::uint64_t next_base = base + kPfChunk;
  unsigned it = 0;
  // binary32 cell-unit scale and margin (rounded up; the slacks cover the rest)
  // decode_row's coordinate unit: the fixed-point step in 3-D, 1 in 2-D
  PfConst<D> pc;
  {
    const double unit = D == 3 ? og.qh : 1.0;
    pc.field = a.field;
    pc.inv_e = static_cast<float>(og.inv_edge * unit);
    pc.margin_c = static_cast<float>(og.margin * og.inv_edge) * 1.0001f + 1e-30f;
    pc.lo_mag = 0.f;
    pc.pos_ok = true;
    pc.contain = a.exact != 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      pc.lo_mag = fmaxf(pc.lo_mag, static_cast<float>(fabs(og.g.lo[d]) / unit) * 1.0001f);
      pc.pos_ok = pc.pos_ok && fabs(og.g.lo[d]) * og.inv_edge + static_cast<double>(og.ldims[0][d]) < 67108864.0;
      pc.ctop[d] = kFloorBias + og.ldims[0][d] - 1;
    }
    pc.dim0 = static_cast<unsigned>(og.ldims[0][0]);
    pc.dim1 = static_cast<unsigned>(og.ldims[0][1]);
  }
  // Row bookkeeping in 32 bits (S < 2^32, capi.cu): a chunk is its first row
  // and its number of rows inside [row_begin, row_end) (0: past the end).
  auto span = [&](std::uint64_t b, std::uint32_t& first, std::uint32_t& count) {
    const std::uint64_t left = b < row_end ? row_end - b : 0ull;
    count = static_cast<std::uint32_t>(left < kPfChunk ? left : kPfChunk);
    first = static_cast<std::uint32_t>(b);
  };
  std::uint32_t c_first, c_count, n_first, n_count;
  span(base, c_first, c_count);
  span(next_base, n_first, n_count);
  const std::uint32_t last_row = static_cast<std::uint32_t>(row_end ? row_end - 1 : 0);
  // software pipeline: the vertex ids of the next row are in flight while
  // this row's coordinates are gathered and tested
  std::uint32_t s = c_first + lane;  // this lane's row
  bool valid = lane < c_count;
  std::uint32_t self = part_of(s_off, a.k, valid ? s : last_row);
  auto part_end = [&](std::uint32_t p) -> std::uint32_t {  // first row of the next part
    return p + 1 < a.k ? static_cast<std::uint32_t>(s_off[p + 1]) : 0xFFFFFFFFu;
  };
  std::uint32_t next_off = part_end(self);
  // (asynchronous copies into a per-warp staging area: LDGSTS, no destination
  // registers held across the row's work; each lane stages and reads its own
  // row, so cp.async.wait_group is the only synchronisation)
  std::uint32_t(&I)[D + 1][32] = s_ids[threadIdx.x >> 5];
  auto stage_ids = [&](std::uint32_t r, bool ok) {
    if (ok) {
#pragma unroll
      for (int j = 0; j <= D; ++j) {
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&I[j][lane]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(a.verts + r + std::uint64_t(j) * a.S)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage_ids(s, valid);
  // candidate-queue slots are claimed per warp in chunks of kQChunk (one
  // atomic per chunk instead of one per iteration on the single counter);
  // the slots a warp leaves unused at exit are written as kNoRow holes
  unsigned qbase = 0, qleft = 0;
  auto append = [&](bool want, std::uint32_t row, float reach) {
    const unsigned mc = __ballot_sync(0xffffffffu, want);
    const unsigned nc = __popc(mc);
    if (!nc) return;
    unsigned nbase = 0;
    if (lane == 0 && nc > qleft) nbase = atomicAdd(ncand, kQChunk);
    nbase = __shfl_sync(0xffffffffu, nbase, 0);
    const unsigned rank = __popc(mc & lt);
    const unsigned q = rank < qleft ? qbase + rank : nbase + (rank - qleft);
    if (nc > qleft) {  // the current chunk is used up, the rest goes to the new one
      qbase = nbase + (nc - qleft);
      qleft = kQChunk - (nc - qleft);
    } else {
      qbase += nc;
      qleft -= nc;
    }
    if (want) {
      cand[q] = row;
      cand[cap + q] = __float_as_uint(reach);
    }
  };
  // Rows the fast pass does not prove negative wait in a per-warp batch
  // (shared memory) until 32 have gathered; then every lane takes one and
  // runs, converged, the full decision (prefilter_decide on the recorded
  // sphere and field word) and, for the rows it leaves open, the binary32
  // neighbour proofs (foreign mask / near-octant codes); only the rows those
  // leave open go to the queues of the later stages.
  // {row, self, r, e (< 0: no binary32 sphere), field word lo/hi, P0[D], rel[D], vertex ids[D + 1]}
  std::uint32_t(&B)[kPfBatchWords<D>][kPfBatch] = s_bat[threadIdx.x >> 5];
  unsigned bcount = 0;
  auto flush_batch = [&](unsigned nproc) {
    __syncwarp();
    const unsigned e = bcount - nproc + lane;
    bool to_q = false, to_w = false, to_s = false;
    std::uint32_t row = 0, ids[D + 1];
    float reach = -1.f, crp = -1.f, cU[D];
    int cneed = kNeedUnknown;
#pragma unroll
    for (int d = 0; d < D; ++d) cU[d] = 0.f;
#pragma unroll
    for (int j = 0; j <= D; ++j) ids[j] = 0;
    if (lane < nproc) {
      row = B[0][e];
      const std::uint32_t bself = B[1][e];
#pragma unroll
      for (int j = 0; j <= D; ++j) ids[j] = B[6 + 2 * D + j][e];
      Sphere32<D> sp;
      sp.r = __uint_as_float(B[2][e]);
      sp.e = __uint_as_float(B[3][e]);
      float rout = kRoutNoMask;
      std::uint32_t cmask = 0;
      int res = 2;
      if (sp.e >= 0.f) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
          sp.P0[d] = __uint_as_float(B[6 + d][e]);
          sp.rel[d] = __uint_as_float(B[6 + D + d][e]);
        }
        const std::uint64_t f64 = static_cast<std::uint64_t>(B[4][e]) | (static_cast<std::uint64_t>(B[5][e]) << 32);
        res = prefilter_decide<D>(pc, sp, bself, f64, cU, &reach, &rout, &cmask, &cneed, &crp);
      } else {
        reach = kReachCheckOrient;  // no binary32 sphere: the exact orientation decides degeneracy
      }
      if (a.counters && res == 1) atomicAdd(&a.counters[8], 1ull);
      // the centre cell's foreign mask (no loads: it came with the field
      // word), else (the centre's field code is not the row's part) the
      // near-octant neighbours' codes
      int r = res == 2 ? -1 : res;
      if (res == 2) {
        if (rout >= -1.f)
          r = exact_mask_test<D>(cmask, cU, reach, rout, a.exact != 0);
        else if (reach > 0.f && !a.exact)  // (overlap-based: grid policy only)
          r = octant_proof<D>(og, a, cU, reach, bself) ? 1 : -1;
        if (a.counters && r >= 0) atomicAdd(&a.counters[r == 1 ? 10 : 15], 1ull);
      }
      if (r >= 0) {
        __stcs(a.positive + row, static_cast<std::uint8_t>(r));
        if (r == 1)
#pragma unroll
          for (int j = 0; j <= D; ++j) a.vflags[ids[j]] = 1;
      } else if (reach != kReachCheckOrient && cneed > kFlatHalf) {
        to_w = true;  // wide cell range: the pyramid descent (k_border_wide), next to the exact stage
      } else if (sq && reach != kReachCheckOrient && crp > 0.f) {
        to_s = true;  // the binary32 cell scan (k_border_scan32)
      } else {
        to_q = true;
        if (reach > 0.f) reach = -1.f;  // the exact stage only needs the kReachCheckOrient marker
      }
    }
    {
      const unsigned ms = __ballot_sync(0xffffffffu, to_s);
      if (ms) {
        unsigned sb = 0;
        if (lane == 0) sb = atomicAdd(nsq, static_cast<unsigned>(__popc(ms)));
        sb = __shfl_sync(0xffffffffu, sb, 0);
        if (to_s) {
          const std::uint64_t qs = sb + __popc(ms & lt);
          sq[qs] = row;
#pragma unroll
          for (int d = 0; d < D; ++d) sq[std::uint64_t(1 + d) * scap + qs] = __float_as_uint(cU[d]);
          sq[std::uint64_t(D + 1) * scap + qs] = __float_as_uint(crp);
          sq[std::uint64_t(D + 2) * scap + qs] = __float_as_uint(reach);
        }
      }
    }
    // wide rows: {row, vertex ids}, heavy ones from the front of the queue,
    // the others from the back when the queue is split (device path)
    {
      const bool heavy = to_w && (!nwlight || cneed > kWideHeavyNeed);
      const bool light = to_w && !heavy;
      const unsigned mh = __ballot_sync(0xffffffffu, heavy), ml = __ballot_sync(0xffffffffu, light);
      if (mh | ml) {
        unsigned hb = 0, lb = 0;
        if (lane == 0) {
          if (mh) hb = atomicAdd(nwide, static_cast<unsigned>(__popc(mh)));
          if (ml) lb = atomicAdd(nwlight, static_cast<unsigned>(__popc(ml)));
        }
        hb = __shfl_sync(0xffffffffu, hb, 0);
        lb = __shfl_sync(0xffffffffu, lb, 0);
        if (to_w) {
          const std::uint64_t q = heavy ? hb + __popc(mh & lt) : wcap - 1 - (lb + __popc(ml & lt));
          wq[q] = row;
#pragma unroll
          for (int j = 0; j <= D; ++j) wq[std::uint64_t(j + 1) * wcap + q] = ids[j];
          // the recorded cell-unit centre and inner reach (exact policy: blocks inside it are accepted)
#pragma unroll
          for (int d = 0; d < D; ++d) wq[std::uint64_t(D + 2 + d) * wcap + q] = __float_as_uint(cU[d]);
          wq[std::uint64_t(2 * D + 2) * wcap + q] = __float_as_uint(reach);
        }
      }
    }
    bcount -= nproc;
    __syncwarp();
    append(to_q, row, reach);
  };
  while (c_count) {
    std::uint32_t v[D + 1];
    std::uint64_t w[D + 1];
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = valid ? I[j][lane] : kInfVertex;
    // the next row of this lane: the next 32 of the chunk, or the lookahead chunk
    const bool same = it + 1 < kPfIters;
    const std::uint32_t li_next = same ? (it + 1) * 32u + lane : lane;  // its index inside that chunk
    const std::uint32_t s_next = (same ? c_first : n_first) + li_next;
    const bool valid_next = li_next < (same ? c_count : n_count);
    stage_ids(s_next, valid_next);
    const bool inf = valid && v[D] == kInfVertex;
    // a warp's rows only grow (claims are monotonic): advance the part cursor
    {
      const std::uint32_t sc = valid ? s : last_row;
      while (next_off <= sc) {
        ++self;
        next_off = part_end(self);
      }
    }
    bool is_cand = false;
    Sphere32<D> sp;
    std::uint64_t f64 = 0;
    if (valid && !inf) {
      float A[D][D], P0e[D], eta;
      gather_row<D>(a.xq, v, a.n, w);
      decode_row<D>(w, A, sp.P0, P0e, &eta);
      // a binary32 sphere with its bound proves |det| > 0 (the orientation
      // of the binary64 vertices is nonzero); rows without one are checked
      // with the exact orientation in the exact stage (kReachCheckOrient)
      bool neg = false;
      if (enclosing_sphere_f32<D>(A, eta, P0e, sp))
        neg = prefilter_fast_negative<D>(pc, sp, self, &f64);
      else
        sp.e = -1.f;
      if (neg)
        __stcs(a.positive + s, static_cast<std::uint8_t>(0));
      else
        is_cand = true;
    }
    // deferred rows into the warp's batch
    {
      const unsigned mb = __ballot_sync(0xffffffffu, is_cand);
      if (is_cand) {
        const unsigned slot = bcount + __popc(mb & lt);
        B[0][slot] = s;
        B[1][slot] = self;
        B[2][slot] = __float_as_uint(sp.r);
        B[3][slot] = __float_as_uint(sp.e);
        B[4][slot] = static_cast<std::uint32_t>(f64);
        B[5][slot] = static_cast<std::uint32_t>(f64 >> 32);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          B[6 + d][slot] = __float_as_uint(sp.P0[d]);
          B[6 + D + d][slot] = __float_as_uint(sp.rel[d]);
        }
#pragma unroll
        for (int j = 0; j <= D; ++j) B[6 + 2 * D + j][slot] = v[j];
      }
      bcount += __popc(mb);
      if (bcount >= 32) flush_batch(32);
    }
    // hull rows
    {
      const unsigned mi = __ballot_sync(0xffffffffu, inf);
      if (mi) {
        unsigned bi = 0;
        if (lane == 0) bi = atomicAdd(a.inf_count, static_cast<unsigned>(__popc(mi)));
        bi = __shfl_sync(0xffffffffu, bi, 0);
        if (inf) a.inf_queue[bi + __popc(mi & lt)] = s;
      }
    }
    s = s_next;
    valid = valid_next;
    if (++it == kPfIters) {  // warp-uniform
      it = 0;
      unsigned long long c2 = 0;
      if (lane == 0) c2 = atomicAdd(cursor, static_cast<unsigned long long>(kPfChunk));
      c_first = n_first;
      c_count = n_count;
      span(row_begin + __shfl_sync(0xffffffffu, c2, 0), n_first, n_count);
    }
  }
  if (bcount) flush_batch(bcount);
  for (unsigned i = lane; i < qleft; i += 32) cand[qbase + i] = kNoRow;
  if (a.counters && lane == 0 && qleft) atomicAdd(&a.counters[11], static_cast<unsigned long long>(qleft));
}

// per-lane candidate record for the flattened scan (shared memory, per warp)
// Term of axis d's cell coordinate in the level-0 tiled index (og_index is
// the sum over the axes plus loff[0]).
template <int D>
__device__ __forceinline__ unsigned long long cell_off(int cell, int d, const unsigned long long* bst, bool multi) {
  constexpr int SH = og_shift<D>();
  constexpr int F = og_fan<D>();
  return multi ? (static_cast<unsigned long long>(cell >> SH) * bst[d]) * 64ull +
                     (static_cast<unsigned long long>(cell & (F - 1)) << (SH * d))
               : 0ull;
}

template <int D>
struct CandSlot {
  // per axis and cell of the range: the squared gap to the centre, so
  // box_sphere's d2 is ((g0^2 + g1^2) + g2^2) exactly as box_sphere forms it;
  // the cell's term of the level-0 tiled index is recomputed from lo
  double g2[D][kFlatSpan];
  double r2;
  int lo[D];
  unsigned span[D];
  unsigned inv[D];  // ceil(2^16 / span)
  unsigned self;
  unsigned excl;    // first position of this candidate in the flattened stream
  unsigned row;     // simplex row (exact policy: reload its vertices for the point tests)
  unsigned qi;      // its queue position
};

// Candidates from the prefilter; rows with wide cell ranges (modes 2, 3) are
// forwarded to the wide queue (k_border_wide).
template <int D, bool Ex>
__global__ void __launch_bounds__(kExactWarps * 32, 6) k_border_exact(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp,
                                                                   const std::uint32_t* __restrict__ cand,
                                                                   std::uint64_t cap,
                                                                   const unsigned* __restrict__ ncand_p,
                                                                   unsigned* __restrict__ next,
                                                                   std::uint32_t* __restrict__ wide,
                                                                   unsigned* __restrict__ nwide,
                                                                   unsigned* __restrict__ fin,
                                                                   unsigned* __restrict__ nlight) {
  __shared__ OwnerGrid<D> og;
  __shared__ CandSlot<D> slots[kExactWarps][32];
  __shared__ unsigned char nzl[kExactWarps][32];
  extern __shared__ std::uint64_t s_off_sh[];
  if (threadIdx.x == 0) og = *ogp;
  if (a.k + 1 <= kSmemOffsMax)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  // part offsets in shared memory, or read in place for very large k
  const PartOffs s_off{s_off_sh, a.offsets, a.k + 1 <= kSmemOffsMax};
  const unsigned ncand = *ncand_p;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned wid = threadIdx.x >> 5;
  CandSlot<D>* sl = slots[wid];
  const bool multi_level = og.levels > 1;
  unsigned long long bst[D];  // level-1 block strides of the tiled level-0 index
  bst[0] = 1;
#pragma unroll
  for (int d = 1; d < D; ++d) bst[d] = bst[d - 1] * static_cast<unsigned long long>(multi_level ? og.ldims[1][d - 1] : 1);
  const unsigned fd0 = static_cast<unsigned>(og.ldims[0][0]), fd1 = static_cast<unsigned>(og.ldims[0][1]);
  unsigned char* nz = nzl[wid];
  const unsigned full = 0xffffffffu;
  // the next batch is claimed while this one is processed (the atomic's
  // round trip on the shared cursor overlaps the work)
  unsigned base = claim_batch(next);
  for (;;) {
    if (base >= ncand) break;
    unsigned nclaim = 0;
    if (lane == 0) nclaim = atomicAdd(next, 32u);
    const unsigned t = base + lane;
    const std::uint32_t crow = t < ncand ? cand[t] : kNoRow;
    const bool has = crow != kNoRow;
    std::uint64_t s = 0;
    std::uint32_t self = 0, v[D + 1];
    double c[D], r2 = 0.0;
    int lo[D], span[D];
    int mode = 0;  // 0 decided, 1 flattened scan, 2 two-level scan, 3 pyramid descent
    bool pre_pos = false;
    if (has) {
      s = crow;
      self = s_off.part(a.k, s);
#pragma unroll
      for (int j = 0; j <= D; ++j) v[j] = __ldg(a.verts + std::uint64_t(j) * a.S + s);
      // (the binary32 neighbour proofs ran in the prefilter's batches)
      {
        double p[D + 1][D];
        load_simplex<D>(a, v, p);
        circumsphere_inflated<D>(p, c, &r2);
        mode = leaf_range<D>(og, c, r2, lo, span);
      }
    }
    bool pos = pre_pos;
    if (a.counters) {
      const unsigned m1 = __ballot_sync(full, mode == 1);
      if (lane == 0 && m1) atomicAdd(&a.counters[2], static_cast<unsigned long long>(__popc(m1)));
    }
    {
      // forward wide ranges. With nlight, the pyramid rows (mode 3: the
      // costliest descents) fill the queue from the front and the two-level
      // rows from the back, so k_border_wide starts the long ones first.
      const unsigned lt = (1u << lane) - 1u;
      const unsigned mh = __ballot_sync(full, nlight ? mode == 3 : mode >= 2);
      const unsigned ml = nlight ? __ballot_sync(full, mode == 2) : 0u;
      if (mh | ml) {
        unsigned hb = 0, lb = 0;
        if (lane == 0) {
          if (mh) hb = atomicAdd(nwide, static_cast<unsigned>(__popc(mh)));
          if (ml) lb = atomicAdd(nlight, static_cast<unsigned>(__popc(ml)));
        }
        hb = __shfl_sync(full, hb, 0);
        lb = __shfl_sync(full, lb, 0);
        if ((mh >> lane) & 1u || (ml >> lane) & 1u) {
          const std::uint64_t q = ((mh >> lane) & 1u) ? hb + __popc(mh & lt) : cap - 1 - (lb + __popc(ml & lt));
          wide[q] = static_cast<std::uint32_t>(s);
#pragma unroll
          for (int j = 0; j <= D; ++j) wide[std::uint64_t(j + 1) * cap + q] = v[j];
          wide[std::uint64_t(2 * D + 2) * cap + q] = __float_as_uint(-1.f);  // no recorded ball
        }
      }
    }

    // ---- mode 1: flattened stream of (candidate, row) pairs, a row being the
    // cells along axis 0 for fixed (i1, i2); a lane tests its row's <= 5 cells
    // with independent owner-code loads.
    unsigned cnt = 0;
    if (mode == 1) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        // the range lies in the grid (cell + 1 <= dims), so the upper bound of
        // a cell is the lower bound of the next: one cell_lo per boundary
        double bhi = cell_lo<D>(og.g, lo[d], d);
        for (int i = 0; i < span[d]; ++i) {
          const double blo = bhi;
          bhi = cell_lo<D>(og.g, lo[d] + i + 1, d);
          double g = 0.0;
          if (c[d] < blo) g = blo - c[d];
          else if (c[d] > bhi) g = c[d] - bhi;
          sl[lane].g2[d][i] = g * g;
        }
        sl[lane].lo[d] = lo[d];
        sl[lane].span[d] = static_cast<unsigned>(span[d]);
        // ceil(2^16 / span) for span <= kFlatSpan: the correctly rounded
        // binary32 quotient is exact or >= 0.1 away from an integer
        sl[lane].inv[d] = static_cast<unsigned>(ceilf(__fdiv_rn(65536.f, static_cast<float>(span[d]))));
      }
      sl[lane].r2 = r2;
      sl[lane].self = self;
      sl[lane].row = static_cast<unsigned>(s);
      sl[lane].qi = t;
      cnt = D == 3 ? unsigned(span[1] * span[2]) : unsigned(span[1]);
    }
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(full, incl, o);
      if (lane >= static_cast<unsigned>(o)) incl += y;
    }
    const unsigned total = __shfl_sync(full, incl, 31);
    const unsigned excl = incl - cnt;
    const unsigned nzmask = __ballot_sync(full, cnt > 0);
    if (a.counters && lane == 0) atomicAdd(&a.counters[5], static_cast<unsigned long long>(total));
    if (cnt) {
      sl[lane].excl = excl;
      nz[__popc(nzmask & ((1u << lane) - 1u))] = static_cast<unsigned char>(lane);
    }
    __syncwarp();
    unsigned done = 0;
    int cur = -1;
    for (unsigned b0 = 0; b0 < total; b0 += 32) {
      const bool st = cnt && excl >= b0 && excl < b0 + 32;
      const unsigned smask = __reduce_or_sync(full, st ? 1u << (excl - b0) : 0u);
      const unsigned q = b0 + lane;
      bool h = false;
      unsigned cl = 0;
      if (q < total) {
        cl = nz[cur + __popc(smask & ((2u << lane) - 1u))];
        const CandSlot<D>& r = sl[cl];
        const unsigned rem = q - r.excl;
        double g12;  // g1^2 (+ g2^2 added after g0^2, box_sphere's order)
        double g2z = 0.0;
        int c1, c2 = 0;  // the row's cell coordinates on axes 1 (and 2)
        if constexpr (D == 3) {
          const unsigned i2 = (rem * r.inv[1]) >> 16;  // rem / span1 (rem * span1 < 2^16)
          const unsigned i1 = rem - i2 * r.span[1];
          c1 = r.lo[1] + static_cast<int>(i1);
          c2 = r.lo[2] + static_cast<int>(i2);
          g12 = r.g2[1][i1];
          g2z = r.g2[2][i2];
        } else {
          c1 = r.lo[1] + static_cast<int>(rem);
          g12 = r.g2[1][rem];
        }
        const double rr = r.r2;
        const std::uint32_t sf = r.self;
        if constexpr (!Ex) {
          // the row's cells are consecutive words of the linear window field
          // (code of a non-empty cell in the low half-word)
          const unsigned long long lb =
              (D == 3 ? static_cast<unsigned long long>(static_cast<unsigned>(c1) + fd1 * static_cast<unsigned>(c2))
                      : static_cast<unsigned long long>(static_cast<unsigned>(c1))) * fd0 +
              static_cast<unsigned>(r.lo[0]);
          std::uint32_t fw[kFlatSpan];
          bool geo[kFlatSpan];
#pragma unroll
          for (int i0 = 0; i0 < kFlatSpan; ++i0) {
            geo[i0] = false;
            fw[i0] = kFieldEmptyBit;
            if (i0 < static_cast<int>(r.span[0])) {
              double d2 = r.g2[0][i0] + g12;
              if constexpr (D == 3) d2 += g2z;
              geo[i0] = d2 <= rr;
              if (geo[i0]) fw[i0] = static_cast<std::uint32_t>(__ldg(a.field + lb + i0));
            }
          }
#pragma unroll
          for (int i0 = 0; i0 < kFlatSpan; ++i0) h = h || (!(fw[i0] & kFieldEmptyBit) && (fw[i0] & 0xFFFFu) != sf);
        } else {
          const unsigned long long base =
              og.loff[0] + cell_off<D>(c1, 1, bst, multi_level) + (D == 3 ? cell_off<D>(c2, 2, bst, multi_level) : 0ull);
          std::uint16_t code[kFlatSpan];
          bool geo[kFlatSpan];
          unsigned long long cidx[kFlatSpan];
#pragma unroll
          for (int i0 = 0; i0 < kFlatSpan; ++i0) {
            geo[i0] = false;
            code[i0] = kOwnerEmpty;
            cidx[i0] = 0;
            if (i0 < static_cast<int>(r.span[0])) {
              double d2 = r.g2[0][i0] + g12;
              if constexpr (D == 3) d2 += g2z;
              geo[i0] = d2 <= rr;
              cidx[i0] = base + cell_off<D>(r.lo[0] + i0, 0, bst, multi_level);
              if (geo[i0]) code[i0] = __ldg(a.owner + cidx[i0]);
            }
          }
          // exact policy: the points of the foreign overlapping cells
          bool loaded = false;
          double pv[D + 1][D];
          int par = 1;
          for (int i0 = 0; i0 < static_cast<int>(r.span[0]) && !h; ++i0) {
            if (!(geo[i0] && code[i0] != kOwnerEmpty && code[i0] != sf)) continue;
            if (!loaded) {
              std::uint32_t vv[D + 1];
#pragma unroll
              for (int j = 0; j <= D; ++j) vv[j] = __ldg(a.verts + std::uint64_t(j) * a.S + r.row);
              load_simplex<D>(a, vv, pv);
              par = a.parity[r.row];
              loaded = true;
            }
            h = cell_points_inside<D>(a, cidx[i0], pv, par, sf, r.row);
          }
        }
      }
      done |= __reduce_or_sync(full, h ? 1u << cl : 0u);
      cur += __popc(smask);
    }
    if (mode == 1) pos = (done >> lane) & 1u;
    if (a.counters && lane == 0) atomicAdd(&a.counters[7], static_cast<unsigned long long>(__popc(done)));
    __syncwarp();

    if (has && mode < 2) {
      __stcs(a.positive + s, static_cast<std::uint8_t>(pos ? 1 : 0));
      if (pos)
#pragma unroll
        for (int j = 0; j <= D; ++j) a.vflags[v[j]] = 1;
    }
    base = __shfl_sync(full, nclaim, 0);
  }
  rewind_cursor(next, fin, ncand);
}

// Grid policy, flattened cell scan in binary32 (the rows the prefilter's
// neighbour proofs left open, cell range <= kFlatSpan per axis): the
// prefilter's cell-unit centre U, outer radius Rp (every slack included) and
// inner reach (every slack subtracted) decide each cell of the range from
// its box distance to U (box [i, i + 1] per axis in cell units, see
// prefilter_decide): a foreign cell with distance < reach overlaps the
// binary64 sphere (positive), a cell with distance > Rp cannot; a foreign
// cell in between (a shell of relative width ~1e-5) sends the row to the
// binary64 exact stage (k_border_exact). No vertex or coordinate loads for
// the rows decided here, except the vertex ids of the positive ones.
// Queue: SoA {row, U[D], Rp, reach}.
constexpr int kScanWarps = 4;

template <int D, bool Ex>
struct ScanBalls {};  // grid policy: the cell-unit balls only
template <int D>
struct ScanBalls<D, true> {
  double c64[D];  // exact policy: U in coordinates, and the two radii squared in coordinate units
  double pin2, pout2;
};

template <int D, bool Ex>
struct ScanSlot : ScanBalls<D, Ex> {
  float g2[D][kFlatSpan];  // squared box gaps to U per axis and cell of the range
  float rin2, rout2;       // reach^2 (shrunk) and Rp^2 (grown), cell units
  int lo[D];
  unsigned span[D];
  unsigned inv[D];  // ceil(2^16 / span)
  unsigned self;
  unsigned excl;    // first position of this candidate in the flattened stream
};

template <int D, bool Ex>
__global__ void __launch_bounds__(kScanWarps * 32) k_border_scan32(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp,
                                                                  const std::uint32_t* __restrict__ sq,
                                                                  std::uint64_t scap,
                                                                  const unsigned* __restrict__ nsq_p,
                                                                  unsigned* __restrict__ next,
                                                                  unsigned* __restrict__ fin,
                                                                  std::uint32_t* __restrict__ cand,
                                                                  std::uint64_t cap,
                                                                  unsigned* __restrict__ ncand) {
  __shared__ OwnerGrid<D> og;
  __shared__ ScanSlot<D, Ex> slots[kScanWarps][32];
  __shared__ unsigned char nzl[kScanWarps][32];
  extern __shared__ std::uint64_t s_off_sh[];
  if (threadIdx.x == 0) og = *ogp;
  if (a.k + 1 <= kSmemOffsMax)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  const PartOffs s_off{s_off_sh, a.offsets, a.k + 1 <= kSmemOffsMax};
  const unsigned nsq = *nsq_p;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  const unsigned wid = threadIdx.x >> 5;
  ScanSlot<D, Ex>* sl = slots[wid];
  unsigned char* nz = nzl[wid];
  const unsigned full = 0xffffffffu;
  const unsigned fd0 = static_cast<unsigned>(og.ldims[0][0]), fd1 = static_cast<unsigned>(og.ldims[0][1]);
  int top[D];
#pragma unroll
  for (int d = 0; d < D; ++d) top[d] = og.ldims[0][d] - 1;
  // exact policy: the level-0 tiled index of a cell (the per-cell point lists)
  const bool multi_level = og.levels > 1;
  unsigned long long bst[D];
  bst[0] = 1;
#pragma unroll
  for (int d = 1; d < D; ++d) bst[d] = bst[d - 1] * static_cast<unsigned long long>(multi_level ? og.ldims[1][d - 1] : 1);
  const CellPt<D>* cpts = static_cast<const CellPt<D>*>(a.cell_pts);
  unsigned base = claim_batch(next);
  for (;;) {
    if (base >= nsq) break;
    unsigned nclaim = 0;
    if (lane == 0) nclaim = atomicAdd(next, 32u);
    const unsigned t = base + lane;
    const bool has = t < nsq;
    std::uint32_t row = 0, self = 0;
    unsigned cnt = 0;
    bool wide_row = false;
    if (has) {
      row = sq[t];
      float U[D];
#pragma unroll
      for (int d = 0; d < D; ++d) U[d] = __uint_as_float(sq[std::uint64_t(1 + d) * scap + t]);
      const float rp = __uint_as_float(sq[std::uint64_t(D + 1) * scap + t]);
      const float reach = __uint_as_float(sq[std::uint64_t(D + 2) * scap + t]);
      self = s_off.part(a.k, row);
      ScanSlot<D, Ex>& r = sl[lane];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int lo = max(floor_small(U[d] - rp), 0);
        const int hi = min(floor_small(U[d] + rp), top[d]);
        const int span = hi - lo + 1;
        wide_row = wide_row || span > kFlatSpan || span < 1;
        r.lo[d] = lo;
        r.span[d] = static_cast<unsigned>(span);
#pragma unroll
        for (int i = 0; i < kFlatSpan; ++i) {
          const float c = static_cast<float>(lo + i);
          const float g = fmaxf(fmaxf(c - U[d], U[d] - (c + 1.f)), 0.f);
          r.g2[d][i] = g * g;
        }
        r.inv[d] = static_cast<unsigned>(ceilf(__fdiv_rn(65536.f, static_cast<float>(max(span, 1)))));
      }
      // (a few binary32 roundings of the squared distances, far inside the margins)
      // (the per-cell comparisons' own slack, d2 * 1.000002 + 1e-12 < rin2 and
      // d2 * 0.99999 - 1e-6 <= rout2, folded into the thresholds with the
      // rounding directed to the conservative side)
      r.rin2 = reach > 0.f ? __fmul_rd((reach * reach * 0.999998f - 1e-12f) - 1e-12f, 0.999998f) : -1.f;
      r.rout2 = __fmul_ru((rp * rp + 1e-6f) * 1.00001f + 1e-6f, 1.0000101f);
      r.self = self;
      if constexpr (Ex) {
        // the balls in coordinates: centre lo + U edge (binary64, ~1e-16
        // relative), radii scaled by the edge, 1e-9 relative margins (the
        // binary64 distances below round ~1e-15 relative)
#pragma unroll
        for (int d = 0; d < D; ++d) r.c64[d] = og.g.lo[d] + static_cast<double>(U[d]) * og.g.edge;
        const double ri = reach > 0.f ? static_cast<double>(reach) * og.g.edge : 0.0;
        const double ro = static_cast<double>(rp) * og.g.edge;
        r.pin2 = reach > 0.f ? ri * ri * (1.0 - 1e-9) : -1.0;
        r.pout2 = ro * ro * (1.0 + 1e-9) + 1e-300;
      }
      if (!wide_row) cnt = D == 3 ? r.span[1] * r.span[2] : r.span[1];
    }
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(full, incl, o);
      if (lane >= static_cast<unsigned>(o)) incl += y;
    }
    const unsigned total = __shfl_sync(full, incl, 31);
    const unsigned excl = incl - cnt;
    const unsigned nzmask = __ballot_sync(full, cnt > 0);
    if (cnt) {
      sl[lane].excl = excl;
      nz[__popc(nzmask & lt)] = static_cast<unsigned char>(lane);
    }
    __syncwarp();
    unsigned hitm = 0, ambm = 0;
    int cur = -1;
    for (unsigned b0 = 0; b0 < total; b0 += 32) {
      const bool st = cnt && excl >= b0 && excl < b0 + 32;
      const unsigned smask = __reduce_or_sync(full, st ? 1u << (excl - b0) : 0u);
      const unsigned q = b0 + lane;
      bool hit = false, amb = false;
      unsigned cl = 0;
      if (q < total) {
        cl = nz[cur + __popc(smask & ((2u << lane) - 1u))];
        const ScanSlot<D, Ex>& r = sl[cl];
        const unsigned rem = q - r.excl;
        float g12, g2z = 0.f;
        int c1, c2 = 0;
        if constexpr (D == 3) {
          const unsigned i2 = (rem * r.inv[1]) >> 16;  // rem / span1 (rem * span1 < 2^16)
          const unsigned i1 = rem - i2 * r.span[1];
          c1 = r.lo[1] + static_cast<int>(i1);
          c2 = r.lo[2] + static_cast<int>(i2);
          g12 = r.g2[1][i1];
          g2z = r.g2[2][i2];
        } else {
          c1 = r.lo[1] + static_cast<int>(rem);
          g12 = r.g2[1][rem];
        }
        const unsigned long long lb =
            (D == 3 ? static_cast<unsigned long long>(static_cast<unsigned>(c1) + fd1 * static_cast<unsigned>(c2))
                    : static_cast<unsigned long long>(static_cast<unsigned>(c1))) * fd0 +
            static_cast<unsigned>(r.lo[0]);
        std::uint32_t fw[kFlatSpan];
        float d2[kFlatSpan];
#pragma unroll
        for (int i0 = 0; i0 < kFlatSpan; ++i0) {
          d2[i0] = r.g2[0][i0] + g12 + g2z;
          fw[i0] = kFieldEmptyBit;
          if (i0 < static_cast<int>(r.span[0]) && d2[i0] <= r.rout2)
            fw[i0] = static_cast<std::uint32_t>(__ldg(a.field + lb + i0));
        }
        const std::uint32_t sf = r.self;
        if constexpr (!Ex) {
#pragma unroll
          for (int i0 = 0; i0 < kFlatSpan; ++i0) {
            const bool foreign = !(fw[i0] & kFieldEmptyBit) && (fw[i0] & 0xFFFFu) != sf;
            const bool in = d2[i0] < r.rin2;
            hit = hit || (foreign && in);
            amb = amb || (foreign && !in);
          }
        } else {
          // exact policy: the other parts' points of the foreign cells, by
          // their binary64 distance to the ball centre: strictly inside the
          // inner ball -> strictly inside the circumsphere (positive); beyond
          // the outer ball -> not inside; in between -> the binary64 stage
          const unsigned long long tb =
              og.loff[0] + cell_off<D>(c1, 1, bst, multi_level) + (D == 3 ? cell_off<D>(c2, 2, bst, multi_level) : 0ull);
          for (int i0 = 0; i0 < static_cast<int>(r.span[0]) && !hit; ++i0) {
            if ((fw[i0] & kFieldEmptyBit) || (fw[i0] & 0xFFFFu) == sf) continue;
            const unsigned long long idx = tb + cell_off<D>(r.lo[0] + i0, 0, bst, multi_level);
            for (std::uint32_t t = a.cell_start[idx], te = a.cell_start[idx + 1]; t < te; ++t) {
              const CellPt<D> q = cpts[t];
              if (q.label == sf) continue;
              double dq = 0.0;
#pragma unroll
              for (int d = 0; d < D; ++d) {
                const double x = q.x[d] - r.c64[d];
                dq = fma(x, x, dq);
              }
              if (dq < r.pin2) {
                hit = true;
                break;
              }
              amb = amb || dq <= r.pout2;
            }
          }
        }
      }
      hitm |= __reduce_or_sync(full, hit ? 1u << cl : 0u);
      ambm |= __reduce_or_sync(full, amb ? 1u << cl : 0u);
      cur += __popc(smask);
    }
    __syncwarp();
    const bool pos = has && !wide_row && ((hitm >> lane) & 1u);
    const bool open = has && !pos && (wide_row || ((ambm >> lane) & 1u));
    if (has && !open) {
      __stcs(a.positive + row, static_cast<std::uint8_t>(pos ? 1 : 0));
      if (pos)
#pragma unroll
        for (int j = 0; j <= D; ++j) a.vflags[__ldg(a.verts + std::uint64_t(j) * a.S + row)] = 1;
    }
    if (a.counters) {
      const unsigned mh = __ballot_sync(full, has), mp = __ballot_sync(full, pos), mo = __ballot_sync(full, open);
      if (lane == 0) {
        atomicAdd(&a.counters[16], static_cast<unsigned long long>(__popc(mh)));
        if (mp) atomicAdd(&a.counters[17], static_cast<unsigned long long>(__popc(mp)));
        if (mo) atomicAdd(&a.counters[18], static_cast<unsigned long long>(__popc(mo)));
      }
    }
    // the undecided rows: the binary64 exact stage
    {
      const unsigned mo = __ballot_sync(full, open);
      if (mo) {
        unsigned ob = 0;
        if (lane == 0) ob = atomicAdd(ncand, static_cast<unsigned>(__popc(mo)));
        ob = __shfl_sync(full, ob, 0);
        if (open) {
          cand[ob + __popc(mo & lt)] = row;
          cand[cap + ob + __popc(mo & lt)] = __float_as_uint(-1.f);
        }
      }
    }
    base = __shfl_sync(full, nclaim, 0);
  }
  rewind_cursor(next, fin, nsq);
}

// Candidates whose binary32 sphere failed (reach == kReachCheckOrient): the
// exact orientation of their binary64 vertices; zero is DegenerateSimplex
// (geometry.cpp:279-297). Rare rows, off the critical path (side stream).
template <int D>
__global__ void __launch_bounds__(256) k_border_orient(BorderArgs a, const std::uint32_t* __restrict__ cand,
                                                      std::uint64_t cap, const unsigned* __restrict__ ncand_p) {
  const unsigned ncand = *ncand_p;
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < ncand; t += gridDim.x * blockDim.x) {
    if (cand[t] == kNoRow) continue;
    if (__uint_as_float(cand[cap + t]) != kReachCheckOrient) continue;
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = __ldg(a.verts + std::uint64_t(j) * a.S + cand[t]);
    double p[D + 1][D];
    load_simplex<D>(a, v, p);
    if (a.counters) atomicAdd(a.counters + kCtrOrientRows, 1ull);
    if (orientation_exact<D>(p, a.counters ? a.counters + kCtrOrientExact : nullptr) == 0)
      atomicOr(a.status, kStDegenerate);
  }
}

// Wide candidates (cell range wider than 5 per axis, or non-finite spheres):
// one warp descends the owner pyramid for one candidate at a time. A block
// expansion reads its 64 contiguous child codes (two coalesced 64-byte loads)
// and tests them on 32 lanes; children that are foreign, overlap the sphere
// and are neither leaves nor contained in it go on a per-warp LIFO stack in
// shared memory. Same decisions as og_sphere_hits_foreign (exact pruning),
// without serialising a whole descent on one lane.
constexpr int kWideWarps = 4;
#ifndef WIDE_CLAIM
#define WIDE_CLAIM 4
#endif
#ifndef WIDE_CTAS
#define WIDE_CTAS 8
#endif
constexpr unsigned kWideClaim = WIDE_CLAIM;  // rows a warp claims at a time in the wide / hull kernels
constexpr int kWideStack = 256;  // deeper stacks (> 4 levels of dense partial blocks) take the serial fallback

template <int D>
struct WideEntry {
  int c[D];
  int level;
};

// Warp-cooperative exact descent of the owner pyramid over the leaf range
// [a, b]: test(L, block) returns 0 reject, 1 descend, 2 accept (leaf or every
// sub-box passes); fallback() answers alone when the stack would overflow.
template <int D, class Test, class Fallback>
__device__ bool warp_descent(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner, const int* a,
                             const int* b, std::uint32_t self, const Test& test, const Fallback& fallback,
                             WideEntry<D>* stk, unsigned long long* counters = nullptr) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned full = 0xffffffffu;
  int L0 = 0;
  for (; L0 < og.levels - 1; ++L0) {
    bool ok = true;
#pragma unroll
    for (int d = 0; d < D; ++d) ok = ok && ((b[d] >> (L0 * og.shift)) - (a[d] >> (L0 * og.shift)) <= 1);
    if (ok) break;
  }
  int top = 0;
  // start blocks (<= 2 per axis)
  {
    int s0[D], n0[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      s0[d] = a[d] >> (L0 * og.shift);
      n0[d] = (b[d] >> (L0 * og.shift)) - s0[d] + 1;
    }
    const int total = D == 3 ? n0[0] * n0[1] * n0[2] : n0[0] * n0[1];
    int r = 0;
    int cc[D];
    if (static_cast<int>(lane) < total) {
      int rem = static_cast<int>(lane);
#pragma unroll
      for (int d = 0; d < D; ++d) {  // n0[d] is 1 or 2
        cc[d] = s0[d] + (n0[d] == 2 ? (rem & 1) : 0);
        rem = n0[d] == 2 ? rem >> 1 : rem;
      }
      const std::uint16_t code = owner[og_index<D>(og, L0, cc)];
      if (code != kOwnerEmpty && code != self) r = test(L0, cc);
    }
    if (__any_sync(full, r == 2)) return true;
    const unsigned pm = __ballot_sync(full, r == 1);
    if (r == 1) {
      WideEntry<D>& e = stk[__popc(pm & ((1u << lane) - 1u))];
#pragma unroll
      for (int d = 0; d < D; ++d) e.c[d] = cc[d];
      e.level = L0;
    }
    top = __popc(pm);
    __syncwarp();
  }
  while (top > 0) {
    const WideEntry<D> e = stk[top - 1];
    --top;
    __syncwarp();
    if (counters && lane == 0) atomicAdd(&counters[6], 1ull);
    const int lv = e.level - 1;
    const int csh = lv * og.shift;
    const std::uint16_t* ch = owner + og.loff[lv] + lin_i<D>(og.ldims[e.level], e.c) * 64;
    int res[2];
    int cc[2][D];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int j = half * 32 + static_cast<int>(lane);
      og_child<D>(e.c, j, cc[half]);
      bool in = true;
#pragma unroll
      for (int d = 0; d < D; ++d) in = in && cc[half][d] >= (a[d] >> csh) && cc[half][d] <= (b[d] >> csh);
      res[half] = 0;
      if (in) {
        const std::uint16_t code = ch[j];
        if (code != kOwnerEmpty && code != self) res[half] = test(lv, cc[half]);
      }
    }
    if (__any_sync(full, res[0] == 2 || res[1] == 2)) return true;
    const unsigned p0 = __ballot_sync(full, res[0] == 1), p1 = __ballot_sync(full, res[1] == 1);
    const int np = __popc(p0) + __popc(p1);
    if (top + np > kWideStack) return fallback();  // uniform fallback
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const unsigned pm = half ? p1 : p0;
      if (res[half] == 1) {
        WideEntry<D>& w = stk[top + (half ? __popc(p0) : 0) + __popc(pm & ((1u << lane) - 1u))];
#pragma unroll
        for (int d = 0; d < D; ++d) w.c[d] = cc[half][d];
        w.level = lv;
      }
    }
    top += np;
    __syncwarp();
  }
  return false;
}

template <int D, bool Ex, class Leaf>
__device__ bool warp_sphere_descent(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner, const double* c,
                                    double r2, std::uint32_t self, WideEntry<D>* stk, const Leaf& leaf,
                                    unsigned long long* counters = nullptr, const float* U = nullptr,
                                    float reach = -1.f) {
  if (isnan(r2)) return false;
  bool fin = isfinite(r2);
#pragma unroll
  for (int d = 0; d < D; ++d) fin = fin && isfinite(c[d]);
  int a[D], b[D];
  if (fin) {
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
  auto test = [&](int L, const int* cc) -> int {
    double blo[D], bhi[D];
    og_block_box<D>(og, L, cc, blo, bhi);
    if (!box_sphere<D>(blo, bhi, c, r2)) return 0;
    if constexpr (Ex) {
      // a block (foreign code: it holds another part's point) entirely
      // inside the prefilter's inner ball has that point strictly inside the
      // circumsphere: accepted without its leaves (cell units: the block's
      // cell range, far corner from U, the prefilter's margins)
      if (reach > 0.f) {
        const int sh = L * og.shift;
        float dd = 0.f;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const float b0 = static_cast<float>(cc[d] << sh);
          const float b1 = static_cast<float>(min((cc[d] + 1) << sh, og.ldims[0][d]));
          const float far = fmaxf(U[d] - b0, b1 - U[d]);
          dd = fmaf(far, far, dd);
        }
        if (dd * 1.000002f + 1e-6f < reach * reach) return 2;
      }
      return L > 0 ? 1 : (leaf(cc) ? 2 : 0);
    } else {
      if (L == 0 || box_inside_sphere<D>(blo, bhi, c, r2)) return 2;
      return 1;
    }
  };
  auto fallback = [&]() {
    if constexpr (Ex) return og_sphere_exact_serial<D>(og, owner, c, r2, self, leaf);
    else return og_sphere_hits_foreign<D>(og, owner, c, r2, self);
  };
  return warp_descent<D>(og, owner, a, b, self, test, fallback, stk, counters);
}

template <int D, bool Ex>
__global__ void __launch_bounds__(kWideWarps * 32, Ex ? 6 : WIDE_CTAS) k_border_wide(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp,
                                                                 const std::uint32_t* __restrict__ wide,
                                                                 std::uint64_t cap,
                                                                 const unsigned* __restrict__ nwide_p,
                                                                 unsigned* __restrict__ next,
                                                                 unsigned* __restrict__ fin,
                                                                 const unsigned* __restrict__ nlight_p) {
  __shared__ OwnerGrid<D> og;
  __shared__ WideEntry<D> stacks[kWideWarps][kWideStack];
  extern __shared__ std::uint64_t s_off_sh[];
  if (threadIdx.x == 0) og = *ogp;
  if (a.k + 1 <= kSmemOffsMax)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  // part offsets in shared memory, or read in place for very large k
  const PartOffs s_off{s_off_sh, a.offsets, a.k + 1 <= kSmemOffsMax};
  // rows [0, nheavy) from the front of the queue, then the nlight rows
  // stored from the back (see k_border_exact)
  const unsigned nheavy = *nwide_p;
  const unsigned nwide = nheavy + (nlight_p ? *nlight_p : 0u);
  const unsigned lane = threadIdx.x & 31u;
  WideEntry<D>* stk = stacks[threadIdx.x >> 5];
  const unsigned full = 0xffffffffu;
  for (;;) {
    // few rows per claim: a row is a whole-warp descent of very uneven cost,
    // and warps holding 32 of them leave the others idle at the end
    const unsigned base = claim_batch(next, kWideClaim);
    if (base >= nwide) break;
    const unsigned t = base + lane;
    const bool has = lane < kWideClaim && t < nwide;
    std::uint64_t s = 0;
    std::uint32_t self = 0, v[D + 1];
    double c[D], r2 = 0.0;
    float U[D], reach = -1.f;
    if (has) {
      const std::uint64_t slot = t < nheavy ? t : cap - 1 - (t - nheavy);
      s = wide[slot];
      self = s_off.part(a.k, s);
#pragma unroll
      for (int j = 0; j <= D; ++j) v[j] = wide[std::uint64_t(j + 1) * cap + slot];
      if constexpr (Ex) {
        reach = __uint_as_float(wide[std::uint64_t(2 * D + 2) * cap + slot]);
#pragma unroll
        for (int d = 0; d < D; ++d) U[d] = reach > 0.f ? __uint_as_float(wide[std::uint64_t(D + 2 + d) * cap + slot]) : 0.f;
      }
      double p[D + 1][D];
      load_simplex<D>(a, v, p);
      circumsphere_inflated<D>(p, c, &r2);
    }
    bool pos = false;
    const unsigned todo0 = __ballot_sync(full, has);
    for (unsigned todo = todo0; todo; todo &= todo - 1) {
      const int l = __ffs(todo) - 1;
      double cl[D];
#pragma unroll
      for (int d = 0; d < D; ++d) cl[d] = __shfl_sync(full, c[d], l);
      const double rl = __shfl_sync(full, r2, l);
      const std::uint32_t sl = __shfl_sync(full, self, l);
      // exact policy: lanes test their leaf cells' points against the
      // candidate's circumsphere (vertices broadcast, coordinates reloaded)
      std::uint32_t vl[D + 1];
#pragma unroll
      for (int j = 0; j <= D; ++j) vl[j] = __shfl_sync(full, v[j], l);
      const std::uint64_t srow = __shfl_sync(full, s, l);
      double pv[D + 1][D];
      int par = 1;
      bool loaded = false;
      auto leaf = [&](const int* cell) -> bool {
        if (!loaded) {
          load_simplex<D>(a, vl, pv);
          par = a.parity[srow];
          loaded = true;
        }
        return cell_points_inside<D>(a, og_index<D>(og, 0, cell), pv, par, sl, srow);
      };
      float Ul[D];
#pragma unroll
      for (int d = 0; d < D; ++d) Ul[d] = __shfl_sync(full, Ex ? U[d] : 0.f, l);
      const float reach_l = __shfl_sync(full, reach, l);
      const bool hit = warp_sphere_descent<D, Ex>(og, a.owner, cl, rl, sl, stk, leaf, a.counters, Ul, reach_l);
      if (static_cast<int>(lane) == l) pos = hit;
      if (a.counters && hit && lane == 0) atomicAdd(&a.counters[9], 1ull);
      __syncwarp();
    }
    if (has) {
      __stcs(a.positive + s, static_cast<std::uint8_t>(pos ? 1 : 0));
      if (pos)
#pragma unroll
        for (int j = 0; j <= D; ++j) a.vflags[v[j]] = 1;
    }
  }
  rewind_cursor(next, fin, nwide);
}

// K6: rows with the infinite vertex (hull facets). Lanes set up 32 rows
// (facet ids, the finite neighbour's inner vertex, its exact orientation);
// under the grid policy each row's halfspace descent then runs on the whole
// warp (warp_descent), the bbox policy tests the k-1 root boxes per lane.
template <int D, bool Ex>
__global__ void __launch_bounds__(kWideWarps * 32) k_border_infinite(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp,
                                                                     unsigned* __restrict__ next,
                                                                     unsigned* __restrict__ fin) {
  __shared__ OwnerGrid<D> og;
  __shared__ WideEntry<D> stacks[kWideWarps][kWideStack];
  extern __shared__ std::uint64_t s_off_sh[];
  if (threadIdx.x == 0) og = *ogp;
  if (a.k + 1 <= kSmemOffsMax)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  // part offsets in shared memory, or read in place for very large k
  const PartOffs s_off{s_off_sh, a.offsets, a.k + 1 <= kSmemOffsMax};
  const unsigned full = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u;
  WideEntry<D>* stk = stacks[threadIdx.x >> 5];
  unsigned long long* const pesc = a.counters ? a.counters + kCtrOrientExact : nullptr;
  const unsigned count = *a.inf_count;
  const bool use_hull_set = Ex && a.hull_valid && *a.hull_valid;
  const unsigned long long n_hull = use_hull_set ? *a.hull_count : 0ull;
  for (;;) {
    const unsigned q0 = claim_batch(next, kWideClaim);
    if (q0 >= count) break;
    const unsigned q = q0 + lane;
    const bool has = lane < kWideClaim && q < count;
    std::uint64_t s = 0;
    std::uint32_t self = 0, fv[D];
    int inner_sign = 0;
    double fx[D][D];  // facet vertex coordinates
    if (has) {
      s = a.inf_queue[q];
      self = s_off.part(a.k, s);
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
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int d = 0; d < D; ++d) fx[j][d] = a.xyz[std::size_t(fv[j]) * D + d];
      const double* pts[D + 1];
#pragma unroll
      for (int j = 0; j < D; ++j) pts[j] = fx[j];
      pts[D] = a.xyz + std::size_t(inner) * D;
      inner_sign = orient_dev<D>(pts, pesc);
    }
    bool pos = false;
    if (a.policy == SBDT_POLICY_BBOX) {
      if (has) {
        const double* facet[D];
#pragma unroll
        for (int j = 0; j < D; ++j) facet[j] = fx[j];
        for (std::uint32_t j = 0; j < a.k && !pos; ++j) {
          if (j == self) continue;
          double blo[D], bhi[D];
          if (bbox_policy_box<D>(og, a.pbbox, j, blo, bhi) && corners_outside<D>(facet, inner_sign, blo, bhi, pesc) > 0)
            pos = true;
        }
      }
    } else {
      for (unsigned todo = __ballot_sync(full, has); todo; todo &= todo - 1) {
        const int l = __ffs(todo) - 1;
        double fl[D][D];
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
          for (int d = 0; d < D; ++d) fl[j][d] = __shfl_sync(full, fx[j][d], l);
        const int sl_sign = __shfl_sync(full, inner_sign, l);
        const std::uint32_t sl_self = __shfl_sync(full, self, l);
        const double* facet[D];
#pragma unroll
        for (int j = 0; j < D; ++j) facet[j] = fl[j];
        int lo[D], hi[D];
#pragma unroll
        for (int d = 0; d < D; ++d) lo[d] = 0, hi[d] = og.ldims[0][d] - 1;
        auto leaf = [&](const int* cell) -> bool {
          return cell_points_outside<D>(a, og_index<D>(og, 0, cell), facet, sl_sign, sl_self);
        };
        sbdt_pred::PlaneFilter<D> pf;
        sbdt_pred::plane_filter_init<D>(pf, facet, sl_sign);
        auto test = [&](int L, const int* cc) -> int {
          double blo[D], bhi[D];
          og_block_box<D>(og, L, cc, blo, bhi);
          // all corners at once through the facet's plane with its error
          // bound; the exact per-corner orient only when that is undecided
          const int f = sbdt_pred::plane_filter_box<D>(pf, blo, bhi);
          const int out = f >= 0 ? (f == 0 ? 0 : (f == 2 ? (1 << D) : 1)) : corners_outside<D>(facet, sl_sign, blo, bhi, pesc);
          if (out == 0) return 0;
          if (out == (1 << D)) return 2;  // the whole box is strictly outside
          if (L > 0) return 1;
          if constexpr (Ex) return leaf(cc) ? 2 : 0;
          else return 2;
        };
        auto fallback = [&]() {
          if constexpr (Ex) return og_halfspace_exact_serial<D>(og, a.owner, facet, sl_sign, sl_self, leaf);
          else return og_halfspace_hits_foreign<D>(og, a.owner, facet, sl_sign, sl_self);
        };
        bool hit;
        if (Ex && use_hull_set) {
          // Exact policy: some foreign point strictly outside the facet's
          // plane <=> some foreign HULL vertex (a finite vertex of an
          // infinite row of its partial) is: a partition's points are convex
          // combinations of its hull vertices, so if all of those lie in the
          // closed inner halfspace, so do all its points (and a partition's
          // own points never lie outside its own hull facets). A point
          // strictly outside lies in a cell with a corner strictly outside,
          // so the reference's candidate-cell filter changes nothing.
          const double* q4[D + 1];
#pragma unroll
          for (int j = 0; j < D; ++j) q4[j] = fl[j];
          bool out = false;
          for (unsigned long long u0 = 0; u0 < n_hull && !out; u0 += 32) {
            bool o = false;
            const unsigned long long u = u0 + lane;
            if (u < n_hull) {
              const std::uint32_t id = a.hull_ids[u];
              if (a.labels[id] != sl_self) {
                q4[D] = a.xyz + std::size_t(id) * D;
                const int r = orient_dev<D>(q4, pesc);
                o = r != 0 && r != sl_sign;
              }
            }
            out = __any_sync(full, o);
          }
          hit = out;
        } else {
          hit = warp_descent<D>(og, a.owner, lo, hi, sl_self, test, fallback, stk);
        }
        if (static_cast<int>(lane) == l) pos = hit;
        __syncwarp();
      }
    }
    if (has) {
      a.positive[s] = pos ? 1 : 0;
      if (a.spheres)
#pragma unroll
        for (int d = 0; d <= D; ++d) a.spheres[s * (D + 1) + d] = 0.0;
      if (pos)
#pragma unroll
        for (int j = 0; j < D; ++j) a.vflags[fv[j]] = 1;
    }
  }
  rewind_cursor(next, fin, count);
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

// ---- exact policy: per-cell point lists and the escalation pass --------------
template <int D>
__global__ void k_cell_count(const double* __restrict__ xyz, const std::uint32_t* __restrict__ labels, std::uint64_t n,
                             const OwnerGrid<D>* __restrict__ ogp, std::uint32_t* __restrict__ cnt) {
  __shared__ OwnerGrid<D> og;
  if (threadIdx.x == 0) og = *ogp;
  __syncthreads();
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    if (labels[i] == SBDT_UNINDEXED) continue;
    int c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) c[d] = static_cast<int>(cell_coord_fast<D>(og.g, og.inv_edge, xyz[i * D + d], d));
    atomicAdd(&cnt[og_index<D>(og, 0, c)], 1u);
  }
}

template <int D>
__global__ void k_cell_scatter(const double* __restrict__ xyz, const std::uint32_t* __restrict__ labels,
                               std::uint64_t n, const OwnerGrid<D>* __restrict__ ogp,
                               const std::uint32_t* __restrict__ start, std::uint32_t* __restrict__ fill,
                               CellPt<D>* __restrict__ pts) {
  __shared__ OwnerGrid<D> og;
  if (threadIdx.x == 0) og = *ogp;
  __syncthreads();
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    if (labels[i] == SBDT_UNINDEXED) continue;
    CellPt<D> q;
    int c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      q.x[d] = xyz[i * D + d];
      c[d] = static_cast<int>(cell_coord_fast<D>(og.g, og.inv_edge, q.x[d], d));
    }
    q.label = labels[i];
    q.pid = static_cast<std::uint32_t>(i);
    const unsigned long long idx = og_index<D>(og, 0, c);
    pts[start[idx] + atomicAdd(&fill[idx], 1u)] = q;
  }
}

// Undecided filtered in_sphere tests, decided with expansion arithmetic
// (predicates.hpp; an independent exact method from the reference's
// scaled-integer fallback, geometry.cpp:32-146). One scratch area per thread.
constexpr int kEscThreads = 256;

template <int D>
__global__ void __launch_bounds__(128) k_border_escalate(BorderArgs a, double* __restrict__ scratch) {
  const unsigned count = min(*a.esc_count, a.esc_cap);
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  double* buf = scratch + std::size_t(tid) * (D == 3 ? sbdt_pred::kInSphere3Scratch : sbdt_pred::kInSphere2Scratch);
  const CellPt<D>* pts = static_cast<const CellPt<D>*>(a.cell_pts);
  for (unsigned e = tid; e < count; e += gridDim.x * blockDim.x) {
    const std::uint64_t s = a.esc[2ull * e];
    if (a.positive[s]) continue;  // decided by another point
    const std::uint32_t t = a.esc[2ull * e + 1];
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = a.verts[std::uint64_t(j) * a.S + s];
    const double* p[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) p[j] = a.xyz + std::size_t(v[j]) * D;
    if (a.parity[s] != 1) {
      const double* tmp = p[0];
      p[0] = p[1];
      p[1] = tmp;
    }
    const double* q = pts[t].x;
    int r;
    if constexpr (D == 3) r = sbdt_pred::in_sphere3_exact_buf(p[0], p[1], p[2], p[3], q, buf);
    else r = sbdt_pred::in_sphere2_exact_buf(p[0], p[1], p[2], q, buf);
    if (r > 0) {
      a.positive[s] = 1;
#pragma unroll
      for (int j = 0; j <= D; ++j) a.vflags[v[j]] = 1;
    }
  }
}

// Exact policy, rows whose undecided in_sphere pairs overflowed the
// escalation queue: one thread per row decides it again from scratch — the
// binary64 sphere, the serial exact descent over the foreign cells it
// overlaps, every foreign point of those cells with the filtered in_sphere
// and, where undecided, the exact one in this thread's scratch (the
// escalation kernel's, which has finished). Rare: a degrade path, not a
// fast path.
template <int D>
__global__ void __launch_bounds__(128) k_border_redo(BorderArgs a, const OwnerGrid<D>* __restrict__ ogp,
                                                     double* __restrict__ scratch) {
  const unsigned count = *a.redo_count;
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  double* buf = scratch + std::size_t(tid) * (D == 3 ? sbdt_pred::kInSphere3Scratch : sbdt_pred::kInSphere2Scratch);
  const OwnerGrid<D>& og = *ogp;
  const CellPt<D>* pts = static_cast<const CellPt<D>*>(a.cell_pts);
  for (unsigned e = tid; e < count; e += gridDim.x * blockDim.x) {
    const std::uint64_t s = a.redo_rows[e];
    if (a.positive[s]) continue;  // decided by a queued pair
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = a.verts[std::uint64_t(j) * a.S + s];
    double p[D + 1][D];
    load_simplex<D>(a, v, p);
    double c[D], r2;
    circumsphere_inflated<D>(p, c, &r2);
    const std::uint32_t self = part_of(a.offsets, a.k, s);
    const double* A = a.parity[s] != 1 ? p[1] : p[0];
    const double* B = a.parity[s] != 1 ? p[0] : p[1];
    auto leaf = [&](const int* cell) -> bool {
      const unsigned long long idx = og_index<D>(og, 0, cell);
      for (std::uint32_t t = a.cell_start[idx], te = a.cell_start[idx + 1]; t < te; ++t) {
        const CellPt<D> q = pts[t];
        if (q.label == self) continue;
        int r;
        if constexpr (D == 3) r = sbdt_pred::in_sphere3_filtered(A, B, p[2], p[3], q.x);
        else r = sbdt_pred::in_sphere2_filtered(A, B, p[2], q.x);
        if (r == 2) {
          if constexpr (D == 3) r = sbdt_pred::in_sphere3_exact_buf(A, B, p[2], p[3], q.x, buf);
          else r = sbdt_pred::in_sphere2_exact_buf(A, B, p[2], q.x, buf);
        }
        if (r > 0) return true;
      }
      return false;
    };
    if (og_sphere_exact_serial<D>(og, a.owner, c, r2, self, leaf)) {
      a.positive[s] = 1;
#pragma unroll
      for (int j = 0; j <= D; ++j) a.vflags[v[j]] = 1;
    }
  }
}

// Circumspheres only (spheres_out with the grid / exact policies).
template <int D>
__global__ void k_border_spheres(BorderArgs a) {
  for (std::uint64_t s = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < a.S;
       s += std::uint64_t(gridDim.x) * blockDim.x) {
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = a.verts[std::uint64_t(j) * a.S + s];
    if (v[D] == kInfVertex) continue;  // written by k_border_infinite
    double p[D + 1][D], c[D], r2;
    load_simplex<D>(a, v, p);
    circumsphere_inflated<D>(p, c, &r2);
#pragma unroll
    for (int d = 0; d < D; ++d) a.spheres[s * (D + 1) + d] = c[d];
    a.spheres[s * (D + 1) + D] = r2;
  }
}

__global__ void k_cand_count(const unsigned* ncand, const unsigned* npf_wide, std::uint64_t S,
                             unsigned long long* counters, const unsigned* esc_count, unsigned esc_cap) {
  counters[0] = S;  // rows scanned by the prefilter (finite + infinite)
  counters[1] = ncand[0] - counters[11];  // queue slots minus the holes
  counters[3] = ncand[2] + ncand[6];      // wide rows forwarded by the exact stage
  counters[4] = npf_wide[0] + npf_wide[3];  // wide rows routed by the prefilter
  // exact policy: (row, point) in_sphere tests the filter left undecided
  counters[kCtrInSphereExact] = esc_count ? min(*esc_count, esc_cap) : 0u;
}

__global__ void k_u32_to_u64(const std::uint32_t* in, std::uint64_t* out) { *out = *in; }

// ---------------------------------------------------------------------------
// Exact policy: the hull vertex set of the partials (finite vertices of their
// infinite rows) for k_border_infinite, and whether it is complete (every
// partition that holds points has rows, hence hull facets).
template <int D>
__global__ void k_hull_mark(BorderArgs a, std::uint8_t* __restrict__ hflags) {
  const unsigned count = *a.inf_count;
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x) {
    const std::uint64_t s = a.inf_queue[q];
#pragma unroll
    for (int j = 0; j < D; ++j) hflags[a.verts[std::uint64_t(j) * a.S + s]] = 1;
  }
}

__global__ void k_part_present(const std::uint32_t* __restrict__ labels, std::uint64_t n,
                               std::uint8_t* __restrict__ present) {
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint32_t l = labels[i];
    if (l != SBDT_UNINDEXED && !present[l]) present[l] = 1;
  }
}

__global__ void k_hull_valid(const std::uint64_t* __restrict__ offsets, std::uint32_t k,
                             const std::uint8_t* __restrict__ present, unsigned* __restrict__ valid) {
  __shared__ unsigned ok;
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  for (std::uint32_t p = threadIdx.x; p < k; p += blockDim.x)
    if (present[p] && offsets[p + 1] == offsets[p]) ok = 0;
  __syncthreads();
  if (threadIdx.x == 0) *valid = ok;
}

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
  // recursion levels: the top level's grid (global bbox, n_total), SBDT_UNINDEXED points skipped
  const std::uint64_t n_grid = in->grid_n_total ? in->grid_n_total : in->n;
  const unsigned long long cap =
      in->grid_max_cells ? in->grid_max_cells
                         : static_cast<unsigned long long>(4.0 * double(n_grid > in->n ? n_grid : in->n) * scale) + 4096;
  const unsigned long long owner_len = 2 * cap + 64 * kMaxLevels + 4096;
  SBDT_WS(og, OwnerGrid<D>, "border.og", 1);
  SBDT_WS(owner, std::uint16_t, "border.owner", owner_len);
  SBDT_WS(bbox, unsigned long long, "border.bbox", 2 * D);
  // hull rows <= rows (small partitions can be mostly hull: >50% at ~5 points per part)
  SBDT_WS(infq, std::uint32_t, "border.infq", in->S + 1024);
  SBDT_WS(infc, unsigned, "border.infc", 1);
  unsigned long long* pbbox = nullptr;
  if (in->policy == SBDT_POLICY_BBOX) {
    SBDT_WS(pb, unsigned long long, "border.pbbox", std::uint64_t(in->k) * 2 * D);
    pbbox = pb;
  }

  // grid and exact policies: prefilter + exact + wide pipeline (spheres, when
  // requested, by a separate pass); bbox: one lane per row (k_border_finite)
  const bool tiled = in->policy != SBDT_POLICY_BBOX;
  const bool exact_policy = in->policy == SBDT_POLICY_EXACT;
  std::uint64_t* xq = nullptr;
  if (tiled) {
    SBDT_WS(q, std::uint64_t, "border.xq", in->n + 1);
    xq = q;
  }
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  StageTimer tgrid(ctx, "border.grid");
  const unsigned long long* bb = reinterpret_cast<const unsigned long long*>(in->d_bbox_ordered);
  if (in->grid_bbox) {
    GridBox gb{};
    for (int d = 0; d < D; ++d) gb.lo[d] = in->grid_bbox[d], gb.hi[d] = in->grid_bbox[D + d];
    k_set_bbox<D><<<1, 1, 0, st>>>(gb, bbox);
    ++ctx->launches;
    bb = bbox;
  } else if (!bb) {
    k_bbox_points_init<<<1, 32, 0, st>>>(bbox, D);
    const std::uint64_t want = (in->n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 8 ? want : std::uint64_t(sms) * 8);
    k_bbox_points<D><<<blocks > 0 ? blocks : 1, 256, 0, st>>>(in->d_xyz, in->n, bbox);
    ctx->launches += 2;
    bb = bbox;
  }
  k_owner_params<D><<<1, 1, 0, st>>>(bb, n_grid, cg, cap, owner_len, og, ctx->d_status);
  k_owner_clear<D><<<sms * 8, 256, 0, st>>>(og, owner);
  ++ctx->launches;
  if (pbbox) {
    k_pbbox_init<<<(in->k * 2 * D + 255) / 256, 256, 0, st>>>(pbbox, in->k * 2 * D, D);
    ctx->launches += 1;
  }
  {
    const std::uint64_t want = (in->n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 16 ? want : std::uint64_t(sms) * 16);
    const bool pb_sh = pbbox && in->k * 2 * D <= kPbboxSmem;
    const std::size_t sh = pb_sh ? sizeof(unsigned long long) * in->k * 2 * D : 0;
    k_owner_mark<D><<<blocks > 0 ? blocks : 1, 256, sh, st>>>(in->d_xyz, in->d_labels, in->n, og, owner,
                                                               pb_sh ? pbbox : nullptr, in->k, xq);
    if (pbbox && !pb_sh) {
      k_pbbox_global<D><<<blocks > 0 ? blocks : 1, 256, 0, st>>>(in->d_xyz, in->d_labels, in->n, pbbox);
      ++ctx->launches;
    }
  }
  k_owner_level<D><<<sms * 8, 256, 0, st>>>(og, owner, 1);
  k_owner_level<D><<<sms * 2, 256, 0, st>>>(og, owner, 2);
  k_owner_levels_tail<D><<<1, 1024, 0, st>>>(og, owner, 3);
  // exact policy: per-cell point lists over the level-0 tiled index
  std::uint32_t* cell_start = nullptr;
  void* cell_pts = nullptr;
  if (exact_policy) {
    SBDT_WS(ccnt, std::uint32_t, "border.cell_cnt", owner_len + 1);
    SBDT_WS(cstart, std::uint32_t, "border.cell_start", owner_len + 1);
    SBDT_WS(cbs, std::uint32_t, "border.cell_bs", (owner_len + 1) / kScanTile + 2);
    SBDT_WS(cpts, CellPt<D>, "border.cell_pts", in->n + 1);
    SBDT_CUDA_TRY(cudaMemsetAsync(ccnt, 0, sizeof(std::uint32_t) * (owner_len + 1), st));
    const std::uint64_t want = (in->n + 255) / 256;
    const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 16 ? want : std::uint64_t(sms) * 16);
    k_cell_count<D><<<blocks > 0 ? blocks : 1, 256, 0, st>>>(in->d_xyz, in->d_labels, in->n, og, ccnt);
    exclusive_scan(ccnt, cstart, owner_len + 1, cbs, nullptr, st, &ctx->launches);
    SBDT_CUDA_TRY(cudaMemsetAsync(ccnt, 0, sizeof(std::uint32_t) * (owner_len + 1), st));
    k_cell_scatter<D><<<blocks > 0 ? blocks : 1, 256, 0, st>>>(in->d_xyz, in->d_labels, in->n, og, cstart, ccnt, cpts);
    ctx->launches += 2;
    cell_start = cstart;
    cell_pts = cpts;
  }
  std::uint64_t* field = nullptr;
  if (tiled) {
    SBDT_WS(fw, std::uint64_t, "border.field", cap + 1);  // level-0 cells <= cap
    field = fw;
    // the dynamic shared-memory opt-in, once per context (= per device)
    if (!(ctx->attr_set & (1u << D))) {
      SBDT_CUDA_TRY(cudaFuncSetAttribute(k_field_tiles<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(field_smem_bytes<D>())));
      ctx->attr_set |= 1u << D;
    }
    k_field_tiles<D><<<sms * 3, kFieldThreads, field_smem_bytes<D>(), st>>>(og, owner, field);
    ctx->launches += 1;
  }
  ctx->launches += 6;

  SBDT_CUDA_TRY(cudaMemsetAsync(in->d_vertex_flags, 0, in->n, st));
  SBDT_CUDA_TRY(cudaMemsetAsync(infc, 0, sizeof(unsigned), st));
  tgrid.end();
  BorderArgs a;
  a.xyz = in->d_xyz;
  a.xq = xq;
  a.n = in->n;
  a.k = in->k;
  a.offsets = in->d_offsets;
  a.verts = in->d_verts;
  a.nbrs = in->d_nbrs;
  a.parity = in->d_parity;
  a.S = in->S;
  a.policy = in->policy;
  a.owner = owner;
  a.field = field;
  a.pbbox = pbbox;
  a.positive = in->d_positive;
  a.vflags = in->d_vertex_flags;
  a.spheres = in->d_spheres;
  a.inf_queue = infq;
  a.inf_count = infc;
  a.status = ctx->d_status;
  a.exact = exact_policy ? 1 : 0;
  a.cell_start = cell_start;
  a.cell_pts = cell_pts;
  a.esc = nullptr;
  a.esc_count = nullptr;
  a.esc_cap = 0;
  a.redo_bits = nullptr;
  a.redo_rows = nullptr;
  a.redo_count = nullptr;
  a.labels = in->d_labels;
  a.hull_ids = nullptr;
  a.hull_count = nullptr;
  a.hull_valid = nullptr;
  std::uint8_t *hflags = nullptr, *hpresent = nullptr;
  if (exact_policy) {
    SBDT_WS(hf, std::uint8_t, "border.hull_flags", in->n + 64);
    SBDT_WS(hi, std::uint32_t, "border.hull_ids", in->n + 64);
    SBDT_WS(hc, std::uint64_t, "border.hull_count", 1);
    SBDT_WS(hp, std::uint8_t, "border.part_present", in->k + 64);
    SBDT_WS(hv, unsigned, "border.hull_valid", 1);
    hflags = hf;
    hpresent = hp;
    a.hull_ids = hi;
    a.hull_count = reinterpret_cast<const unsigned long long*>(hc);
    a.hull_valid = hv;
  }
  // exact policy: the hull vertex set, once the hull queue is complete
  auto build_hull_set = [&]() -> int {
    if (!exact_policy) return kOk;
    SBDT_CUDA_TRY(cudaMemsetAsync(hflags, 0, in->n, st));
    SBDT_CUDA_TRY(cudaMemsetAsync(hpresent, 0, in->k, st));
    k_hull_mark<D><<<sms * 4, 256, 0, st>>>(a, hflags);
    const std::uint64_t want = (in->n + 255) / 256;
    k_part_present<<<static_cast<unsigned>(want < std::uint64_t(sms) * 8 ? (want ? want : 1) : std::uint64_t(sms) * 8),
                     256, 0, st>>>(in->d_labels, in->n, hpresent);
    k_hull_valid<<<1, 256, 0, st>>>(in->d_offsets, in->k, hpresent, const_cast<unsigned*>(a.hull_valid));
    ctx->launches += 3;
    return compact_flags(ctx, hflags, in->n, const_cast<std::uint32_t*>(a.hull_ids),
                         reinterpret_cast<std::uint64_t*>(const_cast<unsigned long long*>(a.hull_count)));
  };
  if (exact_policy) {
    unsigned long long want = 2ull * in->S + 2ull * in->n + (1ull << 20);
    // test hook: a tiny queue exercises the overflow (redo) path
    if (const char* cap_env = std::getenv("SBDT_TEST_ESC_CAP")) want = std::strtoull(cap_env, nullptr, 10);
    a.esc_cap = static_cast<unsigned>(want < 0x7FFFFFFFull ? want : 0x7FFFFFFFull);
    SBDT_WS(esc, std::uint32_t, "border.esc", 2ull * a.esc_cap + 2);
    SBDT_WS(escn, unsigned, "border.esc_n", 2);  // {queued pairs, redo rows}
    SBDT_WS(rbits, unsigned, "border.redo_bits", in->S / 32 + 1);
    SBDT_WS(rrows, std::uint32_t, "border.redo_rows", in->S + 1);
    SBDT_CUDA_TRY(cudaMemsetAsync(escn, 0, 2 * sizeof(unsigned), st));
    SBDT_CUDA_TRY(cudaMemsetAsync(rbits, 0, sizeof(unsigned) * (in->S / 32 + 1), st));
    a.esc = esc;
    a.esc_count = escn;
    a.redo_bits = rbits;
    a.redo_rows = rrows;
    a.redo_count = escn + 1;
  }
  a.counters = nullptr;
  if (ctx->census) {
    SBDT_WS(cnt, unsigned long long, "border.counters", kBorderCounters);
    SBDT_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * kBorderCounters, st));
    a.counters = cnt;
  }
  const std::size_t offs_sh = in->k + 1 <= kSmemOffsMax ? sizeof(std::uint64_t) * (in->k + 1) : 0;
  SBDT_WS(icur, unsigned, "border.inf_cursor", 2);  // {cursor, CTAs done}
  SBDT_CUDA_TRY(cudaMemsetAsync(icur, 0, 2 * sizeof(unsigned), st));
  auto infinite = [&](cudaStream_t on) {
    if (exact_policy) k_border_infinite<D, true><<<sms * 4, kWideWarps * 32, offs_sh, on>>>(a, og, icur, icur + 1);
    else k_border_infinite<D, false><<<sms * 4, kWideWarps * 32, offs_sh, on>>>(a, og, icur, icur + 1);
  };
  bool inf_forked = false;  // device path: the hull rows ran on the side stream
  // host path, grid policy: a chunk's positive flags are final once its rows
  // went through all stages; they are downloaded while later chunks run
  const bool stream_out = ctx->positive_host && !exact_policy;
  {
    const std::uint64_t want = (in->S + kBThreads - 1) / kBThreads;
    const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 32 ? want : std::uint64_t(sms) * 32);
    {
      if (tiled && in->S > 0) {
        int per_sm = 1;
        const bool bigk = in->k + 1 > kSmemOffsMax;
        if (bigk) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_border_prefilter<D, true>, kPfThreads, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_border_prefilter<D, false>, kPfThreads, offs_sh);
        const std::uint64_t resA = std::uint64_t(sms) * std::uint64_t(per_sm > 0 ? per_sm : 1);
        // candidates <= rows, plus < kQChunk holes per prefilter warp and launch
        const std::uint64_t launches_A = ctx->chunks.empty() ? 1 : ctx->chunks.size();
        const std::uint64_t qcap = in->S + 32 + launches_A * resA * (kPfThreads / 32) * kQChunk;
        SBDT_WS(cq, std::uint32_t, "border.cand", qcap * 2);  // SoA {row, reach (kReachCheckOrient marker)}
        // {candidates, cursor, wide rows, wide cursor, CTAs done (exact), CTAs done (wide)}
        // {candidates, cursor, wide rows, wide cursor, CTAs done (exact), CTAs done (wide), light wide rows}
        SBDT_WS(cn, unsigned, "border.cand_n", 8);
        SBDT_CUDA_TRY(cudaMemsetAsync(cn, 0, 8 * sizeof(unsigned), st));
        // device path: one exact and one wide launch, the wide queue split
        // by cost class (host path: the launches per chunk share one cursor)
        unsigned* nlight = ctx->chunks.empty() ? cn + 6 : nullptr;
        const std::uint64_t wcap = qcap;  // wide rows <= candidates
        SBDT_WS(wq, std::uint32_t, "border.wide", wcap * (2 * D + 3));  // SoA {row, ids, U[D], reach}
        // rows the prefilter routes to the pyramid descent directly (range
        // wider than the flattened scan's): {row, vertex ids}, counters
        // {heavy rows, cursor, CTAs done, light rows}
        const std::uint64_t pcap = in->S + 64;
        SBDT_WS(pq, std::uint32_t, "border.pf_wide", pcap * (2 * D + 3));
        SBDT_WS(pn, unsigned, "border.pf_wide_n", 4);
        SBDT_CUDA_TRY(cudaMemsetAsync(pn, 0, 4 * sizeof(unsigned), st));
        unsigned* pnlight = ctx->chunks.empty() ? pn + 3 : nullptr;
        // the prefilter's open rows with a narrow range go to the cell scan
        // first (grid policy: cell boxes in binary32; exact policy: the
        // foreign cells' points in binary64 against the recorded balls): SoA
        // {row, U[D], Rp, reach}, counters {rows, cursor, CTAs done}
        std::uint32_t* sq = nullptr;
        unsigned* sn = nullptr;
        const std::uint64_t scap = in->S + 64;
        {
          SBDT_WS(sqw, std::uint32_t, "border.scan_q", scap * (D + 3));
          SBDT_WS(snw, unsigned, "border.scan_n", 4);
          SBDT_CUDA_TRY(cudaMemsetAsync(snw, 0, 4 * sizeof(unsigned), st));
          sq = sqw;
          sn = snw;
        }
        int per_sm_s = 1;
        if (exact_policy)
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s, k_border_scan32<D, true>, kScanWarps * 32, offs_sh);
        else
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s, k_border_scan32<D, false>, kScanWarps * 32, offs_sh);
        const unsigned resS = static_cast<unsigned>(sms * (per_sm_s > 0 ? per_sm_s : 1));
        auto scan32 = [&]() {
          if (exact_policy)
            k_border_scan32<D, true><<<resS, kScanWarps * 32, offs_sh, st>>>(a, og, sq, scap, sn, sn + 1, sn + 2, cq, qcap,
                                                                            cn);
          else
            k_border_scan32<D, false><<<resS, kScanWarps * 32, offs_sh, st>>>(a, og, sq, scap, sn, sn + 1, sn + 2, cq, qcap,
                                                                             cn);
          ++ctx->launches;
        };
        if (exact_policy)
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_border_exact<D, true>, kExactWarps * 32, offs_sh);
        else
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_border_exact<D, false>, kExactWarps * 32, offs_sh);
        const unsigned resX = static_cast<unsigned>(sms * (per_sm > 0 ? per_sm : 1));
        if (exact_policy)
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_border_wide<D, true>, kWideWarps * 32, offs_sh);
        else
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_border_wide<D, false>, kWideWarps * 32, offs_sh);
        const unsigned resW = static_cast<unsigned>(sms * (per_sm > 0 ? per_sm : 1));
        SBDT_WS(pfcur, unsigned long long, "border.pf_cursor", 1);
        auto prefilter = [&](std::uint64_t r0, std::uint64_t r1) -> int {
          const std::uint64_t want = (r1 - r0 + kPfThreads - 1) / kPfThreads;
          SBDT_CUDA_TRY(cudaMemsetAsync(pfcur, 0, sizeof(unsigned long long), st));
          if (bigk)
            k_border_prefilter<D, true><<<static_cast<unsigned>(want < resA ? want : resA), kPfThreads, 0, st>>>(
                a, og, cq, qcap, cn, r0, r1, pfcur, pq, pcap, pn, pnlight, sq, scap, sn);
          else
            k_border_prefilter<D, false><<<static_cast<unsigned>(want < resA ? want : resA), kPfThreads, offs_sh, st>>>(
                a, og, cq, qcap, cn, r0, r1, pfcur, pq, pcap, pn, pnlight, sq, scap, sn);
          return kOk;
        };
        auto exact = [&]() {
          if (exact_policy)
            k_border_exact<D, true><<<resX, kExactWarps * 32, offs_sh, st>>>(a, og, cq, qcap, cn, cn + 1, wq, cn + 2,
                                                                            cn + 4, nlight);
          else
            k_border_exact<D, false><<<resX, kExactWarps * 32, offs_sh, st>>>(a, og, cq, qcap, cn, cn + 1, wq, cn + 2,
                                                                             cn + 4, nlight);
        };
        // the exact stage's forwarded rows (wq), or the prefilter's (pq)
        auto wide = [&](bool from_pf, cudaStream_t on) {
          std::uint32_t* q = from_pf ? pq : wq;
          const std::uint64_t qc = from_pf ? pcap : wcap;
          unsigned* nh = from_pf ? pn : cn + 2;
          unsigned* cur = from_pf ? pn + 1 : cn + 3;
          unsigned* fin = from_pf ? pn + 2 : cn + 5;
          unsigned* nl = from_pf ? pnlight : nlight;
          if (exact_policy)
            k_border_wide<D, true><<<resW, kWideWarps * 32, offs_sh, on>>>(a, og, q, qc, nh, cur, fin, nl);
          else
            k_border_wide<D, false><<<resW, kWideWarps * 32, offs_sh, on>>>(a, og, q, qc, nh, cur, fin, nl);
        };
        if (ctx->chunks.empty()) {
          {
            StageTimer ta(ctx, "border.prefilter");
            const int prc = prefilter(0, in->S);
            if (prc != kOk) return prc;
          }
          // the prefilter's queue length: the orientation checks read only
          // its entries (k_border_scan32 appends to the same queue meanwhile)
          SBDT_CUDA_TRY(cudaMemcpyAsync(cn + 7, cn, sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
          // the hull queue is complete once the prefilter ran: its halfspace
          // kernel (few rows, latency-bound) overlaps the exact stages on the
          // side stream and joins before the escalation / compaction
          {
            const int hrc = build_hull_set();
            if (hrc != kOk) return hrc;
          }
          // the hull-row and wide-row descents are the longest latency-bound
          // chains after the prefilter: their streams get the highest
          // priority, so their CTAs are placed first and the binary32 scan
          // and the exact stage fill the remaining slots
          if (!ctx->side_stream)
            SBDT_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->side_stream, cudaStreamNonBlocking, prio_hi));
          if (!ctx->fork_ev) SBDT_CUDA_TRY(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
          if (!ctx->join_ev) SBDT_CUDA_TRY(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
          SBDT_CUDA_TRY(cudaEventRecord(ctx->fork_ev, st));
          SBDT_CUDA_TRY(cudaStreamWaitEvent(ctx->side_stream, ctx->fork_ev, 0));
          {
            StageTimer ti(ctx, "border.infinite", ctx->side_stream);
            infinite(ctx->side_stream);
          }
          k_border_orient<D><<<sms * 4, 256, 0, ctx->side_stream>>>(a, cq, qcap, cn + 7);
          ++ctx->launches;
          SBDT_CUDA_TRY(cudaEventRecord(ctx->join_ev, ctx->side_stream));
          inf_forked = true;
          // the prefilter's wide rows on a second side stream, next to the exact stage
          if (!ctx->wide_stream)
            SBDT_CUDA_TRY(cudaStreamCreateWithPriority(&ctx->wide_stream, cudaStreamNonBlocking, prio_hi));
          if (!ctx->wide_join_ev) SBDT_CUDA_TRY(cudaEventCreateWithFlags(&ctx->wide_join_ev, cudaEventDisableTiming));
          SBDT_CUDA_TRY(cudaStreamWaitEvent(ctx->wide_stream, ctx->fork_ev, 0));
          {
            StageTimer tw(ctx, "border.wide", ctx->wide_stream);
            wide(true, ctx->wide_stream);
          }
          SBDT_CUDA_TRY(cudaEventRecord(ctx->wide_join_ev, ctx->wide_stream));
          {
            StageTimer ts(ctx, "border.scan32");
            scan32();
          }
          {
            StageTimer tx(ctx, "border.exact");
            exact();
          }
          {
            StageTimer tw(ctx, "border.exact_wide");
            wide(false, st);
          }
          SBDT_CUDA_TRY(cudaStreamWaitEvent(st, ctx->join_ev, 0));
          SBDT_CUDA_TRY(cudaStreamWaitEvent(st, ctx->wide_join_ev, 0));
          ctx->launches += 5;
        } else {
          // host path: every chunk of rows as soon as its upload has landed;
          // the exact and wide kernels drain the queues grown so far (their
          // cursors persist), so all three overlap the remaining uploads
          std::uint64_t r0 = 0;
          for (const auto& c : ctx->chunks) {
            const std::uint64_t r1 = c.first < in->S ? c.first : in->S;
            SBDT_CUDA_TRY(cudaStreamWaitEvent(st, c.second, 0));
            if (r1 > r0) {
              const int prc = prefilter(r0, r1);
              if (prc != kOk) return prc;
              wide(true, st);
              scan32();
              exact();
              wide(false, st);
              ctx->launches += 4;
              if (stream_out) {
                infinite(st);
                ++ctx->launches;
                cudaEvent_t ev = ctx->chunk_done[&c - &ctx->chunks[0]];
                SBDT_CUDA_TRY(cudaEventRecord(ev, st));
                SBDT_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ev, 0));
                SBDT_CUDA_TRY(cudaMemcpyAsync(ctx->positive_host + r0, in->d_positive + r0, r1 - r0,
                                              cudaMemcpyDeviceToHost, ctx->d2h_stream));
              }
            }
            r0 = r1;
          }
          k_border_orient<D><<<sms * 4, 256, 0, st>>>(a, cq, qcap, cn);
          ++ctx->launches;
        }
        if (a.counters) {
          k_cand_count<<<1, 1, 0, st>>>(cn, pn, in->S, a.counters, a.esc_count, a.esc_cap);
          ctx->launches += 1;
        }
      } else if (blocks > 0) {
        for (const auto& c : ctx->chunks) SBDT_CUDA_TRY(cudaStreamWaitEvent(st, c.second, 0));
        StageTimer t(ctx, "border.finite");
        k_border_finite<D><<<blocks, kBThreads, offs_sh, st>>>(a, og);
      }
    }
    for (const auto& c : ctx->chunks) SBDT_CUDA_TRY(cudaStreamWaitEvent(st, c.second, 0));
    if (!inf_forked) {
      const int hrc = build_hull_set();
      if (hrc != kOk) return hrc;
      StageTimer t(ctx, "border.infinite");
      infinite(st);  // the rows not yet drained (all of them unless the chunked path ran it)
    }
    if (exact_policy) {
      StageTimer t(ctx, "border.escalate");
      constexpr std::size_t per = D == 3 ? sbdt_pred::kInSphere3Scratch : sbdt_pred::kInSphere2Scratch;
      SBDT_WS(scr, double, "border.esc_scratch", per * kEscThreads);
      k_border_escalate<D><<<kEscThreads / 128, 128, 0, st>>>(a, scr);
      k_border_redo<D><<<kEscThreads / 128, 128, 0, st>>>(a, og, scr);
      ctx->launches += 2;
    }
    if (tiled && in->d_spheres) {
      const std::uint64_t want = (in->S + 255) / 256;
      k_border_spheres<D><<<static_cast<unsigned>(want < std::uint64_t(sms) * 16 ? want : std::uint64_t(sms) * 16),
                            256, 0, st>>>(a);
      ctx->launches += 1;
    }
    ctx->launches += inf_forked ? 0 : ((tiled && in->S > 0) ? 1 : 2);
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
