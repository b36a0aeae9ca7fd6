// Shared device-side helpers for the sm_100a kernels (libsbdt_gpu.so).
// All translation units are compiled with -fmad=false: every binary64
// expression below rounds exactly like the reference's host code.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "../common/predicates.hpp"

namespace sbdt_gpu {

constexpr std::uint32_t kInfVertex = 0xFFFFFFFFu;
constexpr std::uint16_t kOwnerEmpty = 0xFFFF;
constexpr std::uint16_t kOwnerMulti = 0xFFFE;
constexpr int kMaxLevels = 24;

// Launch accounting (gpu_launches in bench.py's JSON line).
struct LaunchCounter {
  unsigned long long launches = 0;
};

// ---- binary64 helpers --------------------------------------------------------
// Order-preserving map double -> uint64 for atomicMin/atomicMax reductions.
__host__ __device__ __forceinline__ unsigned long long dbl_to_ordered(double x) {
#if defined(__CUDA_ARCH__)
  unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
#else
  unsigned long long u;
  __builtin_memcpy(&u, &x, 8);
#endif
  return (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
}
__host__ __device__ __forceinline__ double ordered_to_dbl(unsigned long long u) {
  u = (u & 0x8000000000000000ULL) ? (u & 0x7FFFFFFFFFFFFFFFULL) : ~u;
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  __builtin_memcpy(&x, &u, 8);
  return x;
#endif
}

// Deterministic cube root (basic IEEE ops only, no contraction): the grid
// edge convention shared bit-for-bit with the oracle (oracle/path.hpp). The
// reference leaves the rounding of (V/n)^(1/D) unspecified.
__host__ __device__ __forceinline__ double cbrt_det(double x) {
  if (!(x > 0.0)) return 0.0;
  int e;
  double m = frexp(x, &e);  // x = m * 2^e, m in [0.5, 1)
  int r = e % 3;
  if (r < 0) r += 3;
  m = ldexp(m, r);  // m in [0.5, 4)
  e -= r;
  double y = 1.0;
  for (int it = 0; it < 8; ++it) y = y - (y * y * y - m) / (3.0 * y * y);
  return ldexp(y, e / 3);
}

// ---- grid ---------------------------------------------------------------------
template <int D>
struct Grid {
  double lo[D];
  double edge;
  long long dims[D];
};

template <int D>
__device__ __forceinline__ long long cell_coord(const Grid<D>& g, double x, int d) {
  const double f = floor((x - g.lo[d]) / g.edge);
  long long c;
  if (!(f >= 0.0)) c = 0;  // also NaN
  else if (f >= static_cast<double>(g.dims[d] - 1)) c = g.dims[d] - 1;
  else c = static_cast<long long>(f);
  return c;
}

// cell_coord through a product with the rounded reciprocal of the edge, exact:
// y = (x - lo) * inv_edge is within ~3.3e-16 |y| of the correctly rounded
// quotient q of cell_coord, so floor(y) == floor(q) unless an integer lies
// within that distance of y; those (rare) cases take the division.
template <int D>
__device__ __forceinline__ long long cell_coord_fast(const Grid<D>& g, double inv_edge, double x, int d) {
  const double y = (x - g.lo[d]) * inv_edge;
  const double fy = floor(y);
  const double fr = y - fy;  // exact
  const double m = fmax(fabs(y), 1.0) * 4e-15;
  if (!(fr > m && fr < 1.0 - m)) return cell_coord<D>(g, x, d);
  long long c;
  if (!(fy >= 0.0)) c = 0;
  else if (fy >= static_cast<double>(g.dims[d] - 1)) c = g.dims[d] - 1;
  else c = static_cast<long long>(fy);
  return c;
}
template <int D>
__device__ __forceinline__ double cell_lo(const Grid<D>& g, long long i, int d) {
  return g.lo[d] + static_cast<double>(i) * g.edge;
}

// box_sphere_overlap (geometry.hpp:185-201), identical operation order.
template <int D>
__device__ __forceinline__ bool box_sphere(const double* blo, const double* bhi, const double* c, double r2) {
  double d2 = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double g = 0.0;
    if (c[d] < blo[d]) g = blo[d] - c[d];
    else if (c[d] > bhi[d]) g = c[d] - bhi[d];
    d2 += g * g;
  }
  return d2 <= r2;
}

// Far-corner containment: true implies box_sphere() holds for every sub-box
// (rounding is monotone).
template <int D>
__device__ __forceinline__ bool box_inside_sphere(const double* blo, const double* bhi, const double* c, double r2) {
  double d2 = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double a = c[d] - blo[d];
    const double b = bhi[d] - c[d];
    const double f = a > b ? a : b;
    d2 += f * f;
  }
  return d2 <= r2;
}

// Exact orientation (filter, then expansion arithmetic when it cannot
// decide); `escalations` (optional census counter) counts the expansion runs.
template <int D>
__device__ __forceinline__ int orient_dev(const double* const* p, unsigned long long* escalations = nullptr) {
  int r;
  if constexpr (D == 2) r = sbdt_pred::orient2_filtered(p[0], p[1], p[2]);
  else r = sbdt_pred::orient3_filtered(p[0], p[1], p[2], p[3]);
  if (r != 2) return r;
  if (escalations) atomicAdd(escalations, 1ull);
  if constexpr (D == 2) return sbdt_pred::orient2_exact(p[0], p[1], p[2]);
  else return sbdt_pred::orient3_exact(p[0], p[1], p[2], p[3]);
}

// squared_distance (geometry.hpp:102-110): s = 0; s += t*t left to right.
template <int D>
__device__ __forceinline__ double sqdist(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double t = a[d] - b[d];
    s += t * t;
  }
  return s;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Queue cursors: warps claim batches of 32 with atomicAdd, so a drained
// cursor overshoots the queue length; the last CTA of a launch rewinds it to
// the length the launch worked on, so a later launch over a grown queue
// (host-path chunks) resumes exactly there.
__device__ __forceinline__ unsigned claim_batch(unsigned* next, unsigned batch = 32u) {
  unsigned base = 0;
  if ((threadIdx.x & 31u) == 0) base = atomicAdd(next, batch);
  return __shfl_sync(0xffffffffu, base, 0);
}

__device__ __forceinline__ void rewind_cursor(unsigned* next, unsigned* fin, unsigned limit) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(fin, 1u) == gridDim.x - 1) {
      *next = limit;
      *fin = 0u;
      __threadfence();
    }
  }
}

}  // namespace sbdt_gpu

#define SBDT_CUDA_TRY(expr)                                              \
  do {                                                                   \
    cudaError_t e_ = (expr);                                             \
    if (e_ != cudaSuccess) return ::sbdt_gpu::fail_cuda(ctx, e_, #expr); \
  } while (0)
