// K1/K2/K3 — point-to-partition assignment (Alg. 2 line
// "find nearest sample point") on sm_100a.
//
// label(p) = sample_labels[argmin_s squared_distance(p, s)], ties -> lowest
// sample PointId, with squared_distance evaluated exactly as
// geometry.hpp:102-110 (binary64, left-to-right, no contraction), so labels
// are bit-identical to a brute-force scan.
//
// K1  sample grid: samples gathered into 32-byte records {x,y,z,pid,label}
//     bucketed by a uniform grid (~2 samples/cell, one extra cell layer around
//     the sample bbox) -> CSR. O(m), L2 resident.
// K1b Voronoi label table (VLT): every grid cell is split into F^D fine cells;
//     for each fine cell a CONSERVATIVE candidate set of samples that can be
//     the binary64 argmin for some point of the (slightly inflated) cell is
//     computed (dominance test against the nearest sample of the cell
//     centre with a rigorous margin). Record = UNIFORM(label)
//     when all candidates share one label, else up to 7 candidate indices,
//     else OVERFLOW. One warp per grid cell; O(m) work, ~4m records.
// K2  point pass: stream the coordinates, bin into a fine cell, read one
//     32-byte record; uniform -> label, list -> exact binary64 argmin over the
//     candidates, overflow / outside the table -> exact ring search. The
//     global point bbox (min/max) is fused (input of the grid index).
// K3  stable counting sort by label -> Partitioning.parts (ascending ids).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "context.cuh"
#include "scan.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {

struct __align__(16) SampleRec {
  double x[3];
  std::uint32_t pid;
  std::uint32_t label;
};

template <int D>
constexpr int fine_factor() {
  return D == 3 ? 2 : 3;
}
template <int D>
constexpr int fine_per_cell() {
  return D == 3 ? 8 : 9;
}

template <int D>
struct SampleGrid {
  Grid<D> g;
  double margin;         // binning + rounding slack in coordinate units (ring search)
  double inv_ef;         // F / edge (fine binning)
  double ef;             // edge / F
  double delta_f;        // fine-box inflation
  double delta_c;        // coarse-box inflation (> fine inflation)
  unsigned long long cells;
  int refined;            // cells shrunk for clustered samples: only cells with samples nearby get a table record
};

constexpr int kBlock = 256;

// Block-reduce local bbox then one atomic per block per coordinate.
template <int D>
__device__ __forceinline__ void bbox_flush(const double* lo, const double* hi, unsigned long long* bbox) {
  __shared__ unsigned long long s_lo[D], s_hi[D];
  if (threadIdx.x < D) {
    s_lo[threadIdx.x] = 0xFFFFFFFFFFFFFFFFULL;
    s_hi[threadIdx.x] = 0ULL;
  }
  __syncthreads();
#pragma unroll
  for (int d = 0; d < D; ++d) {
    double a = lo[d], b = hi[d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane_id() == 0) {
      atomicMin(&s_lo[d], dbl_to_ordered(a));
      atomicMax(&s_hi[d], dbl_to_ordered(b));
    }
  }
  __syncthreads();
  if (threadIdx.x < D) {
    atomicMin(&bbox[threadIdx.x], s_lo[threadIdx.x]);
    atomicMax(&bbox[D + threadIdx.x], s_hi[threadIdx.x]);
  }
}

__global__ void k_bbox_init(unsigned long long* bbox, int dim) {
  if (threadIdx.x < static_cast<unsigned>(dim)) {
    bbox[threadIdx.x] = 0xFFFFFFFFFFFFFFFFULL;
    bbox[dim + threadIdx.x] = 0ULL;
  }
}

template <int D>
__global__ void k_sample_gather(const double* __restrict__ xyz, const std::uint32_t* __restrict__ sample_ids,
                                const std::uint32_t* __restrict__ sample_labels, std::uint32_t m,
                                SampleRec* __restrict__ recs, unsigned long long* bbox,
                                const double* __restrict__ sxyz) {
  double lo[D], hi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) lo[d] = INFINITY, hi[d] = -INFINITY;
  for (std::uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    const std::uint32_t pid = sample_ids[s];
    SampleRec r;
#pragma unroll
    for (int d = 0; d < 3; ++d) r.x[d] = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      r.x[d] = sxyz ? sxyz[std::size_t(s) * D + d] : xyz[std::size_t(pid) * D + d];
      lo[d] = fmin(lo[d], r.x[d]);
      hi[d] = fmax(hi[d], r.x[d]);
    }
    r.pid = pid;
    r.label = sample_labels[s];
    recs[s] = r;
  }
  bbox_flush<D>(lo, hi, bbox);
}

// Sample-grid parameters for cell edge e over the bbox: one cell of padding
// on every side; the edge doubled until the cell count fits cap.
template <int D>
__device__ void sample_grid_set(const unsigned long long* bbox, double e, unsigned long long cap, SampleGrid<D>* sg) {
  double lo[D], hi[D], ext_max = 0.0, mag = 0.0;
  for (int d = 0; d < D; ++d) {
    lo[d] = ordered_to_dbl(bbox[d]);
    hi[d] = ordered_to_dbl(bbox[D + d]);
    ext_max = fmax(ext_max, hi[d] - lo[d]);
    mag = fmax(mag, fmax(fabs(lo[d]), fabs(hi[d])));
  }
  if (!(e > 0.0)) e = ext_max > 0.0 ? ext_max / 64.0 : 1.0;
  unsigned long long cells;
  long long dims[D];
  for (;;) {
    cells = 1;
    for (int d = 0; d < D; ++d) {
      dims[d] = static_cast<long long>(floor((hi[d] - lo[d]) / e)) + 3;
      cells *= static_cast<unsigned long long>(dims[d]);
    }
    if (cells <= cap) break;
    // grow the edge to about the cap (with a 2% margin; at least by 1%)
    const double g = (D == 2 ? sqrt(static_cast<double>(cells) / cap) : cbrt_det(static_cast<double>(cells) / cap));
    e *= fmax(1.01, g * 1.02);
  }
  for (int d = 0; d < D; ++d) {
    sg->g.lo[d] = lo[d] - e;
    sg->g.dims[d] = dims[d];
  }
  sg->g.edge = e;
  sg->cells = cells;
  mag += e;
  sg->margin = 1e-12 * (mag + ext_max + e);
  constexpr int F = fine_factor<D>();
  sg->ef = e / F;
  sg->inv_ef = 1.0 / sg->ef;
  sg->delta_f = 1e-9 * sg->ef + 1e-12 * (mag + ext_max);
  sg->delta_c = 2.0 * sg->delta_f + 1e-9 * e;
}

// ~2 samples per cell of the bbox volume
template <int D>
__global__ void k_sample_grid_params(const unsigned long long* bbox, std::uint32_t m, unsigned long long cap,
                                     SampleGrid<D>* sg) {
  double vol = 1.0;
  for (int d = 0; d < D; ++d) vol *= ordered_to_dbl(bbox[D + d]) - ordered_to_dbl(bbox[d]);
  const double per = 2.0 * vol / static_cast<double>(m > 0 ? m : 1);
  sample_grid_set<D>(bbox, (D == 2) ? sqrt(per) : cbrt_det(per), cap, sg);
  sg->refined = 0;
}

// Clustered samples (surfaces, lines, dense cores): q = samples per occupied
// cell of that grid. Above 4 the edge shrinks by (q / 2)^(1 / D) (the volume
// estimate: a dense core gets ~2 samples per cell; a lower-dimensional
// structure keeps more, which the table's adaptive sub-boxes absorb, while a
// finer grid would leave the sparse regions' points to long ring searches),
// within cap cells; the table is
// then built only for cells with samples in their 3^D neighbourhood (the
// others send their points to the exact ring search), so the extra empty
// cells cost one head each.
// Occupied cells holding a single sample (the first grid's sparse regions).
template <int D>
__global__ void k_sample_singletons(const std::uint32_t* __restrict__ counts, const SampleGrid<D>* __restrict__ sg,
                                    unsigned* __restrict__ singles) {
  const unsigned long long cells = sg->cells;
  unsigned c = 0;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < cells;
       i += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
    c += counts[i] == 1u ? 1u : 0u;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31u) == 0 && c) atomicAdd(singles, c);
}

template <int D>
__global__ void k_sample_grid_refine(const unsigned long long* bbox, std::uint32_t m, unsigned long long cap,
                                     const unsigned* __restrict__ occupied, SampleGrid<D>* sg) {
  const unsigned occ = occupied[0] > 0 ? occupied[0] : 1u;
  const double q = static_cast<double>(m) / static_cast<double>(occ);
  // many single-sample cells: a wide density range (a dense core with sparse
  // tails), where the refined grid's sparse regions would send their points
  // to long ring searches; refine only structures without them
  if (!(q > 4.0) || !(static_cast<double>(occupied[1]) < 0.15 * static_cast<double>(occ))) return;
  const double r = D == 2 ? sqrt(0.5 * q) : cbrt_det(0.5 * q);
  sample_grid_set<D>(bbox, sg->g.edge / r, cap, sg);
  sg->refined = 1;
}

template <int D>
__device__ __forceinline__ long long linear(const Grid<D>& g, const long long* c) {
  long long id = c[D - 1];
#pragma unroll
  for (int d = D - 2; d >= 0; --d) id = id * g.dims[d] + c[d];
  return id;
}

template <int D>
__global__ void k_sample_count(const SampleRec* __restrict__ recs, std::uint32_t m, const SampleGrid<D>* sgp,
                               std::uint32_t* __restrict__ counts, std::uint32_t* __restrict__ cell_of,
                               unsigned* __restrict__ occupied = nullptr) {
  const Grid<D> g = sgp->g;
  for (std::uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    long long c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) c[d] = cell_coord<D>(g, recs[s].x[d], d);
    const std::uint32_t cell = static_cast<std::uint32_t>(linear<D>(g, c));
    cell_of[s] = cell;
    if (atomicAdd(&counts[cell], 1u) == 0u && occupied) atomicAdd(occupied, 1u);
  }
}

__global__ void k_sample_scatter(const SampleRec* __restrict__ recs, std::uint32_t m,
                                 const std::uint32_t* __restrict__ cell_of, const std::uint32_t* __restrict__ starts,
                                 std::uint32_t* __restrict__ fill, SampleRec* __restrict__ sorted) {
  for (std::uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    const std::uint32_t c = cell_of[s];
    sorted[starts[c] + atomicAdd(&fill[c], 1u)] = recs[s];
  }
}

// Exact nearest-sample label by Chebyshev rings over the sample grid: a ring
// is the last one visited only when a rigorous lower bound (binning error +
// rounding margin) proves every unvisited sample strictly farther in binary64.
template <int D>
__device__ __noinline__ std::uint32_t nearest_label_ring(const double* x, const Grid<D>& g, double margin,
                                            const std::uint32_t* __restrict__ starts,
                                            const SampleRec* __restrict__ sorted) {
  long long ci[D];
#pragma unroll
  for (int d = 0; d < D; ++d) ci[d] = cell_coord<D>(g, x[d], d);
  double best = INFINITY;
  std::uint32_t best_pid = 0xFFFFFFFFu, best_label = 0;
  for (long long r = 0;; ++r) {
    long long lo_c[D], hi_c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      lo_c[d] = ci[d] - r < 0 ? 0 : ci[d] - r;
      hi_c[d] = ci[d] + r > g.dims[d] - 1 ? g.dims[d] - 1 : ci[d] + r;
    }
    // the shell of Chebyshev radius r only: rows along axis 0 over the
    // (D-1)-dimensional cross-section; a row on the shell's side faces is
    // scanned whole, an interior row contributes its two end cells
    long long rows = 1;
#pragma unroll
    for (int d = 1; d < D; ++d) rows *= (hi_c[d] - lo_c[d] + 1);
    for (long long t = 0; t < rows; ++t) {
      long long c[D], rem = t, cheb = 0;
#pragma unroll
      for (int d = 1; d < D; ++d) {
        const long long span = hi_c[d] - lo_c[d] + 1;
        c[d] = lo_c[d] + rem % span;
        rem /= span;
        const long long dd = c[d] > ci[d] ? c[d] - ci[d] : ci[d] - c[d];
        cheb = dd > cheb ? dd : cheb;
      }
      long long xs[2];
      int nx = 0;
      if (cheb == r) {
        xs[0] = lo_c[0];
        xs[1] = hi_c[0];
        nx = -1;  // the whole row
      } else {
        if (ci[0] - r >= 0) xs[nx++] = ci[0] - r;
        if (r > 0 && ci[0] + r <= g.dims[0] - 1) xs[nx++] = ci[0] + r;
      }
      auto scan_cell = [&](long long x0) {
        c[0] = x0;
        const long long cell = linear<D>(g, c);
        for (std::uint32_t s = starts[cell], e = starts[cell + 1]; s < e; ++s) {
          const SampleRec rec = sorted[s];
          const double d2 = sqdist<D>(x, rec.x);
          if (d2 < best || (d2 == best && rec.pid < best_pid)) {
            best = d2;
            best_pid = rec.pid;
            best_label = rec.label;
          }
        }
      };
      if (nx < 0) {
        for (long long x0 = xs[0]; x0 <= xs[1]; ++x0) scan_cell(x0);
      } else {
        for (int k = 0; k < nx; ++k) scan_cell(xs[k]);
      }
    }
    double lb = INFINITY;
    bool any = false;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (ci[d] - r > 0) {
        lb = fmin(lb, x[d] - cell_lo<D>(g, ci[d] - r, d));
        any = true;
      }
      if (ci[d] + r < g.dims[d] - 1) {
        lb = fmin(lb, cell_lo<D>(g, ci[d] + r + 1, d) - x[d]);
        any = true;
      }
    }
    if (!any) break;
    lb -= margin;
    if (lb > 0.0 && (lb * lb) * (1.0 - 1e-12) > best) break;
  }
  return best_label;
}

// ---- helpers shared with the Voronoi label table ---------------------------------
template <int D>
__device__ __forceinline__ void warp_argmin(double& d2, std::uint32_t& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, d2, o);
    const std::uint32_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (od < d2 || (od == d2 && oi < idx)) {
      d2 = od;
      idx = oi;
    }
  }
}

}  // namespace sbdt_gpu

#include "vlt.cuh"

namespace sbdt_gpu {

// ---- K3: stable bucketing of point ids by label ------------------------------
constexpr int kBucketTile = 4096;  // points per CTA tile
constexpr int kBucketThreads = 256;

// Both bucketing kernels work on the labels [l0, l0 + kl) (kl <= kBucketLabels,
// so the shared histograms fit for any k; larger k takes several passes).
constexpr std::uint32_t kBucketLabels = 1024;

__global__ void k_bucket_count(const std::uint32_t* __restrict__ labels, std::uint64_t n, std::uint32_t l0,
                               std::uint32_t kl, std::uint32_t* __restrict__ tile_counts /* [k][tiles] */,
                               std::uint32_t tiles) {
  extern __shared__ std::uint32_t hist[];
  for (std::uint32_t j = threadIdx.x; j < kl; j += blockDim.x) hist[j] = 0;
  __syncthreads();
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kBucketTile;
  for (int t = threadIdx.x; t < kBucketTile; t += blockDim.x) {
    const std::uint64_t i = base + t;
    if (i < n) {
      const std::uint32_t l = labels[i] - l0;
      if (l < kl) atomicAdd(&hist[l], 1u);
    }
  }
  __syncthreads();
  for (std::uint32_t j = threadIdx.x; j < kl; j += blockDim.x)
    tile_counts[std::uint64_t(l0 + j) * tiles + blockIdx.x] = hist[j];
}

// Stable scatter: each warp owns a contiguous slice of the tile; per-warp
// label histograms give exact in-order ranks.
__global__ void __launch_bounds__(kBucketThreads) k_bucket_scatter(const std::uint32_t* __restrict__ labels,
                                                                   std::uint64_t n, std::uint32_t l0,
                                                                   std::uint32_t k,
                                                                   const std::uint32_t* __restrict__ tile_offsets,
                                                                   std::uint32_t tiles,
                                                                   std::uint32_t* __restrict__ part_ids) {
  extern __shared__ std::uint32_t sh[];  // [warps][k], labels l0 .. l0 + k - 1
  constexpr int kWarps = kBucketThreads / 32;
  constexpr int kSlice = kBucketTile / kWarps;
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  for (std::uint32_t j = threadIdx.x; j < k * kWarps; j += blockDim.x) sh[j] = 0;
  __syncthreads();
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kBucketTile + std::uint64_t(warp) * kSlice;
  for (int t = lane; t < kSlice; t += 32) {
    const std::uint64_t i = base + t;
    if (i < n) {
      const std::uint32_t l = labels[i] - l0;
      if (l < k) atomicAdd(&sh[warp * k + l], 1u);
    }
  }
  __syncthreads();
  // exclusive scan across warps per label, plus the tile's global offset
  for (std::uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
    std::uint32_t run = tile_offsets[std::uint64_t(l0 + j) * tiles + blockIdx.x];
    for (int w = 0; w < kWarps; ++w) {
      const std::uint32_t c = sh[w * k + j];
      sh[w * k + j] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int t0 = 0; t0 < kSlice; t0 += 32) {
    const std::uint64_t i = base + t0 + lane;
    const std::uint32_t l = i < n ? labels[i] - l0 : 0xFFFFFFFFu;
    const bool valid = l < k;
    const std::uint32_t lab = valid ? l : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xffffffffu, lab);
    const unsigned rank = __popc(peers & ((1u << lane) - 1u));
    const int leader = __ffs(peers) - 1;
    std::uint32_t basepos = 0;
    if (valid) basepos = sh[warp * k + lab];
    __syncwarp();
    if (valid) part_ids[basepos + rank] = static_cast<std::uint32_t>(i);
    if (valid && static_cast<int>(lane) == leader) sh[warp * k + lab] = basepos + __popc(peers);
    __syncwarp();
  }
}

// tile_offsets[j][t] = part_offset[j] + sum_{t'<t} counts[j][t'] via one flat
// exclusive scan over the label-major [k][tiles] matrix.
__global__ void k_part_offsets(const std::uint32_t* __restrict__ tile_offsets, std::uint32_t k, std::uint32_t tiles,
                               std::uint64_t n, std::uint64_t* __restrict__ part_offsets, unsigned* status) {
  for (std::uint32_t j = threadIdx.x; j <= k; j += blockDim.x)
    part_offsets[j] = (j == k) ? n : tile_offsets[std::uint64_t(j) * tiles];
  // every label < k was counted: a total short of n means some label >= k
  // (a sample label out of range on the device-pointer path)
  if (threadIdx.x == 0 && tile_offsets[std::uint64_t(k) * tiles] != n) atomicOr(status, kStLabelRange);
}

// ---------------------------------------------------------------------------
template <int D>
int assign_impl(sbdt_gpu_ctx* ctx, const double* d_xyz, std::uint64_t n, const std::uint32_t* d_sample_ids,
                const std::uint32_t* d_sample_labels, std::uint32_t m, std::uint32_t* d_labels,
                unsigned long long* d_bbox) {
  cudaStream_t st = ctx->stream;
  const unsigned long long cap0 = 2ULL * m + 1024;  // pools sized from the bbox grid
  const unsigned long long cap = std::min(16ULL * m + 1024, 1ULL << 31);  // cells of a refined grid (clustered samples)
  SBDT_WS(recs, SampleRec, "assign.recs", m);
  SBDT_WS(sorted, SampleRec, "assign.sorted", m);
  SBDT_WS(sbbox, unsigned long long, "assign.sbbox", 2 * D);
  SBDT_WS(sg, SampleGrid<D>, "assign.sg", 1);
  SBDT_WS(counts, std::uint32_t, "assign.counts", cap + 1);
  SBDT_WS(starts, std::uint32_t, "assign.starts", cap + 1);
  SBDT_WS(cell_of, std::uint32_t, "assign.cell_of", m);
  SBDT_WS(blocksums, std::uint32_t, "assign.blocksums", (cap + 1) / kScanTile + 2);
  const unsigned long long fine = cap * fine_per_cell<D>();
  SBDT_WS(heads, std::uint32_t, "assign.heads", fine);
  SBDT_WS(slab, VltEntry, "assign.slab", fine * kSlots);
  const unsigned long long lcap_ll = cap0 * fine_per_cell<D>() * 24 + 4096;  // long lists (dense cells: ~100 per fine cell); full -> ring search
  const unsigned lcap = lcap_ll < (1ull << 28) ? static_cast<unsigned>(lcap_ll) : (1u << 28);
  SBDT_WS(lslab, VltEntry, "assign.lslab", lcap);
  SBDT_WS(lcount, unsigned, "assign.lcount", 1);
  const unsigned long long subcap_ll = cap0 * fine_per_cell<D>() * 8 + 4096;  // sub-box heads; full -> long lists
  const unsigned subcap = subcap_ll < (1ull << 28) ? static_cast<unsigned>(subcap_ll) : (1u << 28);
  SBDT_WS(subheads, std::uint32_t, "assign.subheads", subcap);
  SBDT_WS(subcount, unsigned, "assign.subcount", 1);
  SBDT_WS(dq, std::uint32_t, "assign.dense_q", cap + 1);
  SBDT_WS(dqn, unsigned, "assign.dense_n", 1);
  constexpr unsigned kDenseBlocks = 148 * 8;
  SBDT_WS(dscr, char, "assign.dense_scratch", vlt_dense_bytes_per_warp<D>() * kDenseBlocks * kVltWarps);
  SBDT_WS(slabels, std::uint32_t, "assign.slabels", m);
  SBDT_WS(stats, unsigned, "assign.stats", 6);
  SBDT_WS(oq, std::uint32_t, "assign.oq", n + 1);
  SBDT_WS(oqc, unsigned, "assign.oqc", 1);
  SBDT_WS(oqcur, unsigned, "assign.oq_cursor", 2);  // {cursor, CTAs done}
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const unsigned sblocks = static_cast<unsigned>((m + kBlock - 1) / kBlock);
  {
    StageTimer t0(ctx, "assign.sample_grid");
    k_bbox_init<<<1, 32, 0, st>>>(sbbox, D);
    k_bbox_init<<<1, 32, 0, st>>>(d_bbox, D);
    k_sample_gather<D><<<sblocks, kBlock, 0, st>>>(d_xyz, d_sample_ids, d_sample_labels, m, recs, sbbox,
                                                   ctx->sample_xyz);
    SBDT_WS(occ, unsigned, "assign.occupied", 2);  // {occupied cells, single-sample cells}
    k_sample_grid_params<D><<<1, 1, 0, st>>>(sbbox, m, cap0, sg);
    SBDT_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(std::uint32_t) * (cap0 + 1), st));
    SBDT_CUDA_TRY(cudaMemsetAsync(occ, 0, 2 * sizeof(unsigned), st));
    k_sample_count<D><<<sblocks, kBlock, 0, st>>>(recs, m, sg, counts, cell_of, occ);
    k_sample_singletons<D><<<static_cast<unsigned>(std::min<unsigned long long>((cap0 + 255) / 256, 1024)), 256, 0, st>>>(
        counts, sg, occ + 1);
    k_sample_grid_refine<D><<<1, 1, 0, st>>>(sbbox, m, cap, occ, sg);
    ++ctx->launches;
    SBDT_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(std::uint32_t) * (cap + 1), st));
    k_sample_count<D><<<sblocks, kBlock, 0, st>>>(recs, m, sg, counts, cell_of);
    ctx->launches += 2;
    exclusive_scan(counts, starts, cap + 1, blocksums, nullptr, st, &ctx->launches);
    SBDT_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(std::uint32_t) * (cap + 1), st));
    k_sample_scatter<<<sblocks, kBlock, 0, st>>>(recs, m, cell_of, starts, counts, sorted);
    k_sorted_labels<<<sblocks, kBlock, 0, st>>>(sorted, m, slabels);
    ctx->launches += 7;
  }
  {
    StageTimer t1(ctx, "assign.table");
    if (ctx->census) SBDT_CUDA_TRY(cudaMemsetAsync(stats, 0, sizeof(unsigned) * 6, st));
    SBDT_CUDA_TRY(cudaMemsetAsync(lcount, 0, sizeof(unsigned), st));
    SBDT_CUDA_TRY(cudaMemsetAsync(dqn, 0, sizeof(unsigned), st));
    SBDT_CUDA_TRY(cudaMemsetAsync(subcount, 0, sizeof(unsigned), st));
    k_vlt_build<D, false><<<sms * 16, 32 * kVltWarps, 0, st>>>(sg, starts, sorted, heads, slab, lslab, lcount, lcap,
                                                                  ctx->census ? stats : nullptr, dq, dqn, nullptr,
                                                                  subheads, subcount, subcap);
    // coarse cells with more than kVltCap candidates (clustered samples)
    k_vlt_build<D, true><<<kDenseBlocks, 32 * kVltWarps, 0, st>>>(sg, starts, sorted, heads, slab, lslab, lcount, lcap,
                                                                   ctx->census ? stats : nullptr, dq, dqn, dscr,
                                                                   subheads, subcount, subcap);
    ctx->launches += 1;
    ctx->launches += 1;
  }
  const std::uint64_t want = (n + kBlock - 1) / kBlock;
  const unsigned blocks = static_cast<unsigned>(want < std::uint64_t(sms) * 16 ? want : std::uint64_t(sms) * 16);
  if (blocks > 0) {
    StageTimer t2(ctx, "assign.points");
    SBDT_CUDA_TRY(cudaMemsetAsync(oqc, 0, sizeof(unsigned), st));
    SBDT_CUDA_TRY(cudaMemsetAsync(oqcur, 0, 2 * sizeof(unsigned), st));
    auto overflow = [&]() {
      k_assign_overflow<D><<<sms * 8, 128, 0, st>>>(d_xyz, sg, starts, sorted, slabels, heads, subheads, lslab,
                                                     d_labels, oq, oqc, oqcur, oqcur + 1);
    };
    if (ctx->chunks.empty()) {
      k_assign_vlt<D><<<blocks, kBlock, 0, st>>>(d_xyz, 0, n, sg, heads, subheads, slab, lslab, sorted, slabels, d_labels,
                                                 d_bbox, oq,
                                                 oqc);
    } else {
      // host path: each chunk of points as soon as its upload has landed
      std::uint64_t i0 = 0;
      for (const auto& c : ctx->chunks) {
        const std::uint64_t i1 = c.first < n ? c.first : n;
        SBDT_CUDA_TRY(cudaStreamWaitEvent(st, c.second, 0));
        if (i1 > i0) {
          const std::uint64_t w = (i1 - i0 + kBlock - 1) / kBlock;
          const unsigned b = static_cast<unsigned>(w < std::uint64_t(sms) * 16 ? w : std::uint64_t(sms) * 16);
          k_assign_vlt<D><<<b, kBlock, 0, st>>>(d_xyz, i0, i1, sg, heads, subheads, slab, lslab, sorted, slabels,
                                                d_labels, d_bbox, oq,
                                                oqc);
          ++ctx->launches;
          if (ctx->labels_host) {
            // the chunk's labels are final once its queued points are done:
            // download them while later chunks run
            overflow();
            ++ctx->launches;
            cudaEvent_t ev = ctx->chunk_done[&c - &ctx->chunks[0]];
            SBDT_CUDA_TRY(cudaEventRecord(ev, st));
            SBDT_CUDA_TRY(cudaStreamWaitEvent(ctx->d2h_stream, ev, 0));
            SBDT_CUDA_TRY(cudaMemcpyAsync(ctx->labels_host + i0, d_labels + i0, sizeof(std::uint32_t) * (i1 - i0),
                                          cudaMemcpyDeviceToHost, ctx->d2h_stream));
          }
        }
        i0 = i1;
      }
      --ctx->launches;
    }
    overflow();  // the queued points not yet done (all of them outside the streamed host path)
    ctx->launches += 2;
    if (ctx->census) {  // queued points (long lists + ring searches), dense coarse cells
      SBDT_CUDA_TRY(cudaMemcpyAsync(stats + 4, oqc, sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
      SBDT_CUDA_TRY(cudaMemcpyAsync(stats + 5, dqn, sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
    }
  }
  SBDT_CUDA_TRY(cudaGetLastError());
  return kOk;
}

int bucket_impl(sbdt_gpu_ctx* ctx, const std::uint32_t* d_labels, std::uint64_t n, std::uint32_t k,
                std::uint64_t* d_part_offsets, std::uint32_t* d_part_ids) {
  cudaStream_t st = ctx->stream;
  const std::uint32_t tiles = static_cast<std::uint32_t>((n + kBucketTile - 1) / kBucketTile);
  if (tiles == 0) {
    SBDT_CUDA_TRY(cudaMemsetAsync(d_part_offsets, 0, sizeof(std::uint64_t) * (k + 1), st));
    return kOk;
  }
  StageTimer timer(ctx, "assign.bucket");
  const std::uint64_t cells = std::uint64_t(k) * tiles;
  SBDT_WS(tc, std::uint32_t, "bucket.tc", cells + 1);
  SBDT_WS(bs, std::uint32_t, "bucket.bs", (cells + 1) / kScanTile + 2);
  for (std::uint32_t l0 = 0; l0 < k; l0 += kBucketLabels) {
    const std::uint32_t kl = k - l0 < kBucketLabels ? k - l0 : kBucketLabels;
    k_bucket_count<<<tiles, kBucketThreads, sizeof(std::uint32_t) * kl, st>>>(d_labels, n, l0, kl, tc, tiles);
    ++ctx->launches;
  }
  exclusive_scan(tc, tc, cells, bs, tc + cells, st, &ctx->launches);
  k_part_offsets<<<1, 256, 0, st>>>(tc, k, tiles, n, d_part_offsets, ctx->d_status);
  ++ctx->launches;
  for (std::uint32_t l0 = 0; l0 < k; l0 += kBucketLabels) {
    const std::uint32_t kl = k - l0 < kBucketLabels ? k - l0 : kBucketLabels;
    k_bucket_scatter<<<tiles, kBucketThreads, sizeof(std::uint32_t) * kl * (kBucketThreads / 32), st>>>(
        d_labels, n, l0, kl, tc, tiles, d_part_ids);
    ++ctx->launches;
  }
  SBDT_CUDA_TRY(cudaGetLastError());
  return kOk;
}

// Table statistics of the last timed assign (uniform, list, overflow records).
int assign_stats(sbdt_gpu_ctx* ctx, unsigned* out4) {
  auto it = ctx->bufs.find("assign.stats");
  if (it == ctx->bufs.end()) return kErrInvalid;
  cudaStreamSynchronize(ctx->stream);
  cudaMemcpy(out4, it->second.ptr, sizeof(unsigned) * 6, cudaMemcpyDeviceToHost);
  return kOk;
}

template int assign_impl<2>(sbdt_gpu_ctx*, const double*, std::uint64_t, const std::uint32_t*, const std::uint32_t*,
                            std::uint32_t, std::uint32_t*, unsigned long long*);
template int assign_impl<3>(sbdt_gpu_ctx*, const double*, std::uint64_t, const std::uint32_t*, const std::uint32_t*,
                            std::uint32_t, std::uint32_t*, unsigned long long*);

}  // namespace sbdt_gpu
