// Owner grid (K4): the GridIndex of every partition at once as one uint16 code
// per cell of the global uniform grid — EMPTY, a single owning partition, or
// MULTI — plus a pyramid of coarser levels with the same code per block.
//
// Tiled layout: per-axis fanout F (4 in 3D, 8 in 2D), 64 children per block,
// and the 64 children of a block are CONTIGUOUS (one 128-byte line). Level L
// (below the top) is stored block-major in the tiling of level L+1:
//   index(L, c) = loff[L] + lin(ldims[L+1], c >> sh) * 64 + sub(c & (F-1)).
// Expanding a block is then one coalesced 128-byte load, and the foreign
// children (code not in {EMPTY, self}) come out of per-half-word SIMD
// compares as a 64-bit mask. Padding cells (grid not a multiple of F) are
// EMPTY and are never visited.
//
// Exactness of the descent: a block box is
// the exact union of its cells' boxes (cell_lo is monotone in the index), the
// box_sphere_overlap and halfspace tests are monotone under box containment
// in binary64 / exact arithmetic, and "every sub-box passes" (far corner
// inside the sphere, every corner strictly outside the halfspace) implies the
// leaf test for each occupied leaf below. So the descent answers exactly the
// SPEC's "some occupied leaf cell of another partition passes the test".
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {

template <int D>
struct OwnerGrid {
  Grid<D> g;
  double inv_edge;
  double margin;
  double qh;   // 3-D fixed-point step of the prefilter's packed coordinates (k_owner_mark)
  int levels;  // levels incl. leaf level 0; the top level has exactly one block
  int shift;   // log2 per-axis fanout
  int ldims[kMaxLevels][D];
  unsigned long long loff[kMaxLevels + 1];
  unsigned long long need_cells, need_entries;  // what the bbox needs (read back after a capacity failure)
};

template <int D>
constexpr int og_shift() {
  return D == 3 ? 2 : 3;
}
template <int D>
constexpr int og_fan() {
  return 1 << og_shift<D>();
}

template <int D>
__host__ __device__ __forceinline__ unsigned long long lin_i(const int* dims, const int* c) {
  unsigned long long id = static_cast<unsigned>(c[D - 1]);
#pragma unroll
  for (int d = D - 2; d >= 0; --d) id = id * static_cast<unsigned>(dims[d]) + static_cast<unsigned>(c[d]);
  return id;
}

template <int D>
__device__ __forceinline__ unsigned long long og_index(const OwnerGrid<D>& og, int L, const int* c) {
  if (L == og.levels - 1) return og.loff[L];
  constexpr int sh = og_shift<D>();
  constexpr int F = og_fan<D>();
  int blk[D];
  int sub = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) blk[d] = c[d] >> sh;
  if constexpr (D == 3) sub = (c[0] & (F - 1)) | ((c[1] & (F - 1)) << 2) | ((c[2] & (F - 1)) << 4);
  else sub = (c[0] & (F - 1)) | ((c[1] & (F - 1)) << 3);
  return og.loff[L] + lin_i<D>(og.ldims[L + 1], blk) * 64 + static_cast<unsigned>(sub);
}

// child j (0..63) of block coords b, at the child level
template <int D>
__device__ __forceinline__ void og_child(const int* b, int j, int* c) {
  if constexpr (D == 3) {
    c[0] = (b[0] << 2) | (j & 3);
    c[1] = (b[1] << 2) | ((j >> 2) & 3);
    c[2] = (b[2] << 2) | (j >> 4);
  } else {
    c[0] = (b[0] << 3) | (j & 7);
    c[1] = (b[1] << 3) | (j >> 3);
  }
}

// Grid parameters from the global bbox: edge = c_G (V/n)^(1/D) (SPEC.md:403 /
// build_grid_index post), origin = bbox lo, dims = floor(ext/edge)+1.
template <int D>
__global__ void k_owner_params(const unsigned long long* bbox, std::uint64_t n, double c_G, unsigned long long cap_cells,
                               unsigned long long cap_entries, OwnerGrid<D>* og, unsigned* status) {
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
  for (int d = 0; d < D; ++d) {
    og->g.lo[d] = lo[d];
    const double f = bad ? 0.0 : floor((hi[d] - lo[d]) / e);
    if (!(f < 1.0e9)) bad = true;
    og->g.dims[d] = bad ? 1 : static_cast<long long>(f) + 1;
    cells *= static_cast<unsigned long long>(og->g.dims[d]);
  }
  og->need_cells = bad ? 0ull : cells;
  og->need_entries = 0;
  if (!bad) {  // the tiled layout's entries for these dims (as below)
    int ld[kMaxLevels][D], nl = 0;
    for (;;) {
      bool top = true;
      for (int d = 0; d < D; ++d) {
        ld[nl][d] = static_cast<int>(((og->g.dims[d] - 1) >> (nl * og_shift<D>())) + 1);
        top = top && ld[nl][d] == 1;
      }
      ++nl;
      if (top || nl == kMaxLevels) break;
    }
    unsigned long long ent = 0;
    for (int l = 0; l < nl; ++l) {
      unsigned long long cnt = 64;
      if (l == nl - 1) cnt = 1;
      else
        for (int d = 0; d < D; ++d) cnt *= static_cast<unsigned long long>(ld[l + 1][d]);
      ent += cnt;
    }
    og->need_entries = ent;
  }
  if (bad || cells > cap_cells) {
    atomicOr(status, kStGridCap);
    for (int d = 0; d < D; ++d) og->g.dims[d] = 1;
  }
  og->g.edge = bad ? 1.0 : e;
  og->inv_edge = 1.0 / og->g.edge;
  {
    double span = 0.0;  // the grid covers the bbox: dims * edge >= extent
    for (int d = 0; d < D; ++d) span = fmax(span, static_cast<double>(og->g.dims[d]) * og->g.edge);
    og->qh = span / 2097151.0;  // 21 bits per axis
  }
  og->margin = 1e-9 * (mag + ext_max + og->g.edge);
  constexpr int sh = og_shift<D>();
  og->shift = sh;
  int L = 0;
  for (;;) {
    bool top = true;
    for (int d = 0; d < D; ++d) {
      og->ldims[L][d] = static_cast<int>(((og->g.dims[d] - 1) >> (L * sh)) + 1);
      top = top && og->ldims[L][d] == 1;
    }
    ++L;
    if (top || L == kMaxLevels) break;
  }
  og->levels = L;
  unsigned long long off = 0;
  for (int l = 0; l < L; ++l) {
    og->loff[l] = off;
    unsigned long long cnt = 64;
    if (l == L - 1) cnt = 1;
    else
      for (int d = 0; d < D; ++d) cnt *= static_cast<unsigned long long>(og->ldims[l + 1][d]);
    off += cnt;
  }
  og->loff[L] = off;
  if (off > cap_entries) {
    atomicOr(status, kStGridCap);
    og->levels = 1;  // unusable; the call reports SBDT_ERR_RANGE
    og->loff[1] = 1;
  }
}

// Leaf marking: owner code per occupied cell (CAS on 16-bit words).
template <int D>
__global__ void k_owner_mark(const double* __restrict__ xyz, const std::uint32_t* __restrict__ labels, std::uint64_t n,
                             const OwnerGrid<D>* __restrict__ ogp, std::uint16_t* __restrict__ owner,
                             unsigned long long* __restrict__ pbbox, std::uint32_t k,
                             std::uint64_t* __restrict__ xq = nullptr) {
  __shared__ OwnerGrid<D> og;
  extern __shared__ unsigned long long s_pb[];  // [k][2D] when pbbox != nullptr
  if (threadIdx.x == 0) og = *ogp;
  if (pbbox)
    for (std::uint32_t j = threadIdx.x; j < k * 2 * D; j += blockDim.x)
      s_pb[j] = ((j % (2 * D)) < D) ? 0xFFFFFFFFFFFFFFFFULL : 0ULL;
  __syncthreads();
  // (x - lo) / qh as a product with the rounded reciprocal: a few ulps of
  // 2^21 off the quotient, far inside the 0.5001 qh the prefilter's bound
  // allows for the fixed-point encoding (decode_row)
  const double inv_qh = 1.0 / og.qh;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    double x[D];
    int c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      x[d] = xyz[i * D + d];
      c[d] = static_cast<int>(cell_coord_fast<D>(og.g, og.inv_edge, x[d], d));
    }
    if (xq) {
      // packed prefilter coordinates, indexed by PointId: 3-D 21-bit fixed
      // point of (x - lo) / qh (|error| <= qh / 2), 2-D the binary32 offsets
      // fl(x - lo) (|error| <= u |offset|)
      if constexpr (D == 3) {
        std::uint64_t w = 0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double t = rint((x[d] - og.g.lo[d]) * inv_qh);
          const std::uint64_t q = t <= 0.0 ? 0ull : (t >= 2097151.0 ? 2097151ull : static_cast<std::uint64_t>(t));
          w |= q << (21 * d);
        }
        xq[i] = w;
      } else {
        const float fx = static_cast<float>(x[0] - og.g.lo[0]), fy = static_cast<float>(x[1] - og.g.lo[1]);
        xq[i] = static_cast<std::uint64_t>(__float_as_uint(fx)) | (static_cast<std::uint64_t>(__float_as_uint(fy)) << 32);
      }
    }
    const std::uint32_t lab = labels[i];
    if (lab == SBDT_UNINDEXED) continue;  // not in this level's indices (never a simplex vertex)
    std::uint16_t* slot = owner + og_index<D>(og, 0, c);
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

__device__ __forceinline__ std::uint16_t og_combine(std::uint16_t a, std::uint16_t b) {
  if (a == kOwnerEmpty) return b;
  if (b == kOwnerEmpty) return a;
  return a == b ? a : kOwnerMulti;
}

// Code of block `id` (linear in ldims[L]) at level L >= 1 from its 64
// contiguous children at level L-1.
template <int D>
__device__ __forceinline__ void og_build_block(const OwnerGrid<D>& og, std::uint16_t* owner, int L, unsigned long long id) {
  int c[D];
  unsigned long long rem = id;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    c[d] = static_cast<int>(rem % static_cast<unsigned>(og.ldims[L][d]));
    rem /= static_cast<unsigned>(og.ldims[L][d]);
  }
  const uint4* ch = reinterpret_cast<const uint4*>(owner + og.loff[L - 1] + id * 64);
  std::uint16_t code = kOwnerEmpty;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint4 v = ch[q];
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      code = og_combine(code, static_cast<std::uint16_t>(w[t] & 0xFFFFu));
      code = og_combine(code, static_cast<std::uint16_t>(w[t] >> 16));
    }
  }
  owner[og_index<D>(og, L, c)] = code;
}

template <int D>
__global__ void k_owner_level(const OwnerGrid<D>* __restrict__ ogp, std::uint16_t* __restrict__ owner, int L) {
  __shared__ OwnerGrid<D> og;
  if (threadIdx.x == 0) og = *ogp;
  __syncthreads();
  if (L >= og.levels) return;
  unsigned long long cnt = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) cnt *= static_cast<unsigned>(og.ldims[L][d]);
  for (unsigned long long id = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; id < cnt;
       id += static_cast<unsigned long long>(gridDim.x) * blockDim.x)
    og_build_block<D>(og, owner, L, id);
}

template <int D>
__global__ void k_owner_levels_tail(const OwnerGrid<D>* __restrict__ ogp, std::uint16_t* __restrict__ owner, int L0) {
  __shared__ OwnerGrid<D> og;
  if (threadIdx.x == 0) og = *ogp;
  __syncthreads();
  for (int L = L0; L < og.levels; ++L) {
    unsigned long long cnt = 1;
#pragma unroll
    for (int d = 0; d < D; ++d) cnt *= static_cast<unsigned>(og.ldims[L][d]);
    for (unsigned long long id = threadIdx.x; id < cnt; id += blockDim.x) og_build_block<D>(og, owner, L, id);
    __syncthreads();
  }
}

// packed window word: (min code) << 16 | (0xFFFF - max code), EMPTY counting
// as +inf for the min and 0 for the max; the window combine (EMPTY identity,
// MULTI absorbing) is then a per-half-word min (VIMNMX.U16x2), and the code
// is recovered from (min, max)
__device__ __forceinline__ std::uint32_t nbr_pack(std::uint16_t code) {
  return (static_cast<std::uint32_t>(code) << 16) | (code == kOwnerEmpty ? 0xFFFFu : 0xFFFFu - code);
}
__device__ __forceinline__ std::uint16_t nbr_unpack(std::uint32_t w) {
  const std::uint32_t mn = w >> 16, mx = 0xFFFFu - (w & 0xFFFFu);
  return mn == kOwnerEmpty ? kOwnerEmpty : static_cast<std::uint16_t>(mn == mx ? mn : kOwnerMulti);
}

// ---- window field (grid-policy prefilter) ----------------------------------------
// For every leaf cell c and h = 0..H let W_h(c) be the combined code of the
// (2h+1)^D window of cells centred on c, clipped to the grid (cells outside
// the grid do not exist: EMPTY). The combine is a semilattice (EMPTY
// identity, MULTI absorbing), so W_{h+1} is the 3^D window combine of W_h and
// the box filter is separable (one 1-D pass of half-width 1 per axis).
// One u32 per cell, LINEAR layout (x fastest over ldims[0]):
//   bits 24-31  hs = h* + 1, h* = the largest h <= H with W_h(c) not MULTI
//               (0 when the cell itself is MULTI)
//   bit  16     the cell itself is EMPTY
//   bits 0-15   the cell's code, or W_{h*}(c) when the cell is EMPTY.
// and in the high half of the same u64 the FOREIGN MASK: bit (dx+1) + 3 (dy+1) [+ 9 (dz+1)]
// set iff the neighbour c + (dx, dy[, dz]) is non-empty with a code other
// than the word's code (for a row of that code: the foreign cells of the 3^D
// window; the exact stage's first test, see exact_mask_test).
// The prefilter then needs ONE load per row: a ball whose conservative cell
// range lies in [c - h, c + h] (per axis) with h < hs and code == self
// reaches no foreign occupied cell (every non-empty cell of the window is
// owned by `self`), and a non-empty cell c with another code is foreign.
// A CTA owns a T^D tile (16^3 cells in 3-D, 64^2 in 2-D) and stages it with
// an H-cell halo in shared memory (row pitch RS + 1: the x-lines of the
// in-place passes are bank-conflict free); H rounds of three separable
// passes, one thread per grid line with a sliding window. After round h the
// staged W is exact at least h cells inside the staged region, which covers
// the tile (halo H).
// H = 2 (windows up to 5^D): larger windows decide < 1.5% more rows on the
// BASELINE configs (measured with H = 4) and cost a round of passes each.
template <int D>
constexpr int field_h() {
  return 2;
}
template <int D>
constexpr int field_tile() {
  return D == 3 ? 16 : 64;
}
constexpr std::uint32_t kFieldEmptyBit = 1u << 16;
constexpr int kFieldThreads = 256;

template <int D>
constexpr int field_smem_words() {
  constexpr int RS = field_tile<D>() + 2 * field_h<D>();
  return D == 3 ? (RS + 1) * RS * RS : (RS + 1) * RS;
}
template <int D>
constexpr int field_raw_cells() {
  constexpr int RS = field_tile<D>() + 2 * field_h<D>();
  return D == 3 ? RS * RS * RS : RS * RS;
}
template <int D>
constexpr std::size_t field_smem_bytes() {
  constexpr int T = field_tile<D>();
  return sizeof(std::uint32_t) * (field_smem_words<D>() + (D == 3 ? T * T * T : T * T)) +
         sizeof(std::uint16_t) * field_raw_cells<D>();
}

template <int D>
__global__ void __launch_bounds__(kFieldThreads) k_field_tiles(const OwnerGrid<D>* __restrict__ ogp,
                                                               const std::uint16_t* __restrict__ owner,
                                                               std::uint64_t* __restrict__ field) {
  constexpr int F = og_fan<D>();
  constexpr int SH = og_shift<D>();
  constexpr int H = field_h<D>();
  constexpr int T = field_tile<D>();
  constexpr int RS = T + 2 * H;               // staged cells per axis
  constexpr int P = RS + 1;                   // x pitch
  constexpr int RN = D == 3 ? RS * RS * RS : RS * RS;
  constexpr int LN = D == 3 ? RS * RS : RS;   // lines per pass
  constexpr int ON = D == 3 ? T * T * T : T * T;
  __shared__ OwnerGrid<D> og;
  extern __shared__ std::uint32_t fsm[];
  std::uint32_t* buf = fsm;                          // packed window words (nbr_pack)
  std::uint32_t* outw = fsm + field_smem_words<D>();  // the tile's field words
  // the staged leaf codes, unchanged by the passes (foreign masks), x fastest
  std::uint16_t* raw = reinterpret_cast<std::uint16_t*>(outw + ON);
  if (threadIdx.x == 0) og = *ogp;
  __syncthreads();
  int nt[D], cd0[D];
  unsigned long long ntiles = 1;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    cd0[d] = og.ldims[0][d];
    nt[d] = (cd0[d] + T - 1) / T;
    ntiles *= static_cast<unsigned long long>(nt[d]);
  }
  const std::uint16_t* own0 = owner + og.loff[0];
  const bool single = og.levels < 2;  // one cell: no tiled level-0 layout
  auto gindex = [&](const int* c) -> unsigned long long {  // level-0 tiled index
    if (single) return 0ull;
    unsigned b = static_cast<unsigned>(c[D - 1] >> SH), sub = 0;
#pragma unroll
    for (int d = D - 2; d >= 0; --d) b = b * static_cast<unsigned>(og.ldims[1][d]) + static_cast<unsigned>(c[d] >> SH);
#pragma unroll
    for (int d = 0; d < D; ++d) sub |= static_cast<unsigned>(c[d] & (F - 1)) << (SH * d);
    return static_cast<unsigned long long>(b) * 64u + sub;
  };
  auto sidx = [](const int* t) {  // staged coordinates -> buffer word
    return D == 3 ? t[0] + P * (t[1] + RS * t[2]) : t[0] + P * t[1];
  };
  for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int org[D];
    unsigned long long rem = tile;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      org[d] = static_cast<int>(rem % static_cast<unsigned>(nt[d])) * T;
      rem /= static_cast<unsigned>(nt[d]);
    }
    for (int r = threadIdx.x; r < RN; r += blockDim.x) {
      int c[D], t[D], rr = r;
      bool in = true;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        t[d] = rr % RS;
        rr /= RS;
        c[d] = org[d] - H + t[d];
        in = in && c[d] >= 0 && c[d] < cd0[d];
      }
      const std::uint16_t code = in ? own0[gindex(c)] : kOwnerEmpty;
      buf[sidx(t)] = nbr_pack(code);
      raw[r] = code;
    }
    __syncthreads();
    // h = 0: the cell's own code
    for (int o = threadIdx.x; o < ON; o += blockDim.x) {
      int t[D], oo = o;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        t[d] = oo % T + H;
        oo /= T;
      }
      const std::uint16_t code = nbr_unpack(buf[sidx(t)]);
      outw[o] = code == kOwnerMulti ? static_cast<std::uint32_t>(kOwnerMulti)
                                    : ((1u << 24) | (code == kOwnerEmpty ? kFieldEmptyBit : 0u) | code);
    }
    __syncthreads();  // the passes below overwrite buf in place
    for (int h = 1; h <= H; ++h) {
#pragma unroll
      for (int ax = 0; ax < D; ++ax) {
        const int st = ax == 0 ? 1 : (ax == 1 ? P : P * RS);
        for (int l = threadIdx.x; l < LN; l += blockDim.x) {
          int base;
          if constexpr (D == 3) {
            const int u = l % RS, w = l / RS;
            base = ax == 0 ? (u * P + w * P * RS) : (ax == 1 ? (u + w * P * RS) : (u + w * P));
          } else {
            base = ax == 0 ? l * P : l;
          }
          // in place: a line belongs to one thread, the registers hold the
          // original values of the cells already overwritten; the end cells
          // combine their in-range neighbours only (never read: see above)
          std::uint32_t prev = buf[base], cur = buf[base + st];
          buf[base] = __vminu2(prev, cur);
#pragma unroll 4
          for (int i = 1; i < RS - 1; ++i) {
            const std::uint32_t next = buf[base + (i + 1) * st];
            buf[base + i * st] = __vminu2(__vminu2(prev, cur), next);
            prev = cur;
            cur = next;
          }
          buf[base + (RS - 1) * st] = __vminu2(prev, cur);
        }
        __syncthreads();
      }
      for (int o = threadIdx.x; o < ON; o += blockDim.x) {
        const std::uint32_t w0 = outw[o];
        if ((w0 >> 24) != static_cast<unsigned>(h)) continue;  // stopped growing earlier
        int t[D], oo = o;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          t[d] = oo % T + H;
          oo /= T;
        }
        const std::uint16_t code = nbr_unpack(buf[sidx(t)]);
        if (code == kOwnerMulti) continue;
        const std::uint32_t lo = (w0 & kFieldEmptyBit) ? (kFieldEmptyBit | code) : (w0 & 0xFFFFFu);
        outw[o] = (static_cast<std::uint32_t>(h + 1) << 24) | lo;
      }
      __syncthreads();  // read before the next round's passes overwrite buf
    }
    __syncthreads();
    // linear layout, x fastest: consecutive threads store consecutive cells
    for (int o = threadIdx.x; o < ON; o += blockDim.x) {
      int c[D], oo = o;
      bool in = true;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        c[d] = org[d] + oo % T;
        oo /= T;
        in = in && c[d] < cd0[d];
      }
      if (in) {
        unsigned long long li = static_cast<unsigned>(c[D - 1]);
#pragma unroll
        for (int d = D - 2; d >= 0; --d) li = li * static_cast<unsigned>(cd0[d]) + static_cast<unsigned>(c[d]);
        const std::uint32_t w = outw[o];
        const std::uint16_t own = static_cast<std::uint16_t>(w & 0xFFFFu);
        int t[D], oo2 = o;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          t[d] = oo2 % T + H;
          oo2 /= T;
        }
        // hs >= 2: the 3^D window holds at most one code (the word's), so no
        // neighbour is foreign to it
        std::uint32_t m = 0;
        if ((w >> 24) >= 2u) {
        } else if constexpr (D == 3) {
#pragma unroll
          for (int j = 0; j < 27; ++j) {
            const std::uint16_t nc = raw[(t[0] + j % 3 - 1) + RS * ((t[1] + (j / 3) % 3 - 1) + RS * (t[2] + j / 9 - 1))];
            m |= (nc != kOwnerEmpty && nc != own) ? (1u << j) : 0u;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 9; ++j) {
            const std::uint16_t nc = raw[(t[0] + j % 3 - 1) + RS * (t[1] + j / 3 - 1)];
            m |= (nc != kOwnerEmpty && nc != own) ? (1u << j) : 0u;
          }
        }
        field[li] = static_cast<std::uint64_t>(m) << 32 | w;
      }
    }
    __syncthreads();  // the buffers are reloaded for the next tile
  }
}

// bbox policy with more partitions than k_owner_mark stages in shared
// memory: the partition bboxes by global atomics (ordered keys).
constexpr std::uint32_t kPbboxSmem = 3072;  // [k][2D] words k_owner_mark stages in shared memory (24 KB)

template <int D>
__global__ void k_pbbox_global(const double* __restrict__ xyz, const std::uint32_t* __restrict__ labels,
                               std::uint64_t n, unsigned long long* __restrict__ pbbox) {
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint32_t lab = labels[i];
    if (lab == SBDT_UNINDEXED) continue;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const unsigned long long o = dbl_to_ordered(xyz[i * D + d]);
      atomicMin(&pbbox[lab * 2 * D + d], o);
      atomicMax(&pbbox[lab * 2 * D + D + d], o);
    }
  }
}

// EMPTY over the entries the grid actually uses (loff[levels], known only on
// the device) instead of the worst-case capacity.
template <int D>
__global__ void k_owner_clear(const OwnerGrid<D>* __restrict__ ogp, std::uint16_t* __restrict__ owner) {
  const unsigned long long len = ogp->loff[ogp->levels];
  unsigned long long i = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 8ull;
  const unsigned long long step = static_cast<unsigned long long>(gridDim.x) * blockDim.x * 8ull;
  for (; i < len; i += step) {
    if (i + 8 <= len) {
      *reinterpret_cast<uint4*>(owner + i) = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    } else {
      for (unsigned long long j = i; j < len; ++j) owner[j] = kOwnerEmpty;
    }
  }
}

// ---- queries ----------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void og_block_box(const OwnerGrid<D>& og, int L, const int* c, double* blo, double* bhi) {
  const int s = L * og_shift<D>();
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (og.ldims[0][d] <= (1 << 26)) {  // ((c + 1) << s stays below 2^30 at every level)
      // 32-bit cell indices (the conversion to binary64 is exact either way:
      // the same values as the 64-bit path, one I2F instead of a sequence)
      const int first = c[d] << s;
      const int last1 = min((c[d] + 1) << s, og.ldims[0][d]);
      blo[d] = og.g.lo[d] + static_cast<double>(first) * og.g.edge;
      bhi[d] = og.g.lo[d] + static_cast<double>(last1) * og.g.edge;
    } else {
      const long long first = static_cast<long long>(c[d]) << s;
      long long last1 = static_cast<long long>(c[d] + 1) << s;
      if (last1 > og.g.dims[d]) last1 = og.g.dims[d];
      blo[d] = cell_lo<D>(og.g, first, d);
      bhi[d] = cell_lo<D>(og.g, last1, d);
    }
  }
}

// 64-bit mask of the children of block b (level L >= 1) whose code is
// foreign (not EMPTY, not self) and whose coordinates lie in [ra, rb]
// (child-level range) — one 128-byte load.
template <int D>
__device__ __forceinline__ unsigned long long og_child_mask(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner,
                                                            int L, const int* b, std::uint32_t self, const int* ra,
                                                            const int* rb) {
  const uint4* ch = reinterpret_cast<const uint4*>(owner + og.loff[L - 1] + lin_i<D>(og.ldims[L], b) * 64);
  const unsigned selfx2 = (self & 0xFFFFu) | (self << 16);
  unsigned long long m = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint4 v = __ldg(ch + q);
    const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const unsigned f = __vcmpne2(w[t], 0xFFFFFFFFu) & __vcmpne2(w[t], selfx2);
      const unsigned long long bits = (f & 1u) | ((f >> 15) & 2u);
      m |= bits << (2 * (4 * q + t));
    }
  }
  // range restriction
  constexpr int F = og_fan<D>();
  unsigned long long rm = 0;
  int lo[D], hi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    lo[d] = max(ra[d] - b[d] * F, 0);
    hi[d] = min(rb[d] - b[d] * F, F - 1);
    if (lo[d] > hi[d]) return 0;
  }
  if constexpr (D == 3) {
    const unsigned long long row = ((1ULL << (hi[0] - lo[0] + 1)) - 1) << lo[0];
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y) rm |= row << (4 * y + 16 * z);
  } else {
    const unsigned long long row = ((1ULL << (hi[0] - lo[0] + 1)) - 1) << lo[0];
    for (int y = lo[1]; y <= hi[1]; ++y) rm |= row << (8 * y);
  }
  return m & rm;
}

// Depth-first descent. Start blocks: the blocks of level L0 covering the leaf
// range [a, b] (at most two per axis). test(blo, bhi, level, block) returns
// 0 reject, 1 descend, 2 accept (every sub-box passes). A passing leaf is a
// hit.
template <int D, class Test>
__device__ bool og_descend(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner, std::uint32_t self, int L0,
                           const int* a, const int* b, const Test& test, unsigned long long* stats = nullptr) {
  unsigned n_tests = 0, n_masks = 0;
  struct Flush {
    unsigned long long* st;
    unsigned& t;
    unsigned& m;
    int L;
    __device__ ~Flush() {
      if (st) {
        atomicAdd(&st[2], static_cast<unsigned long long>(t));
        atomicAdd(&st[3], static_cast<unsigned long long>(m));
        atomicAdd(&st[4 + (L > 3 ? 3 : L)], 1ULL);
      }
    }
  } flush{stats, n_tests, n_masks, L0};
  struct Frame {
    unsigned long long mask;
    int c[D];
    int level;
  };
  Frame fr[kMaxLevels];  // depth <= levels - 1
  int s0[D], n0[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    s0[d] = a[d] >> (L0 * og.shift);
    n0[d] = (b[d] >> (L0 * og.shift)) - s0[d] + 1;
  }
  const int total = D == 3 ? n0[0] * n0[1] * n0[2] : n0[0] * n0[1];
  for (int t = 0; t < total; ++t) {
    int cc[D], rem = t;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      cc[d] = s0[d] + rem % n0[d];
      rem /= n0[d];
    }
    const std::uint16_t code = owner[og_index<D>(og, L0, cc)];
    if (code == kOwnerEmpty || code == self) continue;
    double blo[D], bhi[D];
    og_block_box<D>(og, L0, cc, blo, bhi);
    ++n_tests;
    const int r = test(blo, bhi, L0, cc);
    if (r == 0) continue;
    if (L0 == 0 || r == 2) return true;
    // explore this start block
    int depth = 0;
    {
      const int cl = L0 - 1, csh = cl * og.shift;
      int ra[D], rb[D];
#pragma unroll
      for (int d = 0; d < D; ++d) ra[d] = a[d] >> csh, rb[d] = b[d] >> csh;
      ++n_masks;
      fr[0].mask = og_child_mask<D>(og, owner, L0, cc, self, ra, rb);
#pragma unroll
      for (int d = 0; d < D; ++d) fr[0].c[d] = cc[d];
      fr[0].level = L0;
      depth = 1;
    }
    while (depth > 0) {
      Frame& f = fr[depth - 1];
      if (f.mask == 0) {
        --depth;
        continue;
      }
      const int j = __ffsll(static_cast<long long>(f.mask)) - 1;
      f.mask &= f.mask - 1;
      const int lv = f.level - 1;
      int ch[D];
      og_child<D>(f.c, j, ch);
      double blo[D], bhi[D];
      og_block_box<D>(og, lv, ch, blo, bhi);
      ++n_tests;
      const int r2 = test(blo, bhi, lv, ch);
      if (r2 == 0) continue;
      if (lv == 0 || r2 == 2) return true;
      const int cl = lv - 1, csh = cl * og.shift;
      int ra[D], rb[D];
#pragma unroll
      for (int d = 0; d < D; ++d) ra[d] = a[d] >> csh, rb[d] = b[d] >> csh;
      Frame& g2 = fr[depth];
      ++n_masks;
      g2.mask = og_child_mask<D>(og, owner, lv, ch, self, ra, rb);
#pragma unroll
      for (int d = 0; d < D; ++d) g2.c[d] = ch[d];
      g2.level = lv;
      if (g2.mask) ++depth;
    }
  }
  return false;
}

// true iff some cell with owner code not in {EMPTY, self} overlaps the sphere
// (box_sphere_overlap, geometry.hpp:187-201).
template <int D>
__device__ __forceinline__ bool og_sphere_hits_foreign(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner,
                                                       const double* c, double r2, std::uint32_t self,
                                                       unsigned long long* stats = nullptr) {
  if (isnan(r2)) return false;
  bool fin = isfinite(r2);
#pragma unroll
  for (int d = 0; d < D; ++d) fin = fin && isfinite(c[d]);
  int a[D], b[D];
  if (fin) {
    // Conservative leaf range; the margin (1e-9 relative) dominates the
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
  return og_descend<D>(og, owner, self, L, a, b, [&](const double* blo, const double* bhi, int, const int*) {
    if (!box_sphere<D>(blo, bhi, c, r2)) return 0;
    return box_inside_sphere<D>(blo, bhi, c, r2) ? 2 : 1;
  }, stats);
}

// Halfspace variant (halfspace_box_overlap, geometry.cpp:329-345): test = some
// box corner strictly on the outer side of the hull facet plane (exact
// orient), accept = every corner strictly outside.
template <int D>
__device__ int corners_outside(const double* const* facet, int inner_sign, const double* blo, const double* bhi,
                               unsigned long long* escalations = nullptr) {
  const double* pts[D + 1];
#pragma unroll
  for (int i = 0; i < D; ++i) pts[i] = facet[i];
  double corner[D];
  pts[D] = corner;
  int outside = 0;
  for (unsigned cm = 0; cm < (1u << D); ++cm) {
#pragma unroll
    for (int d = 0; d < D; ++d) corner[d] = (cm & (1u << d)) ? bhi[d] : blo[d];
    const int s = orient_dev<D>(pts, escalations);
    if (s != 0 && s != inner_sign) ++outside;
  }
  return outside;
}

template <int D>
__device__ bool og_halfspace_hits_foreign(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner,
                                          const double* const* facet, int inner_sign, std::uint32_t self) {
  int a[D], b[D];
#pragma unroll
  for (int d = 0; d < D; ++d) a[d] = 0, b[d] = og.ldims[0][d] - 1;
  return og_descend<D>(og, owner, self, og.levels - 1, a, b, [&](const double* blo, const double* bhi, int, const int*) {
    const int out = corners_outside<D>(facet, inner_sign, blo, bhi);
    if (out == 0) return 0;
    return out == (1 << D) ? 2 : 1;
  });
}

// ---- exact policy: the points of the candidate cells ------
// Per-cell point lists over the level-0 tiled index (built by k_cell_count /
// k_cell_scatter): start[idx] .. start[idx+1] in pts.
template <int D>
struct CellPt {
  double x[D];
  std::uint32_t label;
  std::uint32_t pid;
};

template <int D>
struct CellPoints {
  const std::uint32_t* start;
  const CellPt<D>* pts;
};

// Serial exact-policy descents (fallbacks of the warp-cooperative ones): a
// leaf passes only if leaf(cell) finds a qualifying point; no block is
// accepted wholesale for spheres (the points must be strictly inside the
// exact circumsphere, not the inflated one), whereas a block entirely in the
// open outer halfspace of a hull facet holds only strictly-outside points.
template <int D, class Leaf>
__device__ bool og_sphere_exact_serial(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner, const double* c,
                                       double r2, std::uint32_t self, const Leaf& leaf) {
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
  int L = 0;
  for (; L < og.levels - 1; ++L) {
    bool ok = true;
#pragma unroll
    for (int d = 0; d < D; ++d) ok = ok && ((b[d] >> (L * og.shift)) - (a[d] >> (L * og.shift)) <= 1);
    if (ok) break;
  }
  return og_descend<D>(og, owner, self, L, a, b, [&](const double* blo, const double* bhi, int lv, const int* cell) {
    if (!box_sphere<D>(blo, bhi, c, r2)) return 0;
    if (lv > 0) return 1;
    return leaf(cell) ? 2 : 0;
  });
}

template <int D, class Leaf>
__device__ bool og_halfspace_exact_serial(const OwnerGrid<D>& og, const std::uint16_t* __restrict__ owner,
                                          const double* const* facet, int inner_sign, std::uint32_t self,
                                          const Leaf& leaf) {
  int a[D], b[D];
#pragma unroll
  for (int d = 0; d < D; ++d) a[d] = 0, b[d] = og.ldims[0][d] - 1;
  return og_descend<D>(og, owner, self, og.levels - 1, a, b,
                       [&](const double* blo, const double* bhi, int lv, const int* cell) {
                         const int out = corners_outside<D>(facet, inner_sign, blo, bhi);
                         if (out == 0) return 0;
                         if (out == (1 << D)) return 2;
                         if (lv > 0) return 1;
                         return leaf(cell) ? 2 : 0;
                       });
}

}  // namespace sbdt_gpu
