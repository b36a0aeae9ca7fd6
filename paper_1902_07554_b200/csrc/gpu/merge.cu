// K10-K13: dc-engine `merge` + `update_neighbors` (PAPER.md
// Alg. 1 merging and neighbourhood blocks) — the step after the border
// triangulation, as one data-parallel pass over the partial rows and one over
// the rows of T_B.
//
//   K10 k_merge_keep      partial row kept <=> finite and not in B (SPEC: "(U
//                         partials) minus border simplices"; infinite rows are
//                         stripped); ballot -> keep bit per row,
//                         popcount per 32-row word; border-tuple count.
//       k_merge_bset      the finite rows of B into an open-addressing set keyed
//                         on facet_key of all D+1 ids.
//   K11 k_merge_include   T_B row included <=> finite and (its vertices span >= 2
//                         partitions, or its tuple is in the set of B).
//       exclusive scan over the words of both bitmaps: output row of a kept /
//       included row = word base + popcount of the lower bits (deterministic
//       order: kept partial rows, then inserted T_B rows, each in row order).
//   K12 k_merge_emit_*    write the row; a facet whose old neighbour survives
//                         is relinked through the same bitmap (part-local ->
//                         output id); every other facet (neighbour dropped or
//                         infinite) goes into a facet-hash join keyed on the
//                         reference's facet_key (triangulation.hpp:73-94,
//                         candidates verified by their vertex ids): the second
//                         owner of a facet links both sides; a third owner is
//                         InconsistentMerge. This is update_neighbors' result
//                         (unique neighbour structure) without its queue.
//   K13 k_merge_hull_*    optional: the merged hull re-derived from the facets
//                         left with a single finite owner: one
//                         infinite row per such facet at a scanned position
//                         ((owner row, facet) order), linked to its owner and,
//                         by a second join over the hull ridges, to its
//                         neighbouring infinite rows. A ridge without exactly
//                         two hull facets is DanglingFacet.
//
// The join tables are 64-bit slots (32-bit key tag | 31-bit facet handle | paired
// bit) probed linearly with atomicCAS; the emitting thread publishes its row's
// vertex ids (__threadfence) before inserting, and probers read them with
// L2-coherent loads.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "context.cuh"
#include "scan.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {

enum MergeStatusBits : unsigned { kStMergeInconsistent = 8u, kStMergeDangling = 16u };

namespace {

constexpr std::uint32_t kNoneId = 0xFFFFFFFFu;
constexpr unsigned long long kSlotEmpty = ~0ull;
constexpr std::uint32_t kPairedBit = 0x80000000u;
constexpr int kMergeThreads = 256;

// splitmix64 finalizer (common.hpp:69-74) and facet_key (triangulation.hpp:68-94).
__device__ __forceinline__ unsigned long long mix64_dev(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
template <int N>
__device__ __forceinline__ unsigned long long key_of(const std::uint32_t* ids) {
  unsigned long long sum = 0, xr = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const unsigned long long m = mix64_dev(ids[i]);
    sum += m;
    xr ^= m;
  }
  return sum ^ (xr << 32 | xr >> 32);
}

struct MergeDev {
  std::uint32_t k;
  const std::uint32_t* labels;
  const std::uint64_t* offsets;
  const std::uint32_t* verts;
  const std::uint32_t* nbrs;
  const std::int8_t* parity;
  const std::uint8_t* border;
  std::uint64_t S;
  const std::uint32_t* tb_verts;
  const std::uint32_t* tb_nbrs;
  const std::int8_t* tb_parity;
  std::uint64_t SB;
  std::uint64_t WS;          // words of the partial bitmap (the T_B bitmap follows)
  std::uint32_t* mask;       // WS + WB keep / include bits
  std::uint32_t* base;       // WS + WB + 1: exclusive scan of the word popcounts
  unsigned long long* bset;  // border tuple set
  unsigned long long bset_mask;
  unsigned long long* join;  // facet join table
  unsigned long long join_mask;
  std::uint32_t* out_verts;
  std::uint32_t* out_nbrs;
  std::int8_t* out_parity;
  std::uint64_t ostride;
  unsigned* status;
  unsigned long long* counters;  // [0] finite border rows
};

__device__ __forceinline__ std::uint32_t out_index(const MergeDev& a, std::uint64_t word, unsigned bit) {
  return a.base[word] + __popc(a.mask[word] & ((1u << bit) - 1u));
}
__device__ __forceinline__ bool bit_set(const MergeDev& a, std::uint64_t word, unsigned bit) {
  return (a.mask[word] >> bit) & 1u;
}

// K10 ------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_keep(MergeDev a) {
  __shared__ unsigned block_count;
  if (threadIdx.x == 0) block_count = 0;
  __syncthreads();
  const std::uint64_t s = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool keep = false, bord = false;
  if (s < a.S) {
    const bool finite = a.verts[std::uint64_t(D) * a.S + s] != kInfVertex;
    const bool b = a.border[s] != 0;
    keep = finite && !b;
    bord = finite && b;
  }
  const unsigned km = __ballot_sync(0xffffffffu, keep);
  const unsigned bm = __ballot_sync(0xffffffffu, bord);
  if (lane_id() == 0) {
    const std::uint64_t w = s >> 5;
    if (w < a.WS) {
      a.mask[w] = km;
      a.base[w] = __popc(km);
    }
    if (bm) atomicAdd(&block_count, unsigned(__popc(bm)));
  }
  __syncthreads();
  if (threadIdx.x == 0 && block_count) atomicAdd(&a.counters[0], static_cast<unsigned long long>(block_count));
}

template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_bset(MergeDev a) {
  const std::uint64_t s = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= a.S || !a.border[s]) return;
  std::uint32_t v[D + 1];
#pragma unroll
  for (int j = 0; j <= D; ++j) v[j] = a.verts[std::uint64_t(j) * a.S + s];
  if (v[D] == kInfVertex) return;
  const unsigned long long key = key_of<D + 1>(v);
  const unsigned long long mine = ((key >> 32) << 32) | static_cast<std::uint32_t>(s);
  for (unsigned long long slot = key & a.bset_mask;; slot = (slot + 1) & a.bset_mask)
    if (atomicCAS(&a.bset[slot], kSlotEmpty, mine) == kSlotEmpty) return;
}

template <int D>
__device__ bool in_border_set(const MergeDev& a, const std::uint32_t* v) {
  const unsigned long long key = key_of<D + 1>(v);
  const std::uint32_t tag = static_cast<std::uint32_t>(key >> 32);
  for (unsigned long long slot = key & a.bset_mask;; slot = (slot + 1) & a.bset_mask) {
    const unsigned long long e = a.bset[slot];
    if (e == kSlotEmpty) return false;
    if (static_cast<std::uint32_t>(e >> 32) != tag) continue;
    const std::uint64_t s = static_cast<std::uint32_t>(e);
    bool eq = true;
#pragma unroll
    for (int j = 0; j <= D; ++j) eq &= a.verts[std::uint64_t(j) * a.S + s] == v[j];
    if (eq) return true;
  }
}

// K11 ------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_include(MergeDev a) {
  const std::uint64_t t = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool inc = false;
  if (t < a.SB) {
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = a.tb_verts[std::uint64_t(j) * a.SB + t];
    if (v[D] != kInfVertex) {
      const std::uint32_t l0 = a.labels[v[0]];
      bool spans = false;
#pragma unroll
      for (int j = 1; j <= D; ++j) spans |= a.labels[v[j]] != l0;
      inc = spans || (a.bset_mask != 0 && in_border_set<D>(a, v));
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, inc);
  if (lane_id() == 0) {
    const std::uint64_t w = a.WS + (t >> 5);
    if ((t >> 5) < (a.SB + 31) / 32) {
      a.mask[w] = m;
      a.base[w] = __popc(m);
    }
  }
}

// Output row ids of the partition starts (K12 needs them too, via offsets).
__global__ void k_merge_offsets(MergeDev a, std::uint64_t* out_offsets) {
  const std::uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > a.k) return;
  const std::uint64_t s = a.offsets[p];
  out_offsets[p] = (s >> 5) < a.WS ? out_index(a, s >> 5, unsigned(s & 31)) : a.base[a.WS];
}

// The facet-hash join. `val` = row * (D+1) + facet; `eq(other_val)` compares
// the other owner's facet with ours. Returns the partner's handle or kNoneId.
template <typename Eq>
__device__ std::uint32_t join_insert(unsigned long long* tab, unsigned long long mask, unsigned long long key,
                                     std::uint32_t val, unsigned* status, Eq eq) {
  const unsigned long long tag = key >> 32;
  const unsigned long long mine = (tag << 32) | val;
  for (unsigned long long slot = key & mask;; slot = (slot + 1) & mask) {
    const unsigned long long old = atomicCAS(&tab[slot], kSlotEmpty, mine);
    if (old == kSlotEmpty) return kNoneId;
    if ((old >> 32) != tag) continue;
    const std::uint32_t ov = static_cast<std::uint32_t>(old);
    if (!eq(ov & ~kPairedBit)) continue;
    if (!(ov & kPairedBit) && atomicCAS(&tab[slot], old, old | kPairedBit) == old) return ov;
    atomicOr(status, kStMergeInconsistent);  // third owner of one facet
    return kNoneId;
  }
}

template <int D>
__device__ __forceinline__ void emit_row(const MergeDev& a, std::uint32_t o, const std::uint32_t* v,
                                         std::int8_t par) {
#pragma unroll
  for (int j = 0; j <= D; ++j) a.out_verts[std::uint64_t(j) * a.ostride + o] = v[j];
  a.out_parity[o] = par;
}

// Join the facet opposite verts[d] of output row o (rows are published: the
// join runs in a later launch than the emission).
template <int D>
__device__ __forceinline__ void join_facet(const MergeDev& a, std::uint32_t o, int d) {
  std::uint32_t f[D];
#pragma unroll
  for (int j = 0, q = 0; j <= D; ++j)
    if (j != d) f[q++] = __ldg(a.out_verts + std::uint64_t(j) * a.ostride + o);
  const std::uint32_t partner = join_insert(
      a.join, a.join_mask, key_of<D>(f), o * (D + 1) + d, a.status, [&](std::uint32_t ov) {
        const std::uint32_t po = ov / (D + 1), pd = ov % (D + 1);
        bool eq = true;
#pragma unroll
        for (int j = 0, q = 0; j <= D; ++j)
          if (j != static_cast<int>(pd)) eq &= __ldg(a.out_verts + std::uint64_t(j) * a.ostride + po) == f[q++];
        return eq;
      });
  if (partner != kNoneId) {
    const std::uint32_t po = partner / (D + 1), pd = partner % (D + 1);
    a.out_nbrs[std::uint64_t(d) * a.ostride + o] = po;
    a.out_nbrs[std::uint64_t(pd) * a.ostride + po] = o;
  }
}

// Warp-aggregated append of the facet handles in `bits` (row o) to a queue.
// Every lane of the warp must call it.
template <int D>
__device__ __forceinline__ void queue_facets(unsigned* count, std::uint32_t* q, std::uint64_t cap, unsigned* status,
                                             std::uint32_t o, unsigned bits) {
  const unsigned lane = lane_id();
  const unsigned c = __popc(bits);
  unsigned incl = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= static_cast<unsigned>(off)) incl += y;
  }
  const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
  if (!total) return;
  unsigned base = 0;
  if (lane == 31) base = atomicAdd(count, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  std::uint64_t pos = std::uint64_t(base) + incl - c;
  while (bits) {
    const int d = __ffs(bits) - 1;
    bits &= bits - 1;
    if (pos < cap) q[pos] = o * (D + 1) + d;
    else atomicOr(status, kStQueueOverflow);
    ++pos;
  }
}

// K12 ------------------------------------------------------------------------
// Emission: the row, its surviving links (relinked through the bitmaps) and
// kNone + a queue entry for every other facet. Whole warps stay resident for
// the queue append.
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_emit_partial(MergeDev a, unsigned* qcount,
                                                                      std::uint32_t* queue, std::uint64_t qcap) {
  const std::uint64_t s = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = s < a.S && bit_set(a, s >> 5, unsigned(s & 31));
  std::uint32_t o = 0;
  unsigned jb = 0;
  if (live) {
    o = out_index(a, s >> 5, unsigned(s & 31));
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = a.verts[std::uint64_t(j) * a.S + s];
    emit_row<D>(a, o, v, a.parity[s]);
    // part of row s: the last p with offsets[p] <= s
    std::uint32_t lo = 0, hi = a.k;
    while (hi - lo > 1) {
      const std::uint32_t mid = (lo + hi) >> 1;
      if (__ldg(a.offsets + mid) <= s) lo = mid;
      else hi = mid;
    }
    const std::uint64_t first = __ldg(a.offsets + lo);
#pragma unroll
    for (int d = 0; d <= D; ++d) {
      const std::uint32_t nb = a.nbrs[std::uint64_t(d) * a.S + s];
      std::uint32_t link = kNoneId;
      if (nb != kNoneId) {
        const std::uint64_t g = first + nb;
        if (g < a.S && bit_set(a, g >> 5, unsigned(g & 31))) link = out_index(a, g >> 5, unsigned(g & 31));
      }
      a.out_nbrs[std::uint64_t(d) * a.ostride + o] = link;
      if (link == kNoneId) jb |= 1u << d;
    }
  }
  queue_facets<D>(qcount, queue, qcap, a.status, o, jb);
}

template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_emit_tb(MergeDev a, unsigned* qcount, std::uint32_t* queue,
                                                                 std::uint64_t qcap) {
  const std::uint64_t t = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = t < a.SB && bit_set(a, a.WS + (t >> 5), unsigned(t & 31));
  std::uint32_t o = 0;
  unsigned jb = 0;
  if (live) {
    o = out_index(a, a.WS + (t >> 5), unsigned(t & 31));
    std::uint32_t v[D + 1];
#pragma unroll
    for (int j = 0; j <= D; ++j) v[j] = a.tb_verts[std::uint64_t(j) * a.SB + t];
    emit_row<D>(a, o, v, a.tb_parity[t]);
#pragma unroll
    for (int d = 0; d <= D; ++d) {
      const std::uint32_t nb = a.tb_nbrs[std::uint64_t(d) * a.SB + t];
      std::uint32_t link = kNoneId;
      if (nb != kNoneId && nb < a.SB && bit_set(a, a.WS + (nb >> 5), nb & 31u))
        link = out_index(a, a.WS + (nb >> 5), nb & 31u);
      a.out_nbrs[std::uint64_t(d) * a.ostride + o] = link;
      if (link == kNoneId) jb |= 1u << d;
    }
  }
  queue_facets<D>(qcount, queue, qcap, a.status, o, jb);
}

// The facet join over the queued facets (update_neighbors).
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_join(MergeDev a, const std::uint32_t* queue,
                                                              std::uint32_t J) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= J) return;
  const std::uint32_t h = queue[i];
  join_facet<D>(a, h / (D + 1), static_cast<int>(h % (D + 1)));
}

// K13 ------------------------------------------------------------------------
// Hull facets = queued facets left without a partner.
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_hull_collect(MergeDev a, const std::uint32_t* queue,
                                                                      std::uint32_t J, unsigned* hcount,
                                                                      std::uint32_t* hull, std::uint64_t hcap) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bit = 0;
  std::uint32_t h = 0;
  if (i < J) {
    h = queue[i];
    bit = a.out_nbrs[std::uint64_t(h % (D + 1)) * a.ostride + h / (D + 1)] == kNoneId;
  }
  // one handle per lane: reuse the facet-queue append with row = h / (D+1)
  queue_facets<D>(hcount, hull, hcap, a.status, h / (D + 1), bit << (h % (D + 1)));
}

// Single-CTA bitonic sort of up to kHullSortMax handles (ascending = (owner
// row, facet) order).
constexpr int kHullSortMax = 16384;
constexpr int kSortThreads = 1024;
__global__ void __launch_bounds__(kSortThreads) k_sort_small(std::uint32_t* data, std::uint32_t n) {
  extern __shared__ std::uint32_t sm[];
  std::uint32_t len = 2;
  while (len < n) len <<= 1;
  for (std::uint32_t i = threadIdx.x; i < len; i += kSortThreads) sm[i] = i < n ? data[i] : 0xFFFFFFFFu;
  __syncthreads();
  for (std::uint32_t k2 = 2; k2 <= len; k2 <<= 1) {
    for (std::uint32_t j = k2 >> 1; j > 0; j >>= 1) {
      for (std::uint32_t i = threadIdx.x; i < len; i += kSortThreads) {
        const std::uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k2) == 0;
          const std::uint32_t x = sm[i], y = sm[l];
          if ((x > y) == up) {
            sm[i] = y;
            sm[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (std::uint32_t i = threadIdx.x; i < n; i += kSortThreads) data[i] = sm[i];
}

// Ordered hull list without the sort (many hull facets): per output row the
// count of its kNone facets, scanned, then the handles written in order.
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_hull_count(MergeDev a, std::uint32_t M,
                                                                    std::uint32_t* cnt) {
  const std::uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= M) return;
  std::uint32_t c = 0;
#pragma unroll
  for (int d = 0; d <= D; ++d) c += a.out_nbrs[std::uint64_t(d) * a.ostride + o] == kNoneId;
  cnt[o] = c;
}
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_hull_list(MergeDev a, std::uint32_t M,
                                                                   const std::uint32_t* base, std::uint32_t* hull) {
  const std::uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= M) return;
  std::uint32_t pos = base[o];
#pragma unroll
  for (int d = 0; d <= D; ++d)
    if (a.out_nbrs[std::uint64_t(d) * a.ostride + o] == kNoneId) hull[pos++] = o * (D + 1) + d;
}

// Hull row M + i for the i-th hull facet: {facet ids, kInf}, parity 0,
// neighbours[D] = owner; the owner's facet is linked back.
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_hull_emit(MergeDev a, std::uint32_t M,
                                                                   const std::uint32_t* hull, std::uint32_t H) {
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= H) return;
  const std::uint32_t hd = hull[i], o = hd / (D + 1), d = hd % (D + 1), h = M + i;
  std::uint32_t hv[D + 1];
#pragma unroll
  for (int j = 0, q = 0; j <= D; ++j)
    if (j != static_cast<int>(d)) hv[q++] = a.out_verts[std::uint64_t(j) * a.ostride + o];
  hv[D] = kInfVertex;
  emit_row<D>(a, h, hv, 0);
#pragma unroll
  for (int j = 0; j < D; ++j) a.out_nbrs[std::uint64_t(j) * a.ostride + h] = kNoneId;
  a.out_nbrs[std::uint64_t(D) * a.ostride + h] = o;
  a.out_nbrs[std::uint64_t(d) * a.ostride + o] = h;
}

// Ridge join: the ridge opposite hv[i] (i < D) of hull row h is {the other
// D-1 facet ids, kInf}; its two hull rows are linked.
template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_ridge_join(MergeDev a, std::uint32_t M, std::uint32_t H) {
  const std::uint64_t t = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= std::uint64_t(H) * D) return;
  const std::uint32_t h = M + static_cast<std::uint32_t>(t / D);
  const int i = static_cast<int>(t % D);
  std::uint32_t r[D];
#pragma unroll
  for (int j = 0, q = 0; j < D; ++j)
    if (j != i) r[q++] = __ldg(a.out_verts + std::uint64_t(j) * a.ostride + h);
  r[D - 1] = kInfVertex;
  const std::uint32_t partner = join_insert(
      a.join, a.join_mask, key_of<D>(r), h * (D + 1) + i, a.status, [&](std::uint32_t ov) {
        const std::uint32_t ph = ov / (D + 1), pi = ov % (D + 1);
        bool eq = true;
#pragma unroll
        for (int j = 0, q = 0; j < D; ++j)
          if (j != static_cast<int>(pi)) eq &= __ldg(a.out_verts + std::uint64_t(j) * a.ostride + ph) == r[q++];
        return eq;
      });
  if (partner != kNoneId) {
    const std::uint32_t ph = partner / (D + 1), pi = partner % (D + 1);
    a.out_nbrs[std::uint64_t(i) * a.ostride + h] = ph;
    a.out_nbrs[std::uint64_t(pi) * a.ostride + ph] = h;
  }
}

template <int D>
__global__ void __launch_bounds__(kMergeThreads) k_merge_hull_check(MergeDev a, std::uint32_t M, std::uint32_t H) {
  const std::uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= H) return;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < D; ++i) bad |= a.out_nbrs[std::uint64_t(i) * a.ostride + M + h] == kNoneId;
  if (bad) atomicOr(a.status, kStMergeDangling);
}

unsigned long long pow2_at_least(unsigned long long x) {
  unsigned long long p = 1024;
  while (p < x) p <<= 1;
  return p;
}

unsigned blocks_for(std::uint64_t n) { return static_cast<unsigned>((n + kMergeThreads - 1) / kMergeThreads); }

}  // namespace

// Writes the merged triangulation into out_* (SoA, stride a->ostride rows).
// Synchronizes the context stream (table sizing); *rows_out = M + H.
template <int D>
int merge_impl(sbdt_gpu_ctx* ctx, const sbdt_merge_args* args, std::uint64_t ostride, std::uint32_t* out_verts,
               std::uint32_t* out_nbrs, std::int8_t* out_parity, std::uint64_t* d_out_offsets,
               std::uint64_t* rows_out) {
  cudaStream_t st = ctx->stream;
  const std::uint64_t S = args->S, SB = args->S_B;
  MergeDev a{};
  a.k = args->k;
  a.labels = args->d_labels;
  a.offsets = args->d_offsets;
  a.verts = args->d_verts;
  a.nbrs = args->d_nbrs;
  a.parity = args->d_parity;
  a.border = args->d_border;
  a.S = S;
  a.tb_verts = args->d_tb_verts;
  a.tb_nbrs = args->d_tb_nbrs;
  a.tb_parity = args->d_tb_parity;
  a.SB = SB;
  a.WS = (S + 31) / 32;
  const std::uint64_t WB = (SB + 31) / 32;
  const std::uint64_t W = a.WS + WB;
  a.out_verts = out_verts;
  a.out_nbrs = out_nbrs;
  a.out_parity = out_parity;
  a.ostride = ostride;
  a.status = ctx->d_status;
  SBDT_WS(mask, std::uint32_t, "merge.mask", W + 1);
  SBDT_WS(base, std::uint32_t, "merge.base", W + 1);
  SBDT_WS(bsums, std::uint32_t, "merge.bsums", W / kScanTile + 2);
  SBDT_WS(counters, unsigned long long, "merge.counters", 4);
  SBDT_WS(hdr, std::uint32_t, "merge.hdr", 4);
  a.mask = mask;
  a.base = base;
  a.counters = counters;
  SBDT_CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * 4, st));
  if (W) SBDT_CUDA_TRY(cudaMemsetAsync(mask, 0, sizeof(std::uint32_t) * W, st));

  StageTimer t_flags(ctx, "merge.flags");
  if (S) {
    k_merge_keep<D><<<blocks_for(a.WS * 32), kMergeThreads, 0, st>>>(a);
    ++ctx->launches;
  }
  unsigned long long n_border = 0;
  SBDT_CUDA_TRY(cudaMemcpyAsync(&n_border, counters, 8, cudaMemcpyDeviceToHost, st));
  SBDT_CUDA_TRY(cudaStreamSynchronize(st));
  a.bset_mask = 0;
  if (n_border) {
    const unsigned long long cap = pow2_at_least(2 * n_border);
    SBDT_WS(bset, unsigned long long, "merge.bset", cap);
    SBDT_CUDA_TRY(cudaMemsetAsync(bset, 0xFF, sizeof(unsigned long long) * cap, st));
    a.bset = bset;
    a.bset_mask = cap - 1;
    k_merge_bset<D><<<blocks_for(S), kMergeThreads, 0, st>>>(a);
    ++ctx->launches;
  }
  if (SB) {
    k_merge_include<D><<<blocks_for(WB * 32), kMergeThreads, 0, st>>>(a);
    ++ctx->launches;
  }
  // base[w] = exclusive prefix of the word popcounts; base[W] = M
  exclusive_scan(base, base, W, bsums, hdr, st, &ctx->launches);
  SBDT_CUDA_TRY(cudaMemcpyAsync(base + W, hdr, 4, cudaMemcpyDeviceToDevice, st));
  k_merge_offsets<<<(a.k + 1 + 127) / 128, 128, 0, st>>>(a, d_out_offsets);
  ++ctx->launches;
  std::uint32_t hb[2] = {0, 0};
  SBDT_CUDA_TRY(cudaMemcpyAsync(&hb[0], hdr, 4, cudaMemcpyDeviceToHost, st));
  SBDT_CUDA_TRY(cudaMemcpyAsync(&hb[1], base + a.WS, 4, cudaMemcpyDeviceToHost, st));
  SBDT_CUDA_TRY(cudaStreamSynchronize(st));
  t_flags.end();
  const std::uint64_t M = hb[0], kept = hb[1];
  *rows_out = M;
  if (M > ostride) return fail(ctx, kErrRange, "merge: output capacity below the merged row count");
  if ((M + 1) * (D + 1) >= kPairedBit) return fail(ctx, kErrRange, "merge: row count exceeds the 31-bit join handle");

  StageTimer t_emit(ctx, "merge.emit");
  // join facets: at most D+1 per dropped partial row (each facet of a dropped
  // row has one kept neighbour) and D+1 per inserted T_B row
  const std::uint64_t qcap = (D + 1) * ((S - kept) + (M - kept)) + 64;
  SBDT_WS(queue, std::uint32_t, "merge.queue", qcap);
  unsigned* qcount = reinterpret_cast<unsigned*>(counters + 1);  // [0] = J, [1] = H
  SBDT_CUDA_TRY(cudaMemsetAsync(qcount, 0, 8, st));
  if (S) {
    k_merge_emit_partial<D><<<blocks_for(S), kMergeThreads, 0, st>>>(a, qcount, queue, qcap);
    ++ctx->launches;
  }
  if (SB) {
    k_merge_emit_tb<D><<<blocks_for(SB), kMergeThreads, 0, st>>>(a, qcount, queue, qcap);
    ++ctx->launches;
  }
  unsigned J = 0;
  SBDT_CUDA_TRY(cudaMemcpyAsync(&J, qcount, 4, cudaMemcpyDeviceToHost, st));
  SBDT_CUDA_TRY(cudaStreamSynchronize(st));
  if (J > qcap) return fail(ctx, kErrRange, "merge: join queue overflow");
  const unsigned long long jcap = pow2_at_least(2ull * J);
  SBDT_WS(join, unsigned long long, "merge.join", jcap);
  a.join = join;
  a.join_mask = jcap - 1;
  if (J) {
    SBDT_CUDA_TRY(cudaMemsetAsync(join, 0xFF, sizeof(unsigned long long) * jcap, st));
    k_merge_join<D><<<blocks_for(J), kMergeThreads, 0, st>>>(a, queue, J);
    ++ctx->launches;
  }
  t_emit.end();

  std::uint64_t H = 0;
  if ((args->flags & SBDT_MERGE_HULL) && J) {
    StageTimer t_hull(ctx, "merge.hull");
    SBDT_WS(hull, std::uint32_t, "merge.hull", J + 64);
    k_merge_hull_collect<D><<<blocks_for(J), kMergeThreads, 0, st>>>(a, queue, J, qcount + 1, hull, J + 64);
    ++ctx->launches;
    unsigned h32 = 0;
    SBDT_CUDA_TRY(cudaMemcpyAsync(&h32, qcount + 1, 4, cudaMemcpyDeviceToHost, st));
    SBDT_CUDA_TRY(cudaStreamSynchronize(st));
    H = h32;
    *rows_out = M + H;
    if (M + H > ostride) return fail(ctx, kErrRange, "merge: output capacity below the merged row count");
    if ((M + H + 1) * (D + 1) >= kPairedBit) return fail(ctx, kErrRange, "merge: row count exceeds the 31-bit join handle");
    if (H) {
      if (H <= static_cast<std::uint64_t>(kHullSortMax)) {
        std::uint32_t len = 2;
        while (len < H) len <<= 1;
        k_sort_small<<<1, kSortThreads, len * sizeof(std::uint32_t), st>>>(hull, static_cast<std::uint32_t>(H));
        ++ctx->launches;
      } else {
        SBDT_WS(hcnt, std::uint32_t, "merge.hcnt", M + 1);
        SBDT_WS(hsums, std::uint32_t, "merge.hsums", M / kScanTile + 2);
        k_merge_hull_count<D><<<blocks_for(M), kMergeThreads, 0, st>>>(a, static_cast<std::uint32_t>(M), hcnt);
        exclusive_scan(hcnt, hcnt, M, hsums, hdr + 2, st, &ctx->launches);
        k_merge_hull_list<D><<<blocks_for(M), kMergeThreads, 0, st>>>(a, static_cast<std::uint32_t>(M), hcnt, hull);
        ctx->launches += 2;
      }
      k_merge_hull_emit<D><<<blocks_for(H), kMergeThreads, 0, st>>>(a, static_cast<std::uint32_t>(M), hull,
                                                                       static_cast<std::uint32_t>(H));
      const unsigned long long rcap = pow2_at_least(2ull * D * H);
      if (rcap > jcap) {
        SBDT_WS(join2, unsigned long long, "merge.join2", rcap);
        a.join = join2;
      }
      a.join_mask = rcap - 1;
      SBDT_CUDA_TRY(cudaMemsetAsync(a.join, 0xFF, sizeof(unsigned long long) * rcap, st));
      k_merge_ridge_join<D><<<blocks_for(H * D), kMergeThreads, 0, st>>>(a, static_cast<std::uint32_t>(M),
                                                                           static_cast<std::uint32_t>(H));
      k_merge_hull_check<D><<<blocks_for(H), kMergeThreads, 0, st>>>(a, static_cast<std::uint32_t>(M),
                                                                       static_cast<std::uint32_t>(H));
      ctx->launches += 3;
    }
  }
  // offsets[k+1] = M, offsets[k+2] = M + H
  const std::uint64_t tail[2] = {M, M + H};
  SBDT_CUDA_TRY(cudaMemcpyAsync(d_out_offsets + args->k + 1, tail, 16, cudaMemcpyHostToDevice, st));
  SBDT_CUDA_TRY(cudaStreamSynchronize(st));
  *rows_out = M + H;
  return kOk;
}

template int merge_impl<2>(sbdt_gpu_ctx*, const sbdt_merge_args*, std::uint64_t, std::uint32_t*, std::uint32_t*,
                           std::int8_t*, std::uint64_t*, std::uint64_t*);
template int merge_impl<3>(sbdt_gpu_ctx*, const sbdt_merge_args*, std::uint64_t, std::uint32_t*, std::uint32_t*,
                           std::int8_t*, std::uint64_t*, std::uint64_t*);

}  // namespace sbdt_gpu
