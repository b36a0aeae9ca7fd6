// K8 — SPEC find_border semantics: the BFS
// from hull_simplices (triangulation.cpp:34-53) that adds a dequeued simplex
// to the border iff it is positive and then enqueues its unmarked neighbours.
// Its result is order-independent: a simplex is a border simplex iff it is
// positive and its connected component in the graph induced on positive
// simplices (neighbour links, part-local) contains a hull simplex. On the GPU
// that is a union-find over the compacted positive simplices (atomic
// hooking to the smaller root + path compression), then a root mark.
#include <cuda_runtime.h>

#include "common.cuh"
#include "context.cuh"
#include "scan.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {

int compact_flags(sbdt_gpu_ctx* ctx, const std::uint8_t* d_flags, std::uint64_t n, std::uint32_t* d_out,
                  std::uint64_t* d_count);

// Union-find over ranks with parent[x] <= x throughout (roots hooked under
// smaller roots, the initial parents are smaller neighbours): the
// representative walk shortens the path as it goes (intermediate pointer
// jumping, ECL-CC); a failed hook continues from the value the CAS saw.
__device__ __forceinline__ std::uint32_t find_root(std::uint32_t* parent, std::uint32_t v) {
  std::uint32_t curr = parent[v];
  if (curr != v) {
    std::uint32_t next, prev = v;
    while (curr > (next = parent[curr])) {
      parent[prev] = next;
      prev = curr;
      curr = next;
    }
  }
  return curr;
}

__device__ __forceinline__ void unite(std::uint32_t* parent, std::uint32_t a, std::uint32_t b) {
  std::uint32_t ra = find_root(parent, a), rb = find_root(parent, b);
  while (ra != rb) {
    if (ra < rb) {
      const std::uint32_t ret = atomicCAS(&parent[rb], rb, ra);
      if (ret == rb) return;
      rb = ret;
    } else {
      const std::uint32_t ret = atomicCAS(&parent[ra], ra, rb);
      if (ret == ra) return;
      ra = ret;
    }
  }
}

__device__ __forceinline__ std::uint32_t part_of_row(const std::uint64_t* offs, std::uint32_t k, std::uint64_t s) {
  std::uint32_t lo = 0, hi = k;
  while (hi - lo > 1) {
    const std::uint32_t mid = (lo + hi) >> 1;
    if (offs[mid] <= s) lo = mid;
    else hi = mid;
  }
  return lo;
}

// The positive rows are ranked through a bitmap (one bit per simplex row)
// and its per-word exclusive prefix: rank(s) = prefix[s / 32] + popc(bits
// below s), so the union-find runs on the compacted positive rows (parent
// array of P words) and a neighbour's positivity and rank come from two
// words that stay in L2 (S / 8 + S / 8 bytes) instead of S-sized gathers.
// The hull rows (an infinite vertex) come from the border stage's hull queue
// as a second bitmap.
struct ReachArgs {
  int dim;
  std::uint32_t k;
  const std::uint64_t* offsets;
  const std::uint32_t* verts;
  const std::uint32_t* nbrs;
  std::uint64_t S;
  const std::uint8_t* positive;
  std::uint32_t* bits;        // positive rows, [W]
  std::uint32_t* wpre;        // exclusive prefix of popc(bits), [W + 1]
  std::uint32_t* hbits;       // hull rows (an infinite vertex), [W]
  const std::uint32_t* infq;  // the border stage's hull rows
  const unsigned* infc;
  std::uint32_t* pos_ids;     // [P]: rank -> row
  std::uint32_t* parent;      // [P]
  std::uint8_t* mark;         // [P]
  std::uint8_t* border;
  std::uint8_t* vflags;
};

__device__ __forceinline__ bool bit_at(const std::uint32_t* b, std::uint64_t s) {
  return (__ldg(b + (s >> 5)) >> (s & 31u)) & 1u;
}
__device__ __forceinline__ std::uint32_t rank_of(const ReachArgs& a, std::uint64_t s) {
  const std::uint32_t w = __ldg(a.bits + (s >> 5));
  return __ldg(a.wpre + (s >> 5)) + __popc(w & ((1u << (s & 31u)) - 1u));
}

// the positive bitmap: a thread reads 4 flag bytes (one word), a warp
// covers 128 rows = 4 bitmap words (bit b of word j from lane 8 j + b / 4)
__global__ void k_reach_bits(ReachArgs a, std::uint32_t* __restrict__ wcnt) {
  const std::uint64_t W = (a.S + 31) / 32;
  const std::uint64_t S4 = a.S / 4;
  const unsigned lane = threadIdx.x & 31u;
  for (std::uint64_t t = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < (W + 3) / 4 * 32;
       t += std::uint64_t(gridDim.x) * blockDim.x) {
    std::uint32_t f = 0;  // four flag bytes of rows 4t .. 4t + 3
    if (t < S4) {
      f = __ldcs(reinterpret_cast<const std::uint32_t*>(a.positive) + t);
    } else {
      for (int b = 0; b < 4; ++b)
        if (4 * t + b < a.S && a.positive[4 * t + b]) f |= 1u << (8 * b);
    }
    const std::uint32_t nib = (f & 0xFFu ? 1u : 0u) | (f & 0xFF00u ? 2u : 0u) | (f & 0xFF0000u ? 4u : 0u) |
                              (f & 0xFF000000u ? 8u : 0u);
    // word j of this warp = lanes 8j .. 8j + 7, 4 bits each
    std::uint32_t w = nib << (4 * (lane & 7u));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    const std::uint64_t wi = (t >> 3);  // 8 threads per word
    if ((lane & 7u) == 0 && wi < W) {
      a.bits[wi] = w;
      a.hbits[wi] = 0u;
      wcnt[wi] = static_cast<std::uint32_t>(__popc(w));
    }
  }
}

__global__ void k_reach_hull(ReachArgs a) {
  const unsigned cnt = *a.infc;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const std::uint32_t s = a.infq[i];
    atomicOr(a.hbits + (s >> 5), 1u << (s & 31u));
  }
}

// rank -> row (one thread per bitmap word)
__global__ void k_reach_init(ReachArgs a) {
  const std::uint64_t W = (a.S + 31) / 32;
  for (std::uint64_t wi = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; wi < W;
       wi += std::uint64_t(gridDim.x) * blockDim.x) {
    std::uint32_t w = a.bits[wi];
    std::uint32_t i = a.wpre[wi];
    while (w) {
      const int b = __ffs(w) - 1;
      w &= w - 1;
      a.pos_ids[i++] = static_cast<std::uint32_t>(wi * 32 + b);
    }
  }
}

constexpr std::uint32_t kReachSmemOffs = 1024;  // part offsets staged in shared memory up to this many (k + 1)

// Per positive row (rank i): the ranks of its positive neighbours with a
// smaller row (kNoRank otherwise), stored rank-major for the hooking pass,
// the hull seed test (triangulation.cpp:34-53: the row or one of its
// neighbours has an infinite vertex) and the initial parent (ECL-CC style:
// the smallest of the row's own rank and those neighbour ranks, so most
// links are already inside a tree before any atomic).
constexpr std::uint32_t kNoRank = 0xFFFFFFFFu;

__global__ void k_reach_link(ReachArgs a, const std::uint32_t* __restrict__ ptotal, std::uint32_t* __restrict__ nrank) {
  extern __shared__ std::uint64_t s_off_sh[];
  if (a.k + 1 <= kReachSmemOffs)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  const bool small = a.k + 1 <= kReachSmemOffs;  // else in place (very large k)
  const std::uint32_t P = *ptotal;
  const int D = a.dim;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const std::uint64_t s = a.pos_ids[i];
    const std::uint64_t off = small ? s_off_sh[part_of_row(s_off_sh, a.k, s)] : a.offsets[part_of_row(a.offsets, a.k, s)];
    bool hull = bit_at(a.hbits, s);
    std::uint32_t p = i;
    for (int d = 0; d <= D; ++d) {
      const std::uint64_t nb = off + a.nbrs[std::uint64_t(d) * a.S + s];
      hull = hull || bit_at(a.hbits, nb);
      std::uint32_t r = kNoRank;
      if (nb < s && bit_at(a.bits, nb)) {
        r = rank_of(a, nb);
        p = min(p, r);
      }
      nrank[std::uint64_t(d) * P + i] = r;
    }
    a.parent[i] = p;
    a.mark[i] = hull ? 2 : 0;  // seed (resolved to its root after the hooking)
  }
}

// The hooking runs in two phases. The rows come in a spatially coherent order
// (the host builder's Morton order), so most links join ranks that are close:
// phase 1 (k_reach_hook_tiles) takes a tile of kReachTile consecutive ranks
// per CTA, runs the union-find over the links INSIDE the tile in shared
// memory (same hooking rule: the larger root under the smaller one) and
// writes every rank's tile root as its global parent; phase 2 (k_reach_hook)
// unites over the links that leave a tile, on trees that are one hop deep.
constexpr std::uint32_t kReachTile = 8192;
constexpr unsigned kReachTileThreads = 1024;
constexpr int kReachEpt = kReachTile / kReachTileThreads;  // ranks per thread

// Inside a tile the components are found by min-label propagation with
// hooking and pointer jumping (FastSV style) instead of CAS hooking:
// consecutive ranks are mostly neighbours, and hooking root under root chains
// them into paths as long as the tile, which every later find walks (measured:
// 0.50-0.62 ms for this phase). lbl[x] <= x is always a rank of x's component;
// a round lowers, for every link (u, v), the labels of u, v and of their
// current label holders to the smaller of the two labels (shared-memory
// atomicMin), then every rank jumps to its label's label; at the fixed point
// both ends of every link carry the same label and lbl[lbl[x]] = lbl[x], i.e.
// the label is the component's root (its smallest rank in the tile).
__global__ void __launch_bounds__(kReachTileThreads) k_reach_hook_tiles(ReachArgs a,
                                                                        const std::uint32_t* __restrict__ ptotal,
                                                                        const std::uint32_t* __restrict__ nrank) {
  __shared__ std::uint32_t sp[kReachTile];
  const std::uint32_t P = *ptotal;
  const int D = a.dim;
  const std::uint32_t ntiles = (P + kReachTile - 1) / kReachTile;
  for (std::uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const std::uint32_t base = tile * kReachTile;
    const std::uint32_t cnt = min(kReachTile, P - base);
    // this thread's ranks and their in-tile links (local indices), in registers
    std::uint32_t lk[kReachEpt][4];
#pragma unroll
    for (int q = 0; q < kReachEpt; ++q) {
      const std::uint32_t e = threadIdx.x + q * kReachTileThreads;
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        std::uint32_t r = kNoRank;
        if (e < cnt && d <= D) r = __ldg(nrank + std::uint64_t(d) * P + base + e);
        lk[q][d] = (r != kNoRank && r >= base) ? r - base : kNoRank;
      }
      if (e < cnt) sp[e] = e;
    }
    __syncthreads();
    for (;;) {
      bool changed = false;
#pragma unroll
      for (int q = 0; q < kReachEpt; ++q) {
        const std::uint32_t e = threadIdx.x + q * kReachTileThreads;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          const std::uint32_t r = lk[q][d];
          if (r == kNoRank) continue;
          const std::uint32_t la = sp[e], lb = sp[r];
          if (la < lb) {
            atomicMin(&sp[lb], la);
            atomicMin(&sp[r], la);
            changed = true;
          } else if (lb < la) {
            atomicMin(&sp[la], lb);
            atomicMin(&sp[e], lb);
            changed = true;
          }
        }
      }
      const int any = __syncthreads_or(changed ? 1 : 0);
      // pointer jumping (each word is written by its owner only in this phase)
#pragma unroll
      for (int q = 0; q < kReachEpt; ++q) {
        const std::uint32_t e = threadIdx.x + q * kReachTileThreads;
        if (e < cnt) {
          std::uint32_t x = sp[e];
          x = sp[x];
          x = sp[x];
          sp[e] = x;
        }
      }
      __syncthreads();
      if (!any) break;
    }
#pragma unroll
    for (int q = 0; q < kReachEpt; ++q) {
      const std::uint32_t e = threadIdx.x + q * kReachTileThreads;
      if (e < cnt) a.parent[base + e] = base + sp[e];
    }
    __syncthreads();
  }
}

// every positive-positive link that leaves its tile, once (from the larger
// row): union-find with path halving, the larger root hooked under the
// smaller one
__global__ void k_reach_hook(ReachArgs a, const std::uint32_t* __restrict__ ptotal,
                             const std::uint32_t* __restrict__ nrank) {
  const std::uint32_t P = *ptotal;
  const int D = a.dim;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const std::uint32_t base = i - i % kReachTile;
    for (int d = 0; d <= D; ++d) {
      const std::uint32_t r = nrank[std::uint64_t(d) * P + i];
      if (r != kNoRank && r < base) unite(a.parent, i, r);
    }
  }
}

// roots of the seeds marked; then every row's root and a count of the rows
// whose component holds no seed
__global__ void k_reach_mark(ReachArgs a, const std::uint32_t* __restrict__ ptotal) {
  const std::uint32_t P = *ptotal;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x)
    if (a.mark[i] & 2u) a.mark[find_root(a.parent, i)] |= 1u;
}

// (the roots go to a separate array: the parent array may still receive
// path-shortening writes of other threads, which store ancestors, not roots)
__global__ void k_reach_roots(ReachArgs a, const std::uint32_t* __restrict__ ptotal, unsigned* __restrict__ unreached,
                              std::uint32_t* __restrict__ rootof) {
  const std::uint32_t P = *ptotal;
  unsigned c = 0;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const std::uint32_t r = find_root(a.parent, i);
    rootof[i] = r;
    c += (a.mark[r] & 1u) ? 0u : 1u;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31u) == 0 && c) atomicAdd(unreached, c);
}

// border flags (and the BFS vertex flags). When every component holds a seed
// (the usual case) the BFS border is the full-scan positive set: a streaming
// copy of the flags; else per positive row from its root's mark.
__global__ void k_reach_final(ReachArgs a, const std::uint32_t* __restrict__ ptotal,
                              const unsigned* __restrict__ unreached, const std::uint8_t* __restrict__ pos_vflags,
                              std::uint64_t n, const std::uint32_t* __restrict__ rootof) {
  const int D = a.dim;
  if (*unreached == 0) {
    const std::uint64_t t0 = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const std::uint64_t step = std::uint64_t(gridDim.x) * blockDim.x;
    auto copy = [&](std::uint8_t* dst, const std::uint8_t* src, std::uint64_t len) {
      // 16-byte vectors when both ends are aligned (workspace / cudaMalloc
      // bases), bytes for the rest
      const bool vec = ((reinterpret_cast<std::uintptr_t>(dst) | reinterpret_cast<std::uintptr_t>(src)) & 15u) == 0;
      const std::uint64_t nv = vec ? len / 16 : 0;
      for (std::uint64_t q = t0; q < nv; q += step)
        reinterpret_cast<uint4*>(dst)[q] = __ldcs(reinterpret_cast<const uint4*>(src) + q);
      for (std::uint64_t q = nv * 16 + t0; q < len; q += step) dst[q] = src[q];
    };
    copy(a.border, a.positive, a.S);
    if (a.vflags) copy(a.vflags, pos_vflags, n);
    return;
  }
  const std::uint32_t P = *ptotal;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const std::uint64_t s = a.pos_ids[i];
    const bool b = (a.mark[rootof[i]] & 1u) != 0;
    a.border[s] = b ? 1 : 0;
    if (b && a.vflags)
      for (int j = 0; j <= D; ++j) {
        const std::uint32_t v = a.verts[std::uint64_t(j) * a.S + s];
        if (v != kInfVertex) a.vflags[v] = 1;
      }
  }
}

int reach_impl(sbdt_gpu_ctx* ctx, const sbdt_border_args* in) {
  cudaStream_t st = ctx->stream;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  StageTimer timer(ctx, "border.hull_bfs");
  const std::uint64_t W = (in->S + 31) / 32;
  SBDT_WS(bits, std::uint32_t, "reach.bits", W + 1);
  SBDT_WS(hbits, std::uint32_t, "reach.hbits", W + 1);
  SBDT_WS(wcnt, std::uint32_t, "reach.wcnt", W + 1);
  SBDT_WS(wpre, std::uint32_t, "reach.wpre", W + 1);
  SBDT_WS(wbs, std::uint32_t, "reach.wbs", W / kScanTile + 4);
  SBDT_WS(ptot, std::uint32_t, "reach.ptotal", 1);
  SBDT_WS(pos_ids, std::uint32_t, "reach.pos_ids", in->S + 1);
  SBDT_WS(parent, std::uint32_t, "reach.parent", in->S + 1);
  SBDT_WS(mark, std::uint8_t, "reach.mark", in->S + 1);
  SBDT_WS(nrank, std::uint32_t, "reach.nrank", (in->S + 1) * (in->dim + 1));
  SBDT_WS(unreached, unsigned, "reach.unreached", 1);
  // the border stage's hull-row queue (same workspaces, filled by every policy)
  SBDT_WS(infq, std::uint32_t, "border.infq", in->S + 1024);
  SBDT_WS(infc, unsigned, "border.infc", 1);
  SBDT_CUDA_TRY(cudaMemsetAsync(in->d_border, 0, in->S, st));
  if (in->d_bfs_vertex_flags) SBDT_CUDA_TRY(cudaMemsetAsync(in->d_bfs_vertex_flags, 0, in->n, st));
  ReachArgs a{in->dim, in->k, in->d_offsets, in->d_verts, in->d_nbrs, in->S, in->d_positive, bits, wpre, hbits,
              infq, infc, pos_ids, parent, mark, in->d_border, in->d_bfs_vertex_flags};
  const unsigned blocks = static_cast<unsigned>(sms) * 8;
  const std::size_t sh = in->k + 1 <= kReachSmemOffs ? sizeof(std::uint64_t) * (in->k + 1) : 0;
  k_reach_bits<<<blocks, 256, 0, st>>>(a, wcnt);
  k_reach_hull<<<static_cast<unsigned>(sms), 256, 0, st>>>(a);
  exclusive_scan(wcnt, wpre, W, wbs, ptot, st, &ctx->launches);
  k_reach_init<<<blocks, 256, 0, st>>>(a);
  k_reach_link<<<blocks, 256, sh, st>>>(a, ptot, nrank);
  k_reach_hook_tiles<<<static_cast<unsigned>(sms) * 4, kReachTileThreads, 0, st>>>(a, ptot, nrank);
  k_reach_hook<<<blocks, 256, 0, st>>>(a, ptot, nrank);
  k_reach_mark<<<blocks, 256, 0, st>>>(a, ptot);
  SBDT_CUDA_TRY(cudaMemsetAsync(unreached, 0, sizeof(unsigned), st));
  // nrank is free after the hooking: its first P words take the roots
  k_reach_roots<<<blocks, 256, 0, st>>>(a, ptot, unreached, nrank);
  k_reach_final<<<blocks, 256, 0, st>>>(a, ptot, unreached, in->d_vertex_flags, in->n, nrank);
  ctx->launches += 9;
  if (in->d_bfs_vertex_flags && in->d_bfs_vertex_ids && in->d_bfs_vertex_count) {
    const int rc = compact_flags(ctx, in->d_bfs_vertex_flags, in->n, in->d_bfs_vertex_ids, in->d_bfs_vertex_count);
    if (rc != kOk) return rc;
  }
  SBDT_CUDA_TRY(cudaGetLastError());
  return kOk;
}

}  // namespace sbdt_gpu
