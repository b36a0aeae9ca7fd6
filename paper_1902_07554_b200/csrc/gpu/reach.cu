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
#include "sbdt_gpu.h"

namespace sbdt_gpu {

int compact_flags(sbdt_gpu_ctx* ctx, const std::uint8_t* d_flags, std::uint64_t n, std::uint32_t* d_out,
                  std::uint64_t* d_count);

__device__ __forceinline__ std::uint32_t find_root(std::uint32_t* parent, std::uint32_t x) {
  std::uint32_t p = parent[x];
  while (p != x) {
    const std::uint32_t gp = parent[p];
    if (gp != p) parent[x] = gp;  // path halving (benign race: any ancestor is valid)
    x = p;
    p = gp;
  }
  return x;
}

__device__ __forceinline__ void unite(std::uint32_t* parent, std::uint32_t a, std::uint32_t b) {
  for (;;) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a < b) {
      const std::uint32_t t = a;
      a = b;
      b = t;
    }
    // hook the larger root under the smaller one
    if (atomicCAS(&parent[a], a, b) == a) return;
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

struct ReachArgs {
  int dim;
  std::uint32_t k;
  const std::uint64_t* offsets;
  const std::uint32_t* verts;
  const std::uint32_t* nbrs;
  std::uint64_t S;
  const std::uint8_t* positive;
  const std::uint32_t* pos_ids;
  const std::uint64_t* pos_count;
  std::uint32_t* cidx;
  std::uint32_t* parent;
  std::uint8_t* mark;
  std::uint8_t* border;
  std::uint8_t* vflags;
};

__global__ void k_reach_init(ReachArgs a) {
  const std::uint64_t P = *a.pos_count;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    a.cidx[a.pos_ids[i]] = static_cast<std::uint32_t>(i);
    a.parent[i] = static_cast<std::uint32_t>(i);
    a.mark[i] = 0;
  }
}

constexpr std::uint32_t kReachSmemOffs = 1024;  // part offsets staged in shared memory up to this many (k + 1)

__global__ void k_reach_hook(ReachArgs a) {
  extern __shared__ std::uint64_t s_off_sh[];
  if (a.k + 1 <= kReachSmemOffs)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  const bool small = a.k + 1 <= kReachSmemOffs;  // else in place (very large k)
  const std::uint64_t P = *a.pos_count;
  const int D = a.dim;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t s = a.pos_ids[i];
    const std::uint64_t off = small ? s_off_sh[part_of_row(s_off_sh, a.k, s)] : a.offsets[part_of_row(a.offsets, a.k, s)];
    for (int d = 0; d <= D; ++d) {
      const std::uint64_t nb = off + a.nbrs[std::uint64_t(d) * a.S + s];
      if (nb < s && a.positive[nb]) unite(a.parent, static_cast<std::uint32_t>(i), a.cidx[nb]);
    }
  }
}

// hull seed test (triangulation.cpp:34-53) + root mark
__global__ void k_reach_mark(ReachArgs a) {
  extern __shared__ std::uint64_t s_off_sh[];
  if (a.k + 1 <= kReachSmemOffs)
    for (std::uint32_t j = threadIdx.x; j <= a.k; j += blockDim.x) s_off_sh[j] = a.offsets[j];
  __syncthreads();
  const bool small = a.k + 1 <= kReachSmemOffs;  // else in place (very large k)
  const std::uint64_t P = *a.pos_count;
  const int D = a.dim;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t s = a.pos_ids[i];
    bool hull = a.verts[std::uint64_t(D) * a.S + s] == kInfVertex;
    if (!hull) {
      const std::uint64_t off = small ? s_off_sh[part_of_row(s_off_sh, a.k, s)] : a.offsets[part_of_row(a.offsets, a.k, s)];
      for (int d = 0; d <= D && !hull; ++d) {
        const std::uint64_t nb = off + a.nbrs[std::uint64_t(d) * a.S + s];
        hull = a.verts[std::uint64_t(D) * a.S + nb] == kInfVertex;
      }
    }
    if (hull) a.mark[find_root(a.parent, static_cast<std::uint32_t>(i))] = 1;
  }
}

__global__ void k_reach_final(ReachArgs a) {
  const std::uint64_t P = *a.pos_count;
  const int D = a.dim;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < P;
       i += std::uint64_t(gridDim.x) * blockDim.x) {
    const std::uint64_t s = a.pos_ids[i];
    const bool b = a.mark[find_root(a.parent, static_cast<std::uint32_t>(i))] != 0;
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
  SBDT_WS(pos_ids, std::uint32_t, "reach.pos_ids", in->S + 1);
  SBDT_WS(pos_count, std::uint64_t, "reach.pos_count", 1);
  SBDT_WS(cidx, std::uint32_t, "reach.cidx", in->S + 1);
  SBDT_WS(parent, std::uint32_t, "reach.parent", in->S + 1);
  SBDT_WS(mark, std::uint8_t, "reach.mark", in->S + 1);
  int rc = compact_flags(ctx, in->d_positive, in->S, pos_ids, pos_count);
  if (rc != kOk) return rc;
  SBDT_CUDA_TRY(cudaMemsetAsync(in->d_border, 0, in->S, st));
  if (in->d_bfs_vertex_flags) SBDT_CUDA_TRY(cudaMemsetAsync(in->d_bfs_vertex_flags, 0, in->n, st));
  ReachArgs a{in->dim, in->k, in->d_offsets, in->d_verts, in->d_nbrs, in->S, in->d_positive, pos_ids, pos_count,
              cidx, parent, mark, in->d_border, in->d_bfs_vertex_flags};
  const unsigned blocks = static_cast<unsigned>(sms) * 8;
  const std::size_t sh = in->k + 1 <= kReachSmemOffs ? sizeof(std::uint64_t) * (in->k + 1) : 0;
  k_reach_init<<<blocks, 256, 0, st>>>(a);
  k_reach_hook<<<blocks, 256, sh, st>>>(a);
  k_reach_mark<<<blocks, 256, sh, st>>>(a);
  k_reach_final<<<blocks, 256, 0, st>>>(a);
  ctx->launches += 4;
  if (in->d_bfs_vertex_flags && in->d_bfs_vertex_ids && in->d_bfs_vertex_count) {
    rc = compact_flags(ctx, in->d_bfs_vertex_flags, in->n, in->d_bfs_vertex_ids, in->d_bfs_vertex_count);
    if (rc != kOk) return rc;
  }
  SBDT_CUDA_TRY(cudaGetLastError());
  return kOk;
}

}  // namespace sbdt_gpu
