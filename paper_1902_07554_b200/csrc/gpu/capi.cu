// C ABI (include/sbdt_gpu.h): context management, host-buffer entry points
// (H2D -> kernels -> D2H, synchronous) and device-pointer entry points
// (asynchronous on the context stream). No exception crosses this boundary.
#include <algorithm>
#include <thread>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>
#include <new>
#include <string>

#include "common.cuh"
#include "context.cuh"
#include "owner_grid.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {
template <int D>
int assign_impl(sbdt_gpu_ctx*, const double*, std::uint64_t, const std::uint32_t*, const std::uint32_t*,
                std::uint32_t, std::uint32_t*, unsigned long long*);
int bucket_impl(sbdt_gpu_ctx*, const std::uint32_t*, std::uint64_t, std::uint32_t, std::uint64_t*, std::uint32_t*);
template <int D>
int border_impl(sbdt_gpu_ctx*, const sbdt_border_args*);
int reach_impl(sbdt_gpu_ctx*, const sbdt_border_args*);
int assign_stats(sbdt_gpu_ctx*, unsigned*);
template <int D>
int merge_impl(sbdt_gpu_ctx*, const sbdt_merge_args*, std::uint64_t, std::uint32_t*, std::uint32_t*, std::int8_t*,
               std::uint64_t*, std::uint64_t*);
}  // namespace sbdt_gpu

using namespace sbdt_gpu;

namespace {

template <typename T>
int dalloc(sbdt_gpu_ctx* ctx, const char* name, std::size_t count, T** out) {
  cudaError_t e = cudaSuccess;
  *out = static_cast<T*>(workspace(ctx, name, sizeof(T) * (count ? count : 1), &e));
  if (!*out) return fail_cuda(ctx, e, name);
  return kOk;
}

int finish(sbdt_gpu_ctx* ctx) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return fail_cuda(ctx, e, "cudaStreamSynchronize");
  return sbdt_gpu_check_status(ctx);
}

}  // namespace

#define TRY(x)                 \
  do {                         \
    const int rc_ = (x);       \
    if (rc_ != kOk) return rc_; \
  } while (0)

extern "C" {

int sbdt_gpu_host_alloc(uint64_t bytes, void** out) {
  if (!out) return SBDT_ERR_INVALID;
  *out = nullptr;
  const cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    *out = nullptr;
    return e == cudaErrorMemoryAllocation ? SBDT_ERR_OOM : SBDT_ERR_CUDA;
  }
  return SBDT_OK;
}

void sbdt_gpu_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int sbdt_gpu_create(int device, sbdt_gpu_ctx** out) {
  if (!out) return SBDT_ERR_INVALID;
  *out = nullptr;
  sbdt_gpu_ctx* ctx = new (std::nothrow) sbdt_gpu_ctx();
  if (!ctx) return SBDT_ERR_OOM;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_status, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(ctx->d_status, 0, sizeof(unsigned));
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? SBDT_ERR_OOM : SBDT_ERR_CUDA;
    delete ctx;
    return code;
  }
  ctx->own_stream = true;
  *out = ctx;
  return SBDT_OK;
}

void sbdt_gpu_destroy(sbdt_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (auto& kv : ctx->bufs)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  if (ctx->d_status) cudaFree(ctx->d_status);
  for (cudaEvent_t e : ctx->chunk_events) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->chunk_done) cudaEventDestroy(e);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  if (ctx->sample_stage) cudaFreeHost(ctx->sample_stage);
  if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->wide_stream) cudaStreamDestroy(ctx->wide_stream);
  if (ctx->wide_join_ev) cudaEventDestroy(ctx->wide_join_ev);
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* sbdt_gpu_last_error(const sbdt_gpu_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int sbdt_gpu_set_stream(sbdt_gpu_ctx* ctx, void* stream) {
  if (!ctx) return SBDT_ERR_INVALID;
  if (ctx->own_stream && ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  // used as given: NULL is the legacy default stream (torch's default stream)
  ctx->stream = static_cast<cudaStream_t>(stream);
  ctx->own_stream = false;
  return SBDT_OK;
}

int sbdt_gpu_synchronize(sbdt_gpu_ctx* ctx) {
  if (!ctx) return SBDT_ERR_INVALID;
  return finish(ctx);
}

unsigned long long sbdt_gpu_launch_count(const sbdt_gpu_ctx* ctx) { return ctx ? ctx->launches : 0ULL; }

int sbdt_gpu_set_timing(sbdt_gpu_ctx* ctx, int enable) {
  if (!ctx) return SBDT_ERR_INVALID;
  ctx->timing = (enable & 1) != 0;
  ctx->census = (enable & 2) != 0;
  ctx->stages.clear();
  ctx->events_used = 0;
  return SBDT_OK;
}

int sbdt_gpu_stage_times(sbdt_gpu_ctx* ctx, char* names, int names_len, float* ms, int max_stages) {
  if (!ctx) return -SBDT_ERR_INVALID;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return -fail_cuda(ctx, e, "stage_times sync");
  int count = 0;
  std::string all;
  for (const auto& s : ctx->stages) {
    if (count >= max_stages) break;
    float t = 0.f;
    cudaEventElapsedTime(&t, s.start, s.stop);
    ms[count++] = t;
    all += s.name;
    all += '\n';
  }
  if (names && names_len > 0) {
    const std::size_t nb = all.size() < static_cast<std::size_t>(names_len - 1) ? all.size() : names_len - 1;
    std::memcpy(names, all.data(), nb);
    names[nb] = 0;
  }
  ctx->stages.clear();
  ctx->events_used = 0;
  return count;
}

int sbdt_gpu_assign_table_stats(sbdt_gpu_ctx* ctx, unsigned* out6) {
  if (!ctx || !out6) return SBDT_ERR_INVALID;
  return assign_stats(ctx, out6) == kOk ? SBDT_OK : SBDT_ERR_INVALID;
}

int sbdt_gpu_set_fill(sbdt_gpu_ctx* ctx, sbdt_fill_fn fill, void* user) {
  if (!ctx) return SBDT_ERR_INVALID;
  ctx->fill = fill;
  ctx->fill_user = user;
  return SBDT_OK;
}

int sbdt_gpu_border_stats(sbdt_gpu_ctx* ctx, unsigned long long* out, int count) {
  if (!ctx || !out || count < 0) return SBDT_ERR_INVALID;
  auto it = ctx->bufs.find("border.counters");
  if (it == ctx->bufs.end()) return SBDT_ERR_INVALID;
  const int c = count < kBorderCounters ? count : kBorderCounters;
  cudaStreamSynchronize(ctx->stream);
  cudaMemcpy(out, it->second.ptr, sizeof(unsigned long long) * c, cudaMemcpyDeviceToHost);
  return SBDT_OK;
}

int sbdt_gpu_check_status(sbdt_gpu_ctx* ctx) {
  if (!ctx) return SBDT_ERR_INVALID;
  unsigned st = 0;
  cudaError_t e = cudaMemcpy(&st, ctx->d_status, sizeof(unsigned), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail_cuda(ctx, e, "status readback");
  if (st) cudaMemset(ctx->d_status, 0, sizeof(unsigned));
  if (st & kStDegenerate) return fail(ctx, SBDT_ERR_DEGENERATE, "degenerate simplex (zero orientation) in a partial triangulation");
  if (st & kStGridCap) return fail(ctx, SBDT_ERR_RANGE, "grid index would exceed 4 n / c_G^D cells (degenerate bbox?)");
  if (st & kStQueueOverflow) return fail(ctx, SBDT_ERR_RANGE, "escalation queue overflow");
  if (st & 8u) return fail(ctx, SBDT_ERR_MERGE, "InconsistentMerge: a facet with more than two finite owners");
  if (st & 16u) return fail(ctx, SBDT_ERR_MERGE, "DanglingFacet: a hull ridge without exactly two hull facets");
  if (st & kStLabelRange) return fail(ctx, SBDT_ERR_INVALID, "sample label out of range (must be < k)");
  return SBDT_OK;
}

int sbdt_gpu_assign_points_dev(sbdt_gpu_ctx* ctx, int dim, const double* d_coords, uint64_t n,
                               const uint32_t* d_sample_ids, const uint32_t* d_sample_labels, uint32_t m,
                               uint32_t k, uint32_t* d_labels_out, uint64_t* d_part_offsets_out,
                               uint32_t* d_part_ids_out, uint64_t* d_bbox_ordered_out) {
  if (!ctx) return SBDT_ERR_INVALID;
  if (dim != 2 && dim != 3) return fail(ctx, SBDT_ERR_INVALID, "dim must be 2 or 3");
  if (m == 0 || k == 0 || k >= 0xFFFE) return fail(ctx, SBDT_ERR_INVALID, "need m >= 1 and 1 <= k < 65534");
  if (n > 0xFFFFFFFFull) return fail(ctx, SBDT_ERR_INVALID, "n exceeds the 32-bit PointId range");
  unsigned long long* bbox = reinterpret_cast<unsigned long long*>(d_bbox_ordered_out);
  if (!bbox) {
    SBDT_WS(tmp, unsigned long long, "capi.bbox", 6);
    bbox = tmp;
  }
  int rc = (dim == 2) ? assign_impl<2>(ctx, d_coords, n, d_sample_ids, d_sample_labels, m, d_labels_out, bbox)
                      : assign_impl<3>(ctx, d_coords, n, d_sample_ids, d_sample_labels, m, d_labels_out, bbox);
  if (rc != kOk) return rc;
  if (d_part_offsets_out && d_part_ids_out)
    return bucket_impl(ctx, d_labels_out, n, k, d_part_offsets_out, d_part_ids_out);
  return kOk;
}

// Chunked uploads for the host-buffer entry points: copies go to the
// context's copy stream in kUploadChunks pieces, each closed by an event the
// kernels wait for, so the kernels on chunk i overlap the upload of chunk
// i+1 (and the compute stream never waits for the whole input).
static constexpr int kUploadChunks = 8;

// Simplex-row chunk boundaries: the last chunks are smaller, so the kernels
// still to run after the final upload (the tail of the call) are short.
static_assert(kUploadChunks == 8, "row_chunk_end's table has 8 entries");
static uint64_t row_chunk_end(uint64_t S, int c) {
  static constexpr unsigned kCum[kUploadChunks] = {11, 22, 33, 43, 51, 57, 61, 64};  // of 64
  return c < 0 ? 0 : S * kCum[c] / 64;
}

static int prepare_chunks(sbdt_gpu_ctx* ctx) {
  if (!ctx->copy_stream) SBDT_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  if (!ctx->d2h_stream) SBDT_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
  while (ctx->chunk_events.size() < kUploadChunks + 1) {
    cudaEvent_t e;
    SBDT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->chunk_events.push_back(e);
  }
  while (ctx->chunk_done.size() < kUploadChunks) {
    cudaEvent_t e;
    SBDT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->chunk_done.push_back(e);
  }
  ctx->chunks.clear();
  return SBDT_OK;
}

// Clears the chunk state on every exit path of a host-buffer call.
struct ChunkScope {
  sbdt_gpu_ctx* ctx;
  ~ChunkScope() {
    ctx->chunks.clear();
    ctx->sample_xyz = nullptr;
    ctx->positive_host = nullptr;
    ctx->labels_host = nullptr;
  }
};

int sbdt_gpu_assign_points(sbdt_gpu_ctx* ctx, int dim, const double* coords, uint64_t n,
                           const uint32_t* sample_ids, const uint32_t* sample_labels, uint32_t m, uint32_t k,
                           uint32_t* labels_out, uint64_t* part_offsets_out, uint32_t* part_ids_out,
                           double* bbox_out) {
  if (!ctx || !coords || !sample_ids || !sample_labels || !labels_out) return SBDT_ERR_INVALID;
  ctx->res_coords = ctx->res_labels = nullptr;  // re-established on success
  cudaStream_t st = ctx->stream;
  double* d_xyz;
  uint32_t *d_sid, *d_slab, *d_lab, *d_pids = nullptr;
  uint64_t *d_poff = nullptr, *d_bbox;
  TRY(dalloc(ctx, "h.xyz", n * dim, &d_xyz));
  TRY(dalloc(ctx, "h.sid", m, &d_sid));
  TRY(dalloc(ctx, "h.slab", m, &d_slab));
  TRY(dalloc(ctx, "h.lab", n, &d_lab));
  TRY(dalloc(ctx, "h.bbox", 6, &d_bbox));
  const bool parts = part_offsets_out && part_ids_out;
  if (parts) {
    TRY(dalloc(ctx, "h.poff", k + 1, &d_poff));
    TRY(dalloc(ctx, "h.pids", n, &d_pids));
  }
  TRY(prepare_chunks(ctx));
  ChunkScope scope{ctx};
  // samples first (compact coordinates gathered here: the table build needs
  // only them), then the points in chunks on the copy stream
  double* d_sxyz;
  TRY(dalloc(ctx, "h.sxyz", std::uint64_t(m) * dim, &d_sxyz));
  for (uint32_t i = 0; i < m; ++i) {
    if (sample_ids[i] >= n) return fail(ctx, SBDT_ERR_INVALID, "sample id out of range");
    if (sample_labels[i] >= k) return fail(ctx, SBDT_ERR_INVALID, "sample label out of range (must be < k)");
  }
  // the gather is m cache misses into the caller's point array: split over
  // host threads, into a page-locked staging buffer (an async copy)
  const std::size_t sbytes = sizeof(double) * std::size_t(m) * dim;
  if (ctx->sample_stage_bytes < sbytes) {
    if (ctx->sample_stage) cudaFreeHost(ctx->sample_stage);
    ctx->sample_stage = nullptr;
    ctx->sample_stage_bytes = 0;
    SBDT_CUDA_TRY(cudaMallocHost(&ctx->sample_stage, sbytes));
    ctx->sample_stage_bytes = sbytes;
  }
  SBDT_CUDA_TRY(cudaStreamSynchronize(st));  // the previous call's copy out of the staging buffer is done
  double* sxyz = static_cast<double*>(ctx->sample_stage);
  {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned nt = m < 16384 ? 1u : std::min(16u, hw ? hw : 1u);
    auto work = [&](unsigned t) {
      const uint32_t a = static_cast<uint32_t>(std::uint64_t(m) * t / nt),
                     b = static_cast<uint32_t>(std::uint64_t(m) * (t + 1) / nt);
      for (uint32_t i = a; i < b; ++i)
        for (int d = 0; d < dim; ++d) sxyz[std::size_t(i) * dim + d] = coords[std::size_t(sample_ids[i]) * dim + d];
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  SBDT_CUDA_TRY(cudaMemcpyAsync(d_sxyz, sxyz, sbytes, cudaMemcpyHostToDevice, st));
  SBDT_CUDA_TRY(cudaMemcpyAsync(d_sid, sample_ids, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, st));
  SBDT_CUDA_TRY(cudaMemcpyAsync(d_slab, sample_labels, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, st));
  ctx->sample_xyz = d_sxyz;
  for (int c = 0; c < kUploadChunks; ++c) {
    const uint64_t i0 = n * c / kUploadChunks, i1 = n * (c + 1) / kUploadChunks;
    if (i1 > i0)
      SBDT_CUDA_TRY(cudaMemcpyAsync(d_xyz + i0 * dim, coords + i0 * dim, sizeof(double) * (i1 - i0) * dim,
                                    cudaMemcpyHostToDevice, ctx->copy_stream));
    SBDT_CUDA_TRY(cudaEventRecord(ctx->chunk_events[c], ctx->copy_stream));
    ctx->chunks.emplace_back(i1, ctx->chunk_events[c]);
  }
  ctx->labels_host = labels_out;  // streamed per chunk by assign_impl
  TRY(sbdt_gpu_assign_points_dev(ctx, dim, d_xyz, n, d_sid, d_slab, m, k, d_lab, d_poff, d_pids, d_bbox));
  if (parts) {
    SBDT_CUDA_TRY(cudaMemcpyAsync(part_offsets_out, d_poff, sizeof(uint64_t) * (k + 1), cudaMemcpyDeviceToHost, st));
    SBDT_CUDA_TRY(cudaMemcpyAsync(part_ids_out, d_pids, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, st));
  }
  unsigned long long hb[6] = {0, 0, 0, 0, 0, 0};
  if (bbox_out) SBDT_CUDA_TRY(cudaMemcpyAsync(hb, d_bbox, sizeof(uint64_t) * 2 * dim, cudaMemcpyDeviceToHost, st));
  TRY(finish(ctx));
  SBDT_CUDA_TRY(cudaStreamSynchronize(ctx->d2h_stream));
  if (bbox_out)
    for (int i = 0; i < 2 * dim; ++i) bbox_out[i] = ordered_to_dbl(hb[i]);
  ctx->res_coords = coords;
  ctx->res_labels = labels_out;
  ctx->res_n = n;
  ctx->res_dim = dim;
  ctx->res_bbox = true;
  return SBDT_OK;
}

int sbdt_gpu_find_border_dev(sbdt_gpu_ctx* ctx, const sbdt_border_args* a) {
  if (!ctx || !a) return SBDT_ERR_INVALID;
  if (a->dim != 2 && a->dim != 3) return fail(ctx, SBDT_ERR_INVALID, "dim must be 2 or 3");
  if (a->k == 0 || a->k >= 0xFFFE) return fail(ctx, SBDT_ERR_INVALID, "need 1 <= k < 65534");
  if (a->policy != SBDT_POLICY_BBOX && a->policy != SBDT_POLICY_GRID && a->policy != SBDT_POLICY_EXACT)
    return fail(ctx, SBDT_ERR_INVALID, "unknown intersection policy");
  if (!a->d_positive || !a->d_vertex_flags || !a->d_vertex_ids || !a->d_vertex_count)
    return fail(ctx, SBDT_ERR_INVALID, "missing output buffers");
  if (a->S > 0xFFFFFFFFull) return fail(ctx, SBDT_ERR_INVALID, "S exceeds the 32-bit SimplexId range");
  int rc = (a->dim == 2) ? border_impl<2>(ctx, a) : border_impl<3>(ctx, a);
  if (rc != kOk) return rc;
  if ((a->flags & SBDT_BORDER_HULL_BFS) && a->d_border) return reach_impl(ctx, a);
  return kOk;
}

namespace {
int find_border_host(sbdt_gpu_ctx* ctx, int dim, const double* coords, uint64_t n, const uint32_t* labels,
                     uint32_t k, const uint64_t* offsets, const uint32_t* verts, const uint32_t* nbrs,
                     const int8_t* parity, int policy, double c_G, uint32_t flags, uint8_t* positive_out,
                     uint8_t* border_out, uint32_t* vertex_ids_out, uint64_t* n_vertices_out,
                     uint32_t* bfs_vertex_ids_out, uint64_t* n_bfs_vertices_out, double* spheres_out,
                     const double* grid_bbox, uint64_t grid_n_total, uint64_t grid_max_cells) {
  if (!ctx || !coords || !labels || !offsets || !verts || !nbrs || (!parity && policy == SBDT_POLICY_EXACT) ||
      !positive_out || !vertex_ids_out || !n_vertices_out)
    return SBDT_ERR_INVALID;
  if (dim != 2 && dim != 3) return fail(ctx, SBDT_ERR_INVALID, "dim must be 2 or 3");
  const uint64_t S = offsets[k];
  cudaStream_t st = ctx->stream;
  sbdt_border_args a{};
  a.dim = dim;
  a.n = n;
  a.k = k;
  a.S = S;
  a.policy = policy;
  a.c_G = c_G;
  a.flags = flags;
  a.grid_bbox = grid_bbox;
  a.grid_n_total = grid_n_total;
  a.grid_max_cells = grid_max_cells;
  double* d_xyz;
  uint32_t *d_lab, *d_verts, *d_nbrs, *d_vids, *d_bvids = nullptr;
  uint64_t *d_off, *d_cnt, *d_bcnt = nullptr;
  int8_t* d_par;
  uint8_t *d_pos, *d_bor = nullptr, *d_vf, *d_bvf = nullptr;
  double* d_sph = nullptr;
  TRY(dalloc(ctx, "h.xyz", n * dim, &d_xyz));
  TRY(dalloc(ctx, "h.lab", n, &d_lab));
  TRY(dalloc(ctx, "h.off", k + 1, &d_off));
  TRY(dalloc(ctx, "h.verts", S * (dim + 1), &d_verts));
  const bool bfs = (flags & SBDT_BORDER_HULL_BFS) && border_out;
  TRY(dalloc(ctx, "h.nbrs", S * (dim + 1), &d_nbrs));
  TRY(dalloc(ctx, "h.par", S, &d_par));
  TRY(dalloc(ctx, "h.pos", S, &d_pos));
  TRY(dalloc(ctx, "h.vf", n + 64, &d_vf));
  TRY(dalloc(ctx, "h.vids", n, &d_vids));
  TRY(dalloc(ctx, "h.cnt", 1, &d_cnt));
  if (bfs) {
    TRY(dalloc(ctx, "h.bor", S, &d_bor));
    TRY(dalloc(ctx, "h.bvf", n + 64, &d_bvf));
    TRY(dalloc(ctx, "h.bvids", n, &d_bvids));
    TRY(dalloc(ctx, "h.bcnt", 1, &d_bcnt));
  }
  if (spheres_out) TRY(dalloc(ctx, "h.sph", S * (dim + 1), &d_sph));
  TRY(prepare_chunks(ctx));
  ChunkScope scope{ctx};
  cudaStream_t cs = ctx->copy_stream;
  // points, labels and part offsets first (the owner grid needs them), then
  // the simplex rows in chunks; everything on the copy stream, in order
  const bool resident = (flags & SBDT_BORDER_RESIDENT_POINTS) != 0;
  if (resident) {
    if (ctx->res_coords != coords || ctx->res_labels != labels || ctx->res_n != n || ctx->res_dim != dim)
      return fail(ctx, SBDT_ERR_INVALID, "RESIDENT_POINTS: coords/labels are not those of the last assign_points call");
    if (ctx->res_bbox) {
      uint64_t* d_bb;
      TRY(dalloc(ctx, "h.bbox", 6, &d_bb));
      a.d_bbox_ordered = d_bb;  // written by that assign_points call
    }
  } else {
    SBDT_CUDA_TRY(cudaMemcpyAsync(d_xyz, coords, sizeof(double) * n * dim, cudaMemcpyHostToDevice, cs));
    SBDT_CUDA_TRY(cudaMemcpyAsync(d_lab, labels, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, cs));
    ctx->res_coords = coords;
    ctx->res_labels = labels;
    ctx->res_n = n;
    ctx->res_dim = dim;
    ctx->res_bbox = false;
  }
  SBDT_CUDA_TRY(cudaMemcpyAsync(d_off, offsets, sizeof(uint64_t) * (k + 1), cudaMemcpyHostToDevice, cs));
  SBDT_CUDA_TRY(cudaEventRecord(ctx->chunk_events[kUploadChunks], cs));
  SBDT_CUDA_TRY(cudaStreamWaitEvent(st, ctx->chunk_events[kUploadChunks], 0));
  // Without the BFS the ~1% hull rows read one neighbour each: a page-locked
  // caller buffer is mapped into the device address space and read in place
  // instead of uploading a whole SoA row.
  const uint32_t* nbrs_mapped = nullptr;
  if (!bfs) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, nbrs) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      nbrs_mapped = static_cast<const uint32_t*>(pa.devicePointer);
    else
      cudaGetLastError();  // pageable: clear the error, upload the row
  }
  for (int c = 0; c < kUploadChunks; ++c) {
    const uint64_t r0 = row_chunk_end(S, c - 1), r1 = row_chunk_end(S, c);
    if (r1 > r0 && ctx->fill && ctx->fill(ctx->fill_user, SBDT_FILL_ROWS, r0, r1) != 0)
      return fail(ctx, SBDT_ERR_INVALID, "fill hook failed");
    if (r1 > r0) {
      for (int j = 0; j <= dim; ++j)
        SBDT_CUDA_TRY(cudaMemcpyAsync(d_verts + j * S + r0, verts + j * S + r0, sizeof(uint32_t) * (r1 - r0),
                                      cudaMemcpyHostToDevice, cs));
      // parity orients in_sphere (exact policy only); the other policies
      // check degeneracy geometrically and never read it
      if (policy == SBDT_POLICY_EXACT)
        SBDT_CUDA_TRY(cudaMemcpyAsync(d_par + r0, parity + r0, r1 - r0, cudaMemcpyHostToDevice, cs));
      // without the BFS only the hull rows' last neighbour (the finite
      // simplex across the hull facet, row dim of the SoA) is read, and from
      // a page-locked caller buffer it is read in place (zero-copy)
      if (!nbrs_mapped)
        for (int j = bfs ? 0 : dim; j <= dim; ++j)
          SBDT_CUDA_TRY(cudaMemcpyAsync(d_nbrs + j * S + r0, nbrs + j * S + r0, sizeof(uint32_t) * (r1 - r0),
                                        cudaMemcpyHostToDevice, cs));
    }
    SBDT_CUDA_TRY(cudaEventRecord(ctx->chunk_events[c], cs));
    ctx->chunks.emplace_back(r1, ctx->chunk_events[c]);
  }

  a.d_xyz = d_xyz;
  a.d_labels = d_lab;
  a.d_offsets = d_off;
  a.d_verts = d_verts;
  a.d_nbrs = nbrs_mapped ? nbrs_mapped : d_nbrs;
  a.d_parity = d_par;
  a.d_positive = d_pos;
  a.d_border = d_bor;
  a.d_vertex_flags = d_vf;
  a.d_vertex_ids = d_vids;
  a.d_vertex_count = d_cnt;
  a.d_bfs_vertex_flags = d_bvf;
  a.d_bfs_vertex_ids = d_bvids;
  a.d_bfs_vertex_count = d_bcnt;
  a.d_spheres = d_sph;
  const bool streamed = policy == SBDT_POLICY_GRID;  // border_impl streams the flags per chunk
  ctx->positive_host = streamed ? positive_out : nullptr;
  TRY(sbdt_gpu_find_border_dev(ctx, &a));
  uint64_t nv = 0, nb = 0;
  if (!streamed) SBDT_CUDA_TRY(cudaMemcpyAsync(positive_out, d_pos, S, cudaMemcpyDeviceToHost, st));
  SBDT_CUDA_TRY(cudaMemcpyAsync(&nv, d_cnt, 8, cudaMemcpyDeviceToHost, st));
  if (bfs) {
    SBDT_CUDA_TRY(cudaMemcpyAsync(border_out, d_bor, S, cudaMemcpyDeviceToHost, st));
    SBDT_CUDA_TRY(cudaMemcpyAsync(&nb, d_bcnt, 8, cudaMemcpyDeviceToHost, st));
  }
  if (spheres_out)
    SBDT_CUDA_TRY(cudaMemcpyAsync(spheres_out, d_sph, sizeof(double) * S * (dim + 1), cudaMemcpyDeviceToHost, st));
  TRY(finish(ctx));
  if (streamed) SBDT_CUDA_TRY(cudaStreamSynchronize(ctx->d2h_stream));
  SBDT_CUDA_TRY(cudaMemcpy(vertex_ids_out, d_vids, sizeof(uint32_t) * nv, cudaMemcpyDeviceToHost));
  *n_vertices_out = nv;
  if (bfs) {
    if (bfs_vertex_ids_out) SBDT_CUDA_TRY(cudaMemcpy(bfs_vertex_ids_out, d_bvids, sizeof(uint32_t) * nb, cudaMemcpyDeviceToHost));
    if (n_bfs_vertices_out) *n_bfs_vertices_out = nb;
  }
  return SBDT_OK;
}
}  // namespace

int sbdt_gpu_find_border(sbdt_gpu_ctx* ctx, int dim, const double* coords, uint64_t n, const uint32_t* labels,
                         uint32_t k, const uint64_t* offsets, const uint32_t* verts, const uint32_t* nbrs,
                         const int8_t* parity, int policy, double c_G, uint32_t flags, uint8_t* positive_out,
                         uint8_t* border_out, uint32_t* vertex_ids_out, uint64_t* n_vertices_out,
                         uint32_t* bfs_vertex_ids_out, uint64_t* n_bfs_vertices_out, double* spheres_out,
                         const double* grid_bbox, uint64_t grid_n_total) {
  int rc = find_border_host(ctx, dim, coords, n, labels, k, offsets, verts, nbrs, parity, policy, c_G, flags,
                            positive_out, border_out, vertex_ids_out, n_vertices_out, bfs_vertex_ids_out,
                            n_bfs_vertices_out, spheres_out, grid_bbox, grid_n_total, 0);
  if (rc != SBDT_ERR_RANGE || !ctx) return rc;
  // A bbox far from cubical needs more cells than the default 4 n / c_G^dim
  // capacity: retry once with what the grid needs (bounded), instead of
  // rejecting an input the reference's sparse GridIndex accepts.
  auto it = ctx->bufs.find("border.og");
  if (it == ctx->bufs.end()) return rc;
  unsigned long long need[2] = {0, 0};
  const std::size_t off = dim == 2 ? offsetof(OwnerGrid<2>, need_cells) : offsetof(OwnerGrid<3>, need_cells);
  if (cudaMemcpy(need, static_cast<char*>(it->second.ptr) + off, sizeof(need), cudaMemcpyDeviceToHost) != cudaSuccess)
    return rc;
  const unsigned long long want = need[0] > need[1] ? need[0] : need[1];
  if (need[0] == 0 || want > (1ull << 31)) return rc;
  return find_border_host(ctx, dim, coords, n, labels, k, offsets, verts, nbrs, parity, policy, c_G, flags,
                          positive_out, border_out, vertex_ids_out, n_vertices_out, bfs_vertex_ids_out,
                          n_bfs_vertices_out, spheres_out, grid_bbox, grid_n_total, want + 4096);
}

namespace {
int merge_checks(sbdt_gpu_ctx* ctx, const sbdt_merge_args* a, uint64_t capacity, const void* ov, const void* on,
                 const void* op, const void* oo, uint64_t* rows_out) {
  if (!a || !ov || !on || !op || !oo || !rows_out) return fail(ctx, SBDT_ERR_INVALID, "merge: null argument");
  if (a->dim != 2 && a->dim != 3) return fail(ctx, SBDT_ERR_INVALID, "dim must be 2 or 3");
  if (a->k == 0) return fail(ctx, SBDT_ERR_INVALID, "merge: k must be >= 1");
  if ((a->S && (!a->d_verts || !a->d_nbrs || !a->d_parity || !a->d_border)) ||
      (a->S_B && (!a->d_tb_verts || !a->d_tb_nbrs || !a->d_tb_parity || !a->d_labels)) || !a->d_offsets)
    return fail(ctx, SBDT_ERR_INVALID, "merge: null input array");
  if (a->S > 0xFFFFFFFFull || a->S_B > 0xFFFFFFFFull || capacity > 0xFFFFFFFFull)
    return fail(ctx, SBDT_ERR_INVALID, "merge: more than 2^32 rows");
  return kOk;
}
}  // namespace

int sbdt_gpu_merge_dev(sbdt_gpu_ctx* ctx, const sbdt_merge_args* args, uint64_t capacity, uint32_t* d_out_verts,
                       uint32_t* d_out_nbrs, int8_t* d_out_parity, uint64_t* d_out_offsets, uint64_t* rows_out) {
  if (!ctx) return SBDT_ERR_INVALID;
  TRY(merge_checks(ctx, args, capacity, d_out_verts, d_out_nbrs, d_out_parity, d_out_offsets, rows_out));
  *rows_out = 0;
  const int rc = args->dim == 2 ? merge_impl<2>(ctx, args, capacity, d_out_verts, d_out_nbrs, d_out_parity,
                                                d_out_offsets, rows_out)
                                : merge_impl<3>(ctx, args, capacity, d_out_verts, d_out_nbrs, d_out_parity,
                                                d_out_offsets, rows_out);
  if (rc != kOk) return rc;
  return finish(ctx);
}

int sbdt_gpu_merge(sbdt_gpu_ctx* ctx, int dim, const uint32_t* labels, uint64_t n, uint32_t k,
                   const uint64_t* offsets, const uint32_t* verts, const uint32_t* nbrs, const int8_t* parity,
                   const uint8_t* border, const uint32_t* tb_verts, const uint32_t* tb_nbrs,
                   const int8_t* tb_parity, uint64_t S_B, uint32_t flags, uint64_t capacity,
                   uint32_t* out_verts, uint32_t* out_nbrs, int8_t* out_parity, uint64_t* out_offsets,
                   uint64_t* rows_out) {
  if (!ctx) return SBDT_ERR_INVALID;
  if (!offsets || k == 0) return fail(ctx, SBDT_ERR_INVALID, "merge: offsets / k");
  sbdt_merge_args a{};
  a.dim = dim;
  a.k = k;
  a.n = n;
  a.S = offsets[k];
  a.S_B = S_B;
  a.flags = flags;
  // host pointers stand in for the checks; replaced by device copies below
  a.d_labels = labels;
  a.d_offsets = offsets;
  a.d_verts = verts;
  a.d_nbrs = nbrs;
  a.d_parity = parity;
  a.d_border = border;
  a.d_tb_verts = tb_verts;
  a.d_tb_nbrs = tb_nbrs;
  a.d_tb_parity = tb_parity;
  TRY(merge_checks(ctx, &a, capacity, out_verts, out_nbrs, out_parity, out_offsets, rows_out));
  *rows_out = 0;
  const uint64_t S = a.S, D1 = dim + 1;
  uint32_t *d_lab, *d_verts, *d_nbrs, *d_tbv, *d_tbn, *d_ov, *d_on;
  uint64_t *d_off, *d_oo;
  int8_t *d_par, *d_tbp, *d_op;
  uint8_t* d_bor;
  TRY(dalloc(ctx, "m.lab", n, &d_lab));
  TRY(dalloc(ctx, "m.off", k + 1, &d_off));
  TRY(dalloc(ctx, "m.verts", S * D1, &d_verts));
  TRY(dalloc(ctx, "m.nbrs", S * D1, &d_nbrs));
  TRY(dalloc(ctx, "m.par", S, &d_par));
  TRY(dalloc(ctx, "m.bor", S, &d_bor));
  TRY(dalloc(ctx, "m.tbv", S_B * D1, &d_tbv));
  TRY(dalloc(ctx, "m.tbn", S_B * D1, &d_tbn));
  TRY(dalloc(ctx, "m.tbp", S_B, &d_tbp));
  TRY(dalloc(ctx, "m.ov", capacity * D1, &d_ov));
  TRY(dalloc(ctx, "m.on", capacity * D1, &d_on));
  TRY(dalloc(ctx, "m.op", capacity, &d_op));
  TRY(dalloc(ctx, "m.oo", k + 3, &d_oo));
  cudaStream_t st = ctx->stream;
  auto up = [&](void* d, const void* h, std::size_t bytes) {
    return bytes ? cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st) : cudaSuccess;
  };
  SBDT_CUDA_TRY(up(d_off, offsets, 8 * (k + 1)));
  SBDT_CUDA_TRY(up(d_verts, verts, 4 * S * D1));
  SBDT_CUDA_TRY(up(d_nbrs, nbrs, 4 * S * D1));
  SBDT_CUDA_TRY(up(d_par, parity, S));
  SBDT_CUDA_TRY(up(d_bor, border, S));
  if (S_B) {
    SBDT_CUDA_TRY(up(d_lab, labels, 4 * n));
    SBDT_CUDA_TRY(up(d_tbv, tb_verts, 4 * S_B * D1));
    SBDT_CUDA_TRY(up(d_tbn, tb_nbrs, 4 * S_B * D1));
    SBDT_CUDA_TRY(up(d_tbp, tb_parity, S_B));
  }
  a.d_labels = d_lab;
  a.d_offsets = d_off;
  a.d_verts = d_verts;
  a.d_nbrs = d_nbrs;
  a.d_parity = d_par;
  a.d_border = d_bor;
  a.d_tb_verts = d_tbv;
  a.d_tb_nbrs = d_tbn;
  a.d_tb_parity = d_tbp;
  uint64_t rows = 0;
  const int rc = dim == 2 ? merge_impl<2>(ctx, &a, capacity, d_ov, d_on, d_op, d_oo, &rows)
                          : merge_impl<3>(ctx, &a, capacity, d_ov, d_on, d_op, d_oo, &rows);
  *rows_out = rows;
  if (rc != kOk) return rc;
  TRY(sbdt_gpu_check_status(ctx));
  for (uint64_t j = 0; j < D1 && rows; ++j) {
    SBDT_CUDA_TRY(cudaMemcpyAsync(out_verts + j * rows, d_ov + j * capacity, 4 * rows, cudaMemcpyDeviceToHost, st));
    SBDT_CUDA_TRY(cudaMemcpyAsync(out_nbrs + j * rows, d_on + j * capacity, 4 * rows, cudaMemcpyDeviceToHost, st));
  }
  if (rows) SBDT_CUDA_TRY(cudaMemcpyAsync(out_parity, d_op, rows, cudaMemcpyDeviceToHost, st));
  SBDT_CUDA_TRY(cudaMemcpyAsync(out_offsets, d_oo, 8 * (k + 3), cudaMemcpyDeviceToHost, st));
  return finish(ctx);
}

}  // extern "C"
