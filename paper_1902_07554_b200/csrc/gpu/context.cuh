// Device context owned by the C ABI: stream, grow-only workspace, error word.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "sbdt_gpu.h"

struct sbdt_gpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  sbdt_fill_fn fill = nullptr;  // find_border's row producer (sbdt_gpu_set_fill)
  unsigned attr_set = 0;        // kernels whose shared-memory opt-in was set on this device (bit D: k_field_tiles<D>)
  void* fill_user = nullptr;
  std::string last_error;
  unsigned long long launches = 0;
  struct Buf {
    void* ptr = nullptr;
    std::size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs;
  // device-side status word: bit0 degenerate simplex, bit1 grid cap exceeded,
  // bit2 escalation overflow
  unsigned* d_status = nullptr;
  // last find_border statistics (read back by the host after a call)
  unsigned long long stats[8] = {0};
  // optional per-stage CUDA-event timing (bench.py: live per-kernel durations)
  bool timing = false;
  // optional pipeline census (counters; adds atomics, so never in a timed run)
  bool census = false;
  struct Stage {
    std::string name;
    cudaEvent_t start = nullptr, stop = nullptr;
  };
  std::vector<Stage> stages;
  std::vector<cudaEvent_t> event_pool;
  std::size_t events_used = 0;
  // host-buffer entry points: uploads run on copy_stream in chunks; chunk i
  // (points / simplex rows below chunks[i].first) is resident once
  // chunks[i].second has completed. Empty for the *_dev entry points.
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> chunk_events;
  std::vector<std::pair<std::uint64_t, cudaEvent_t>> chunks;
  const double* sample_xyz = nullptr;  // compact sample coordinates (host path), else gathered from the points
  void* sample_stage = nullptr;        // page-locked host staging of those (grow-only)
  std::size_t sample_stage_bytes = 0;
  // host path: positive flags streamed back per chunk on d2h_stream
  std::uint8_t* positive_host = nullptr;
  std::uint32_t* labels_host = nullptr;  // assign_points: labels streamed back per chunk
  cudaStream_t d2h_stream = nullptr;
  // device path: work off the critical path (the hull rows' halfspace kernel)
  // runs on side_stream between fork/join events
  cudaStream_t side_stream = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // the prefilter-routed wide rows (k_border_wide) next to the exact stage
  cudaStream_t wide_stream = nullptr;
  cudaEvent_t wide_join_ev = nullptr;
  std::vector<cudaEvent_t> chunk_done;
  // host buffers whose device copies ("h.xyz", "h.lab", "h.bbox") are current
  // (SBDT_BORDER_RESIDENT_POINTS)
  const void* res_coords = nullptr;
  const void* res_labels = nullptr;
  std::uint64_t res_n = 0;
  int res_dim = 0;
  bool res_bbox = false;
};

namespace sbdt_gpu {

enum Status : int {
  kOk = 0,
  kErrInvalid = 1,
  kErrDegenerate = 2,
  kErrCuda = 3,
  kErrOom = 4,
  kErrRange = 5,
};

enum DeviceStatusBits : unsigned {
  kStDegenerate = 1u,
  kStGridCap = 2u,
  kStQueueOverflow = 4u,
  // 8, 16: merge (InconsistentMerge, DanglingFacet)
  kStLabelRange = 32u,  // a sample label >= k (device-pointer assign path)
};

// find_border census counters (sbdt_gpu_border_stats, census mode only):
//  0 rows, 1 exact-stage rows, 2 flat scans, 3 two-level, 4 pyramid,
//  5 (row, cell row) pairs, 6 pyramid expansions, 7 exact-stage binary32
//  positives, 8 prefilter positives, 9 wide positives, 10 (unused),
//  11 queue holes, then the predicate escalations:
enum BorderCounter : int {
  kCtrOrientRows = 12,     // rows whose binary32 sphere failed: exact orientation checked
  kCtrOrientExact = 13,    // orient evaluations escalated to expansion arithmetic
  kCtrInSphereExact = 14,  // in_sphere tests escalated (exact policy, k_border_escalate)
  kBorderCounters = 20,
};

inline int fail(sbdt_gpu_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->last_error = msg;
  return code;
}
inline int fail_cuda(sbdt_gpu_ctx* ctx, cudaError_t e, const char* what) {
  const int code = (e == cudaErrorMemoryAllocation) ? kErrOom : kErrCuda;
  return fail(ctx, code, std::string(what) + ": " + cudaGetErrorString(e));
}

// Grow-only named workspace buffer (contents undefined on growth).
inline void* workspace(sbdt_gpu_ctx* ctx, const char* name, std::size_t bytes, cudaError_t* err) {
  auto& b = ctx->bufs[name];
  if (b.bytes >= bytes && b.ptr) return b.ptr;
  if (b.ptr) cudaFree(b.ptr);
  b.ptr = nullptr;
  b.bytes = 0;
  std::size_t want = bytes + bytes / 8 + 256;
  cudaError_t e = cudaMalloc(&b.ptr, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *err = e;
    return nullptr;
  }
  b.bytes = want;
  return b.ptr;
}

inline cudaEvent_t pooled_event(sbdt_gpu_ctx* ctx) {
  if (ctx->events_used == ctx->event_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->event_pool.push_back(e);
  }
  return ctx->event_pool[ctx->events_used++];
}

// RAII stage marker: records events around the enclosed launches when timing is on.
struct StageTimer {
  sbdt_gpu_ctx* ctx;
  std::size_t idx = static_cast<std::size_t>(-1);
  cudaStream_t stream;
  StageTimer(sbdt_gpu_ctx* c, const char* name, cudaStream_t on = nullptr) : ctx(c), stream(on ? on : c->stream) {
    if (!ctx->timing) return;
    sbdt_gpu_ctx::Stage s;
    s.name = name;
    s.start = pooled_event(ctx);
    s.stop = pooled_event(ctx);
    cudaEventRecord(s.start, stream);
    idx = ctx->stages.size();
    ctx->stages.push_back(s);
  }
  void end() {
    if (idx != static_cast<std::size_t>(-1)) cudaEventRecord(ctx->stages[idx].stop, stream);
    idx = static_cast<std::size_t>(-1);
  }
  ~StageTimer() { end(); }
};

}  // namespace sbdt_gpu

#define SBDT_WS(var, type, name, count)                                                         \
  type* var = nullptr;                                                                          \
  do {                                                                                          \
    cudaError_t e_ = cudaSuccess;                                                               \
    var = static_cast<type*>(::sbdt_gpu::workspace(ctx, name, sizeof(type) * (std::size_t)(count), &e_)); \
    if (!var) return ::sbdt_gpu::fail_cuda(ctx, e_, "workspace " name);                        \
  } while (0)
