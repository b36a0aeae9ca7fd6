// sbdt/sample_partition.hpp — drop-in `assign_points` for the reference's
// sample-partition module, backed by the sm_100a kernels
// of libsbdt_gpu.so through the C ABI in sbdt_gpu.h.
//
// The reference declares this operation only in its SPEC (the source
// sample_partition.cpp listed at proj/src/CMakeLists.txt:6 does not ship,
// SURVEY.md F1/F2). This header gives it the SPEC's signature with the
// conventions of the shipped headers (proj/include/sbdt/*.hpp): namespace
// sbdt, D in {2,3} as a template parameter, uint32 ids, std::span inputs,
// return by value, an optional TaskPool* (host-side data movement only: the
// work runs on the GPU),
// errors as the reference's exception types (common.hpp:22-65).
//
// Drop into the reference tree next to proj/include/sbdt/geometry.hpp and
// link libsbdt_gpu.so.
#pragma once

#include <chrono>
#include <cstring>
#include <thread>
#include <cstdint>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sbdt/common.hpp"
#include "sbdt/geometry.hpp"
#include "sbdt/task_pool.hpp"
#include "sbdt_gpu.h"

namespace sbdt {

// SPEC.md:307-312
struct Partitioning {
  std::vector<PartitionId> labels;          // per input point, in [0, k)
  std::vector<std::vector<PointId>> parts;  // k lists, ascending point ids
  std::vector<PointId> sample_point_ids;
  std::vector<PartitionId> sample_labels;
};

namespace gpu_detail {

// Wall-clock phases of the last drop-in call on this thread (diagnostics for
// the drop-in benchmark): host preparation, the C ABI call (H2D, kernels,
// D2H), host post-processing.
struct PhaseTimes {
  double prepare_ms = 0, device_ms = 0, finish_ms = 0;
};
inline PhaseTimes& last_phases() {
  thread_local PhaseTimes t;
  return t;
}
inline double wall_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Thread-local grow-only page-locked staging (sbdt_gpu_host_alloc): buffers
// written / read here cross PCIe at full rate.
struct PinnedSlot {
  void* p = nullptr;
  std::size_t bytes = 0;
  PinnedSlot() = default;
  PinnedSlot(const PinnedSlot&) = delete;
  PinnedSlot& operator=(const PinnedSlot&) = delete;
  ~PinnedSlot() {
    if (p) sbdt_gpu_host_free(p);
  }
  template <class T>
  T* get(std::size_t count) {
    const std::size_t want = sizeof(T) * (count ? count : 1);
    if (want > bytes) {
      if (p) sbdt_gpu_host_free(p);
      p = nullptr;
      bytes = 0;
      if (sbdt_gpu_host_alloc(want, &p) != SBDT_OK) throw std::bad_alloc();
      bytes = want;
    }
    return static_cast<T*>(p);
  }
};
inline PinnedSlot& pinned_slot(int which) {
  thread_local PinnedSlot slots[16];
  return slots[which];
}

// fn(p) for p in [0, k): on the caller's TaskPool (the reference's,
// task_pool.hpp:63-80) when it has workers, else inline. Only used for pure
// data movement, so results never depend on it.
template <class Fn>
void for_each_part(TaskPool* pool, std::size_t k, Fn&& fn) {
  if (pool && pool->concurrency() > 1 && k > 1) {
    pool->parallel_for(k, 1, [&](std::size_t b, std::size_t e) {
      for (std::size_t p = b; p < e; ++p) fn(p);
    });
  } else {
    for (std::size_t p = 0; p < k; ++p) fn(p);
  }
}

// fn(b, e) over [0, n) in chunks of `grain`, on the caller's TaskPool when it
// has workers (pure data movement).
template <class Fn>
void for_each_chunk(TaskPool* pool, std::size_t n, std::size_t grain, Fn&& fn) {
  if (pool && pool->concurrency() > 1 && n > grain) {
    pool->parallel_for(n, grain, [&](std::size_t b, std::size_t e) { fn(b, e); });
  } else if (n) {
    fn(0, n);
  }
}

// The points and labels of the last assign_points call on this thread and
// the page-locked copies the C ABI saw (find_border with points_resident).
struct ResidentRecord {
  const double* coords = nullptr;
  std::uint64_t n = 0;
  const PartitionId* labels = nullptr;
  const double* staged_coords = nullptr;
  const std::uint32_t* staged_labels = nullptr;
};
inline ResidentRecord& resident() {
  thread_local ResidentRecord r;
  return r;
}

// One device context per host thread (the C ABI contract).
inline sbdt_gpu_ctx* thread_context() {
  struct Holder {
    sbdt_gpu_ctx* ctx = nullptr;
    ~Holder() {
      if (ctx) sbdt_gpu_destroy(ctx);
    }
  };
  thread_local Holder h;
  if (!h.ctx) {
    const int rc = sbdt_gpu_create(0, &h.ctx);
    if (rc != SBDT_OK) throw std::runtime_error("sbdt_gpu_create failed (status " + std::to_string(rc) + ")");
  }
  return h.ctx;
}

// Status code -> the reference's exception types.
inline void check(sbdt_gpu_ctx* ctx, int rc, const char* what) {
  if (rc == SBDT_OK) return;
  const std::string msg = std::string(what) + ": " + sbdt_gpu_last_error(ctx);
  switch (rc) {
    case SBDT_ERR_DEGENERATE:
      throw DegenerateSimplex(msg);
    case SBDT_ERR_INVALID:
      throw std::invalid_argument(msg);
    case SBDT_ERR_OOM:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(msg);
  }
}

}  // namespace gpu_detail

// each input point is labelled with the label of its
// Euclidean-nearest sample point (squared_distance, geometry.hpp:102-110);
// ties go to the lowest sample point id. Bit-identical to a brute-force scan.
template <int D>
Partitioning assign_points(const PointSet& points, std::span<const PointId> sample_ids,
                           std::span<const PartitionId> sample_labels, PartitionId k, TaskPool* pool = nullptr) {
  static_assert(D == 2 || D == 3, "D must be 2 or 3");
  if (points.dim() != D) throw std::invalid_argument("assign_points: PointSet dimension mismatch");
  if (sample_ids.size() != sample_labels.size() || sample_ids.empty())
    throw std::invalid_argument("assign_points: every sample point must be labelled");
  for (PartitionId l : sample_labels)
    if (l >= k) throw std::invalid_argument("assign_points: sample label >= k");
  const std::uint64_t n = points.size();
  gpu_detail::PhaseTimes& ph = gpu_detail::last_phases();
  const double t0 = gpu_detail::wall_ms();
  Partitioning out;
  // the labels vector is value-initialised by resize: done by a helper thread
  // while the coordinates are staged and the device works
  std::thread labels_init([&] { out.labels.resize(n); });
  struct Join {
    std::thread& t;
    ~Join() {
      if (t.joinable()) t.join();
    }
  } join{labels_init};
  out.sample_point_ids.assign(sample_ids.begin(), sample_ids.end());
  out.sample_labels.assign(sample_labels.begin(), sample_labels.end());
  // the coordinates go through page-locked staging (copied by the pool's
  // threads; a pageable source would be staged by the driver at a fraction of
  // the link rate), the labels and parts come back into page-locked staging
  double* xyz = gpu_detail::pinned_slot(2).get<double>(n * D);
  std::uint32_t* lab = gpu_detail::pinned_slot(3).get<std::uint32_t>(n);
  std::uint64_t* offsets = gpu_detail::pinned_slot(0).get<std::uint64_t>(k + 1);
  std::uint32_t* ids = gpu_detail::pinned_slot(1).get<std::uint32_t>(n);
  const double* src = points.raw().data();
  gpu_detail::for_each_chunk(pool, n * D, std::size_t(1) << 19, [&](std::size_t b, std::size_t e) {
    std::memcpy(xyz + b, src + b, sizeof(double) * (e - b));
  });
  sbdt_gpu_ctx* ctx = gpu_detail::thread_context();
  const double t1 = gpu_detail::wall_ms();
  gpu_detail::check(ctx,
                    sbdt_gpu_assign_points(ctx, D, xyz, n, sample_ids.data(), sample_labels.data(),
                                           static_cast<std::uint32_t>(sample_ids.size()), k, lab, offsets, ids,
                                           nullptr),
                    "assign_points");
  const double t2 = gpu_detail::wall_ms();
  labels_init.join();
  gpu_detail::for_each_chunk(pool, n, std::size_t(1) << 20, [&](std::size_t b, std::size_t e) {
    std::memcpy(out.labels.data() + b, lab + b, sizeof(std::uint32_t) * (e - b));
  });
  out.parts.resize(k);
  gpu_detail::for_each_part(pool, k, [&](std::size_t p) {
    out.parts[p].assign(ids + offsets[p], ids + offsets[p + 1]);
  });
  // find_border(points_resident) on these points and labels reuses the
  // device copies: it is handed the staging pointers this call used
  gpu_detail::resident() = {src, n, out.labels.data(), xyz, lab};
  ph.prepare_ms = t1 - t0, ph.device_ms = t2 - t1, ph.finish_ms = gpu_detail::wall_ms() - t2;
  return out;
}

}  // namespace sbdt
