// sbdt/sample_partition.hpp — drop-in `assign_points` for the reference's
// sample-partition module, backed by the sm_100a kernels
// of libsbdt_gpu.so through the C ABI in sbdt_gpu.h.
//
// The reference declares this operation only in its SPEC (the source
// sample_partition.cpp listed at proj/src/CMakeLists.txt:6 does not ship,
// SURVEY.md F1/F2). This header gives it the SPEC's signature with the
// conventions of the shipped headers (proj/include/sbdt/*.hpp): namespace
// sbdt, D in {2,3} as a template parameter, uint32 ids, std::span inputs,
// return by value, an optional TaskPool* (unused: the work runs on the GPU),
// errors as the reference's exception types (common.hpp:22-65).
//
// Drop into the reference tree next to proj/include/sbdt/geometry.hpp and
// link libsbdt_gpu.so.
#pragma once

#include <cstdint>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sbdt/common.hpp"
#include "sbdt/geometry.hpp"
#include "sbdt_gpu.h"

namespace sbdt {

class TaskPool;

// SPEC.md:307-312
struct Partitioning {
  std::vector<PartitionId> labels;          // per input point, in [0, k)
  std::vector<std::vector<PointId>> parts;  // k lists, ascending point ids
  std::vector<PointId> sample_point_ids;
  std::vector<PartitionId> sample_labels;
};

namespace gpu_detail {

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
  (void)pool;
  static_assert(D == 2 || D == 3, "D must be 2 or 3");
  if (points.dim() != D) throw std::invalid_argument("assign_points: PointSet dimension mismatch");
  if (sample_ids.size() != sample_labels.size() || sample_ids.empty())
    throw std::invalid_argument("assign_points: every sample point must be labelled");
  for (PartitionId l : sample_labels)
    if (l >= k) throw std::invalid_argument("assign_points: sample label >= k");
  const std::uint64_t n = points.size();
  Partitioning out;
  out.labels.resize(n);
  out.sample_point_ids.assign(sample_ids.begin(), sample_ids.end());
  out.sample_labels.assign(sample_labels.begin(), sample_labels.end());
  std::vector<std::uint64_t> offsets(k + 1);
  std::vector<std::uint32_t> ids(n);
  sbdt_gpu_ctx* ctx = gpu_detail::thread_context();
  gpu_detail::check(ctx,
                    sbdt_gpu_assign_points(ctx, D, points.raw().data(), n, sample_ids.data(), sample_labels.data(),
                                           static_cast<std::uint32_t>(sample_ids.size()), k, out.labels.data(),
                                           offsets.data(), ids.data(), nullptr),
                    "assign_points");
  out.parts.resize(k);
  for (PartitionId p = 0; p < k; ++p) out.parts[p].assign(ids.begin() + offsets[p], ids.begin() + offsets[p + 1]);
  return out;
}

}  // namespace sbdt
