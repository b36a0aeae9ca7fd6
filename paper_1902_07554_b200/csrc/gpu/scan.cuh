// Device-wide exclusive prefix sum over uint32 counts (reduce-then-scan).
// Used by the CSR builds (sample grid, per-cell point lists), the stable
// label bucketing (K3) and the border-vertex compaction (K9).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace sbdt_gpu {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;  // per thread
constexpr int kScanTile = kScanThreads * kScanItems;

template <int THREADS>
__device__ __forceinline__ std::uint32_t block_exclusive_scan(std::uint32_t v, std::uint32_t* total) {
  __shared__ std::uint32_t warp_sums[THREADS / 32];
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  std::uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= static_cast<unsigned>(o)) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    std::uint32_t w = lane < THREADS / 32 ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= static_cast<unsigned>(o)) w += y;
    }
    if (lane < THREADS / 32) warp_sums[lane] = w;
  }
  __syncthreads();
  const std::uint32_t prefix = (warp > 0 ? warp_sums[warp - 1] : 0u) + x - v;
  if (total) *total = warp_sums[THREADS / 32 - 1];
  __syncthreads();
  return prefix;
}

__global__ void k_scan_reduce(const std::uint32_t* __restrict__ in, std::uint64_t n,
                              std::uint32_t* __restrict__ block_sums) {
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kScanTile;
  std::uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const std::uint64_t idx = base + std::uint64_t(i) * kScanThreads + threadIdx.x;
    if (idx < n) s += in[idx];
  }
  std::uint32_t total;
  block_exclusive_scan<kScanThreads>(s, &total);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

// Single-CTA exclusive scan of up to any length (serial over chunks).
__global__ void k_scan_single(std::uint32_t* __restrict__ data, std::uint64_t n, std::uint32_t* __restrict__ total_out) {
  std::uint32_t carry = 0;
  for (std::uint64_t base = 0; base < n; base += kScanThreads) {
    const std::uint64_t idx = base + threadIdx.x;
    const std::uint32_t v = idx < n ? data[idx] : 0u;
    std::uint32_t tot;
    const std::uint32_t p = block_exclusive_scan<kScanThreads>(v, &tot);
    if (idx < n) data[idx] = carry + p;
    carry += tot;
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

// `in` and `out` may alias (each thread reads its own elements before the
// block barrier and writes them after), hence no __restrict__.
__global__ void k_scan_apply(const std::uint32_t* in, std::uint64_t n, const std::uint32_t* __restrict__ block_offsets,
                             std::uint32_t* out) {
  const std::uint64_t base = std::uint64_t(blockIdx.x) * kScanTile;
  // each thread owns kScanItems consecutive elements
  const std::uint64_t first = base + std::uint64_t(threadIdx.x) * kScanItems;
  std::uint32_t vals[kScanItems];
  std::uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    vals[i] = (first + i < n) ? in[first + i] : 0u;
    s += vals[i];
  }
  std::uint32_t p = block_exclusive_scan<kScanThreads>(s, nullptr) + block_offsets[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (first + i < n) out[first + i] = p;
    p += vals[i];
  }
}

// out[i] = sum(in[0..i)), out may alias in; block_sums needs ceil(n/kScanTile)+1 slots.
// total (device pointer, optional) receives the grand total.
inline void exclusive_scan(const std::uint32_t* in, std::uint32_t* out, std::uint64_t n, std::uint32_t* block_sums,
                           std::uint32_t* total, cudaStream_t st, unsigned long long* launches) {
  const std::uint64_t blocks = (n + kScanTile - 1) / kScanTile;
  if (blocks == 0) {
    if (total) cudaMemsetAsync(total, 0, 4, st);
    return;
  }
  k_scan_reduce<<<static_cast<unsigned>(blocks), kScanThreads, 0, st>>>(in, n, block_sums);
  k_scan_single<<<1, kScanThreads, 0, st>>>(block_sums, blocks, total);
  k_scan_apply<<<static_cast<unsigned>(blocks), kScanThreads, 0, st>>>(in, n, block_sums, out);
  if (launches) *launches += 3;
}

}  // namespace
}  // namespace sbdt_gpu
