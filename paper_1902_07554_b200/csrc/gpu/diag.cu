// Test / diagnostic entry points (include/sbdt_gpu.h, "diagnostics"): not on
// the find_border / assign_points path.
//  - sbdt_gpu_predicates: the device predicates (predicates.hpp: binary64
//    filter, then expansion arithmetic) on caller arrays, so the tests can pin
//    them case by case against the reference's compiled geometry.cpp
//    (orient2/3 geometry.cpp:150-189, in_sphere2/3 geometry.cpp:191-277) and
//    the golden near-degenerate vectors (SPEC acceptance criterion 2).
//  - sbdt_gpu_microbench: the binding ceilings the border kernels are judged
//    against next to the HBM roofline: the DFMA issue peak and the random
//    8-byte gather rate from an L2-sized and from an HBM-sized table.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "context.cuh"
#include "sbdt_gpu.h"

namespace sbdt_gpu {
namespace {

constexpr int kPredThreads = 256;
constexpr int kPredEscThreads = 256;  // exact in_sphere: one global scratch area per thread

// op 0: orient over D+1 points; op 1: in_sphere of q (point D+1) against the
// simplex of points 0..D. Filter here; undecided in_sphere cases are listed
// for k_pred_escalate, undecided orientations are finished in place.
template <int D>
__global__ void __launch_bounds__(kPredThreads) k_pred_filter(int op, const double* __restrict__ pts,
                                                              std::uint64_t count, std::int8_t* __restrict__ out,
                                                              std::uint32_t* __restrict__ esc,
                                                              unsigned* __restrict__ esc_n,
                                                              unsigned long long* __restrict__ n_exact) {
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    if (op == 0) {
      const double* base = pts + i * (D + 1) * D;
      const double* p[D + 1];
#pragma unroll
      for (int j = 0; j <= D; ++j) p[j] = base + j * D;
      out[i] = static_cast<std::int8_t>(orient_dev<D>(p, n_exact));
    } else {
      const double* base = pts + i * (D + 2) * D;
      int r;
      if constexpr (D == 3) r = sbdt_pred::in_sphere3_filtered(base, base + 3, base + 6, base + 9, base + 12);
      else r = sbdt_pred::in_sphere2_filtered(base, base + 2, base + 4, base + 6);
      out[i] = static_cast<std::int8_t>(r);
      if (r == 2) esc[atomicAdd(esc_n, 1u)] = static_cast<std::uint32_t>(i);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(128) k_pred_escalate(const double* __restrict__ pts, std::int8_t* __restrict__ out,
                                                       const std::uint32_t* __restrict__ esc,
                                                       const unsigned* __restrict__ esc_n, double* __restrict__ scratch,
                                                       unsigned long long* __restrict__ n_exact) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  double* buf = scratch + std::size_t(tid) * (D == 3 ? sbdt_pred::kInSphere3Scratch : sbdt_pred::kInSphere2Scratch);
  const unsigned cnt = *esc_n;
  if (tid == 0) *n_exact += cnt;
  for (unsigned e = tid; e < cnt; e += gridDim.x * blockDim.x) {
    const std::uint32_t i = esc[e];
    const double* b = pts + std::uint64_t(i) * (D + 2) * D;
    int r;
    if constexpr (D == 3) r = sbdt_pred::in_sphere3_exact_buf(b, b + 3, b + 6, b + 9, b + 12, buf);
    else r = sbdt_pred::in_sphere2_exact_buf(b, b + 2, b + 4, b + 6, buf);
    out[i] = static_cast<std::int8_t>(r);
  }
}

template <int D>
int predicates_impl(sbdt_gpu_ctx* ctx, int op, const double* pts, std::uint64_t count, std::int8_t* out,
                    std::uint64_t* n_escalated) {
  cudaStream_t st = ctx->stream;
  const std::uint64_t per = std::uint64_t(op == 0 ? D + 1 : D + 2) * D;
  SBDT_WS(d_pts, double, "diag.pts", count * per);
  SBDT_WS(d_out, std::int8_t, "diag.out", count);
  SBDT_WS(d_esc, std::uint32_t, "diag.esc", op == 1 ? count : 1);
  SBDT_WS(d_n, unsigned long long, "diag.n", 2);
  SBDT_CUDA_TRY(cudaMemcpyAsync(d_pts, pts, count * per * sizeof(double), cudaMemcpyHostToDevice, st));
  SBDT_CUDA_TRY(cudaMemsetAsync(d_n, 0, 2 * sizeof(unsigned long long), st));
  unsigned* esc_n = reinterpret_cast<unsigned*>(d_n + 1);
  const std::uint64_t want = (count + kPredThreads - 1) / kPredThreads;
  const unsigned blocks = static_cast<unsigned>(want < 148ull * 16 ? (want ? want : 1) : 148ull * 16);
  k_pred_filter<D><<<blocks, kPredThreads, 0, st>>>(op, d_pts, count, d_out, d_esc, esc_n, d_n);
  ++ctx->launches;
  if (op == 1) {
    constexpr std::size_t scr = D == 3 ? sbdt_pred::kInSphere3Scratch : sbdt_pred::kInSphere2Scratch;
    SBDT_WS(d_scr, double, "diag.scratch", scr * kPredEscThreads);
    k_pred_escalate<D><<<kPredEscThreads / 128, 128, 0, st>>>(d_pts, d_out, d_esc, esc_n, d_scr, d_n);
    ++ctx->launches;
  }
  SBDT_CUDA_TRY(cudaMemcpyAsync(out, d_out, count, cudaMemcpyDeviceToHost, st));
  unsigned long long ne = 0;
  SBDT_CUDA_TRY(cudaMemcpyAsync(&ne, d_n, sizeof(ne), cudaMemcpyDeviceToHost, st));
  SBDT_CUDA_TRY(cudaStreamSynchronize(st));
  if (n_escalated) *n_escalated = ne;
  return kOk;
}

// ---- binding ceilings -------------------------------------------------------
constexpr int kFmaChains = 8;
constexpr int kFmaIters = 4096;

// Independent DFMA chains per thread (latency hidden by chains x warps);
// 2 flops per DFMA. `out` keeps the chains live.
__global__ void __launch_bounds__(256) k_dfma_peak(double seed, double* out) {
  double x[kFmaChains];
#pragma unroll
  for (int c = 0; c < kFmaChains; ++c) x[c] = seed + 1e-3 * (threadIdx.x + c);
  const double m = 0.999999, a = 1e-7;
  for (int i = 0; i < kFmaIters; ++i)
#pragma unroll
    for (int c = 0; c < kFmaChains; ++c) x[c] = __fma_rn(x[c], m, a);
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kFmaChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // practically never: keeps the chains live
}

// Random 8-byte gathers: every thread loads `per` table entries at hashed
// indices (independent loads, 4 in flight per step), `table` of `size` u64.
__global__ void __launch_bounds__(256) k_gather(const std::uint64_t* __restrict__ table, std::uint64_t size,
                                                unsigned per, std::uint64_t* out) {
  const std::uint64_t tid = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  std::uint64_t h = tid * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  std::uint64_t acc = 0;
  for (unsigned i = 0; i < per; i += 4) {
    std::uint64_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h ^= h >> 29;
      h *= 0xBF58476D1CE4E5B9ull;
      h ^= h >> 32;
      v[j] = __ldg(table + (h % size));
    }
    acc += v[0] ^ v[1] ^ v[2] ^ v[3];
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

__global__ void k_fill_u64(std::uint64_t* t, std::uint64_t size) {
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < size;
       i += std::uint64_t(gridDim.x) * blockDim.x)
    t[i] = i * 0x9E3779B97F4A7C15ull;
}

int microbench_impl(sbdt_gpu_ctx* ctx, int kind, std::uint64_t size, double* result) {
  cudaStream_t st = ctx->stream;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  cudaEvent_t e0, e1;
  SBDT_CUDA_TRY(cudaEventCreate(&e0));
  SBDT_CUDA_TRY(cudaEventCreate(&e1));
  SBDT_WS(sink, double, "diag.sink", 1);
  float best = 1e30f;
  double work = 0.0;
  if (kind == 0) {
    const unsigned blocks = static_cast<unsigned>(sms) * 8;
    work = 2.0 * kFmaChains * kFmaIters * double(blocks) * 256.0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, st);
      k_dfma_peak<<<blocks, 256, 0, st>>>(1.0 + r, sink);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    ctx->launches += 5;
  } else {
    const std::uint64_t entries = size / 8 ? size / 8 : 1;
    SBDT_WS(tab, std::uint64_t, "diag.table", entries);
    k_fill_u64<<<sms * 8, 256, 0, st>>>(tab, entries);
    const unsigned blocks = static_cast<unsigned>(sms) * 16;
    const unsigned per = 256;
    work = double(blocks) * 256.0 * per;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, st);
      k_gather<<<blocks, 256, 0, st>>>(tab, entries, per, reinterpret_cast<std::uint64_t*>(sink));
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r > 0 && ms < best) best = ms;
    }
    ctx->launches += 6;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  SBDT_CUDA_TRY(cudaGetLastError());
  // kind 0: FLOP/s; kind 1: gathers/s
  *result = work / (double(best) * 1e-3);
  return kOk;
}

}  // namespace
}  // namespace sbdt_gpu

using namespace sbdt_gpu;

extern "C" {

int sbdt_gpu_predicates(sbdt_gpu_ctx* ctx, int op, int dim, const double* pts, uint64_t count, int8_t* out,
                        uint64_t* n_escalated) {
  if (!ctx || (op != 0 && op != 1) || (dim != 2 && dim != 3) || (count && (!pts || !out)))
    return SBDT_ERR_INVALID;
  if (count > 0xFFFFFFFFull) return fail(ctx, SBDT_ERR_INVALID, "predicates: count must fit 32 bits");
  if (count == 0) {
    if (n_escalated) *n_escalated = 0;
    return SBDT_OK;
  }
  cudaSetDevice(ctx->device);
  const int rc = dim == 2 ? predicates_impl<2>(ctx, op, pts, count, out, n_escalated)
                          : predicates_impl<3>(ctx, op, pts, count, out, n_escalated);
  return rc == kOk ? SBDT_OK : rc;
}

int sbdt_gpu_microbench(sbdt_gpu_ctx* ctx, int kind, uint64_t bytes, double* result) {
  if (!ctx || !result || kind < 0 || kind > 1 || (kind == 1 && bytes < 8)) return SBDT_ERR_INVALID;
  cudaSetDevice(ctx->device);
  const int rc = microbench_impl(ctx, kind, bytes, result);
  return rc == kOk ? SBDT_OK : rc;
}

}  // extern "C"
