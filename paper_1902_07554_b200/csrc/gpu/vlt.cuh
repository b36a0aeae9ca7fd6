// Voronoi label table (VLT): the assignment's per-point work becomes one table
// lookup for most points. Included by assign.cu (needs SampleRec, SampleGrid,
// nearest_label_ring, bbox_flush).
//
// Every grid cell (~2 samples) is split into F^D fine cells. For each fine
// cell a CONSERVATIVE candidate set of samples is computed: every sample that
// can be the binary64 argmin (squared_distance, lowest pid on ties) for SOME
// point binned into the cell is kept. A sample s is dropped only when one
// dominator t is provably strictly closer over the whole (inflated) cell box:
//   |x-s|^2 - |x-t|^2 = F0 + 2 y.(t-s) >= F0 - 2 sum |t_d - s_d| hw_d  (y = x - c)
// must exceed 1e-5 * ((|c-s|+H)^2 + (|c-t|+H)^2); the test runs in binary32 on
// coordinates relative to the box centre, and 1e-5 is ~100x the total
// binary32 rounding of the inputs and of the test. Dropping is
// thus safe; keeping extra samples only costs time.
//
// Record per fine cell (u32 head): count 0 -> UNIFORM (label << 8), all
// candidates share one label; 1..kSlots -> candidate list in the cell's slab
// slot (16-byte entries: binary32 coordinates relative to the cell centre +
// sample index); SUB (kHeadSubBit) -> the cell is split at its centre into 2^D
// sub-boxes with their own heads (density-adaptive: a list longer than
// kSlots is refined up to kVltDepth times; sub-box lists live in the long
// slab as kHeadPool); kHeadLong -> a long list (header entry holds the
// count), evaluated by the queue kernel; kHeadOverflow -> exact ring search.
// Point decision: binary32 distances with a rigorous per-candidate error bound
// pick the winner when the gap exceeds both bounds; otherwise the tied
// candidates are compared exactly in binary64 (reference formula + pid).
#pragma once

namespace sbdt_gpu {

constexpr int kSlots = 12;                    // head 1..12: list of that length in the cell's slab slot
// head & 15 == 0: UNIFORM (label << 8) or, with bit 4 set, SUB: 2^D sub-box
// heads at subheads[head >> 8]
constexpr std::uint32_t kHeadSubBit = 0x10u;
constexpr std::uint32_t kHeadPool = 13u;      // short list (<= kSlots) in the long slab: header + entries
constexpr std::uint32_t kHeadLong = 14u;      // long list in the long slab (header + entries), queued points
constexpr std::uint32_t kHeadOverflow = 15u;  // exact ring search
constexpr int kVltDepth = 3;                  // sub-box levels below a fine cell (cell size / 2^3)
constexpr int kVltSplitMin = 32;              // lists longer than this are refined
constexpr int kVltLevels = kVltDepth + 2;     // kept-set levels: coarse, fine, sub-boxes
constexpr int kVltWarps = 4;
constexpr int kVltCap = 192;

struct __align__(16) VltEntry {
  float r[3];          // sample - fine-cell centre (binary32)
  std::uint32_t idx;   // index into the cell-sorted SampleRec array
};

template <int D>
struct FineGeom {
  double c[D];
  float hw[D];
  float H;
};

// binary32 dominance: true iff s (rel rs) is never the argmin in the box
// (centre c, half-widths hw, half-diagonal H) because t (rel rt) wins.
template <int D>
__device__ __forceinline__ bool dominated_f(const float* rs, const float* rt, const float* hw, float H) {
  float ds = 0.f, dt = 0.f, slope = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    ds = __fadd_rn(ds, __fmul_rn(rs[d], rs[d]));
    dt = __fadd_rn(dt, __fmul_rn(rt[d], rt[d]));
    slope = __fadd_rn(slope, __fmul_rn(fabsf(__fsub_rn(rt[d], rs[d])), hw[d]));
  }
  const float fmin_ = __fsub_rn(__fsub_rn(ds, dt), __fmul_rn(2.f, slope));
  // |c-s| + H and |c-t| + H only scale the safety margin: MUFU square roots
  // (within 2^-22 relative) rounded up by 1e-6 can only raise it (.ftz: a
  // subnormal distance reads as 0, < 1e-19 below it, far inside the margin)
  float ra, rb;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(ra) : "f"(ds));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(dt));
  const float a = __fadd_ru(ra * 1.000001f, H), b = __fadd_ru(rb * 1.000001f, H);
  return fmin_ > 1e-5f * (a * a + b * b);
}

// One warp per grid cell: coarse candidates (radius + dominance against the
// sample nearest to the cell centre), then per fine cell the nearest coarse
// candidate as dominator. Two instantiations:
//   DENSE = false: all cells, candidate arrays in shared memory (kVltCap);
//                  a cell with more coarse candidates is queued (dq) for
//   DENSE = true : the queued cells, candidate arrays in a global per-warp
//                  scratch (kVltDenseCap; beyond that: ring search). Sample-
//                  clustered inputs (BASELINE config 4) have such cells.
constexpr int kVltDenseCap = 4096;
constexpr int kVltDenseWarps = 4;

template <int D>
constexpr std::size_t vlt_dense_bytes_per_warp() {
  return ((std::size_t(kVltDenseCap) * (8 + 4 * D) + std::size_t(kVltDenseCap) * 2 * kVltLevels) + 255) / 256 * 256;
}

// DFS node of the fine-cell refinement: a box and where its head goes.
template <int D>
struct VltNode {
  double lo[D], hi[D];
  unsigned long long target;  // index into heads (fine cells) or subheads (sub-boxes)
  int level;                  // 1 = fine cell, 2.. = sub-boxes
  int sub;                    // target is in subheads
};
constexpr int kVltStack = 8 + (1 << 3) * kVltDepth;

// Locates the table record of point x: its fine cell, then the sub-boxes
// (split at the centre, x >= centre -> upper half, the same binary64
// expressions as the build). Returns the head; fid = fine cell, centre of
// the final box in fcen; false if x lies outside the table.
template <int D>
__device__ __forceinline__ bool vlt_locate(const double* x, const SampleGrid<D>& sg,
                                           const std::uint32_t* __restrict__ heads,
                                           const std::uint32_t* __restrict__ subheads, std::uint32_t* head_out,
                                           long long* fid_out, double* fcen) {
  constexpr int F = fine_factor<D>();
  constexpr int FC = fine_per_cell<D>();
  bool inside = true;
  long long cell = 0, mul = 1;
  int sub = 0, smul = 1;
  double lo[D], hi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double f = floor((x[d] - sg.g.lo[d]) * sg.inv_ef);
    inside = inside && (f >= 0.0) && (f < static_cast<double>(sg.g.dims[d] * F));
    const int fi = inside ? static_cast<int>(f) : 0;
    cell += static_cast<long long>(fi / F) * mul;
    sub += (fi % F) * smul;
    mul *= sg.g.dims[d];
    smul *= F;
    lo[d] = sg.g.lo[d] + static_cast<double>(fi) * sg.ef;
    hi[d] = sg.g.lo[d] + static_cast<double>(fi + 1) * sg.ef;
  }
  if (!inside) return false;
  const long long fid = cell * FC + sub;
  std::uint32_t head = __ldg(heads + fid);
  while ((head & 0xFFu) == kHeadSubBit) {
    unsigned idx = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double mid = 0.5 * (lo[d] + hi[d]);
      if (x[d] >= mid) {
        idx |= 1u << d;
        lo[d] = mid;
      } else {
        hi[d] = mid;
      }
    }
    head = __ldg(subheads + (head >> 8) + idx);
  }
#pragma unroll
  for (int d = 0; d < D; ++d) fcen[d] = 0.5 * (lo[d] + hi[d]);
  *head_out = head;
  *fid_out = fid;
  return true;
}

// Visits every sample of the cell block [lo_c, lo_c + span) with the whole
// warp. The cells of a row along axis 0 are consecutive in the cell-sorted
// sample array, so a row is one contiguous run; 32 rows at a time, their runs
// are flattened over the lanes (balanced however the samples cluster, no
// per-cell divisions). f(s) runs on the lane that owns sample s; it must not
// contain warp collectives. Must be called by the full warp.
template <int D, class Fn>
__device__ __forceinline__ void warp_visit_samples(const Grid<D>& g, const std::uint32_t* __restrict__ starts,
                                                   const int* lo_c, const int* span, Fn&& f) {
  const unsigned lane = threadIdx.x & 31u;
  const int rows = D == 3 ? span[1] * span[2] : span[1];
  for (int r0 = 0; r0 < rows; r0 += 32) {
    const int r = r0 + static_cast<int>(lane);
    std::uint32_t sb = 0, len = 0;
    if (r < rows) {
      long long c0;
      if constexpr (D == 3) {
        const int q2 = r / span[1], q1 = r - q2 * span[1];
        c0 = (static_cast<long long>(lo_c[2] + q2) * g.dims[1] + (lo_c[1] + q1)) * g.dims[0] + lo_c[0];
      } else {
        c0 = static_cast<long long>(lo_c[1] + r) * g.dims[0] + lo_c[0];
      }
      sb = starts[c0];
      len = starts[c0 + span[0]] - sb;
    }
    std::uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const std::uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= static_cast<unsigned>(o)) incl += y;
    }
    const std::uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const std::uint32_t excl = incl - len;
    for (std::uint32_t b0 = 0; b0 < total; b0 += 32) {
      const std::uint32_t q = b0 + lane;
      // the row holding item q: the last lane j with excl_j <= q (excl is
      // non-decreasing over the lanes)
      int j = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const std::uint32_t e = __shfl_sync(0xffffffffu, excl, j + step);
        if (e <= q) j += step;
      }
      const std::uint32_t ej = __shfl_sync(0xffffffffu, excl, j);
      const std::uint32_t sj = __shfl_sync(0xffffffffu, sb, j);
      if (q < total) f(sj + (q - ej));
    }
  }
}

template <int D>
struct VltScratch {
  std::uint32_t* idx;
  std::uint32_t* lab;
  float* rel;      // [cap][D], relative to the coarse centre
  std::uint16_t* kl;  // [kVltLevels][cap] kept-set index lists per level (level 0 implicit: 0..ncand-1)
};

template <int D, bool DENSE>
__global__ void __launch_bounds__(32 * kVltWarps) k_vlt_build(const SampleGrid<D>* __restrict__ sgp,
                                                              const std::uint32_t* __restrict__ starts,
                                                              const SampleRec* __restrict__ sorted,
                                                              std::uint32_t* __restrict__ heads,
                                                              VltEntry* __restrict__ slab, VltEntry* __restrict__ lslab,
                                                              unsigned* __restrict__ lcount, unsigned lcap,
                                                              unsigned* __restrict__ stats,
                                                              std::uint32_t* __restrict__ dq, unsigned* __restrict__ dqn,
                                                              void* __restrict__ dense_scratch,
                                                              std::uint32_t* __restrict__ subheads,
                                                              unsigned* __restrict__ subcount, unsigned subcap) {
  constexpr int CAP = DENSE ? kVltDenseCap : kVltCap;
  __shared__ SampleGrid<D> sg;
  __shared__ std::uint32_t s_idx[DENSE ? 1 : kVltWarps][DENSE ? 1 : kVltCap];
  __shared__ float s_rel[DENSE ? 1 : kVltWarps][DENSE ? 1 : kVltCap][D];
  __shared__ std::uint32_t s_lab[DENSE ? 1 : kVltWarps][DENSE ? 1 : kVltCap];
  __shared__ std::uint16_t s_kl[kVltWarps][DENSE ? 1 : kVltLevels * kVltCap];
  __shared__ int s_kn[kVltWarps][kVltLevels];
  __shared__ VltNode<D> s_stk[kVltWarps][kVltStack];
  __shared__ int s_cnt[kVltWarps];
  if (threadIdx.x == 0) sg = *sgp;
  __syncthreads();
  const Grid<D>& g = sg.g;
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  VltScratch<D> A;
  if constexpr (DENSE) {
    const std::size_t gw = std::size_t(blockIdx.x) * kVltWarps + warp;
    char* base = static_cast<char*>(dense_scratch) + gw * vlt_dense_bytes_per_warp<D>();
    A.idx = reinterpret_cast<std::uint32_t*>(base);
    A.lab = A.idx + CAP;
    A.rel = reinterpret_cast<float*>(A.lab + CAP);
    A.kl = reinterpret_cast<std::uint16_t*>(A.rel + std::size_t(CAP) * D);
  } else {
    A.idx = s_idx[warp];
    A.lab = s_lab[warp];
    A.rel = &s_rel[warp][0][0];
    A.kl = s_kl[warp];
  }
  constexpr int F = fine_factor<D>();
  constexpr int FC = fine_per_cell<D>();
  unsigned st_uniform = 0, st_list = 0, st_over = 0, st_long = 0;
  const long long cells = DENSE ? static_cast<long long>(*dqn) : static_cast<long long>(sg.cells);
  for (long long item = static_cast<long long>(blockIdx.x) * kVltWarps + warp; item < cells;
       item += static_cast<long long>(gridDim.x) * kVltWarps) {
    const long long cell = DENSE ? static_cast<long long>(dq[item]) : item;
    int cc[D];
    {
      // 32-bit: the sample grid has at most min(16 m + 1024, 2^31) cells
      unsigned rem = static_cast<unsigned>(cell);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const unsigned dd = static_cast<unsigned>(g.dims[d]);
        const unsigned qd = rem / dd;
        cc[d] = static_cast<int>(rem - qd * dd);
        rem = qd;
      }
    }
    if (!DENSE && sg.refined) {
      // refined grid (clustered samples): a record only where samples are
      // within the 3^D neighbourhood; elsewhere (no point expected: points
      // follow the samples) the heads send points to the exact ring search
      bool near = false;
      if (lane < static_cast<unsigned>(D == 3 ? 27 : 9)) {
        long long nid = 0, mul = 1;
        bool in = true;
        unsigned rem = lane;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int nc = cc[d] + static_cast<int>(rem % 3u) - 1;
          rem /= 3u;
          in = in && nc >= 0 && nc < static_cast<int>(g.dims[d]);
          nid += static_cast<long long>(nc) * mul;
          mul *= g.dims[d];
        }
        near = in && starts[nid + 1] > starts[nid];
      }
      if (!__any_sync(0xffffffffu, near)) {
        for (int f = static_cast<int>(lane); f < FC; f += 32) heads[cell * FC + f] = kHeadOverflow;
        continue;
      }
    }
    double c[D];
    float hw[D];
    float H2 = 0.f;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double lo = cell_lo<D>(g, cc[d], d), hi = cell_lo<D>(g, cc[d] + 1, d);
      c[d] = 0.5 * (lo + hi);
      // binary32 half-width rounded up, plus the coarse inflation
      hw[d] = __double2float_ru(0.5 * (hi - lo) + sg.delta_c);
      H2 = __fadd_ru(H2, __fmul_ru(hw[d], hw[d]));
    }
    const float H = __fsqrt_ru(H2);
    // (a) dominator: nearest sample to the centre in growing rings
    double bd = INFINITY;
    std::uint32_t bi = 0xFFFFFFFFu;
    for (int r = 1;; ++r) {
      int lo_c[D], span[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        lo_c[d] = max(cc[d] - r, 0);
        span[d] = min(cc[d] + r, static_cast<int>(g.dims[d]) - 1) - lo_c[d] + 1;
      }
      warp_visit_samples<D>(g, starts, lo_c, span, [&](std::uint32_t s) {
        const double d2 = sqdist<D>(c, sorted[s].x);
        if (d2 < bd || (d2 == bd && s < bi)) {
          bd = d2;
          bi = s;
        }
      });
      warp_argmin<D>(bd, bi);
      if (bi != 0xFFFFFFFFu) break;
      bool whole = true;
#pragma unroll
      for (int d = 0; d < D; ++d) whole = whole && (cc[d] - r <= 0) && (cc[d] + r >= g.dims[d] - 1);
      if (whole) break;
    }
    // (b) coarse candidates within R = |c - s0| + 2H (+ margins)
    float r0[D];
#pragma unroll
    for (int d = 0; d < D; ++d) r0[d] = static_cast<float>(sorted[bi].x[d] - c[d]);
    const double R = (sqrt(bd) + 2.0 * static_cast<double>(H)) * (1.0 + 1e-6) + sg.margin;
    const double R2 = R * R;
    if (lane == 0) s_cnt[warp] = 0;
    __syncwarp();
    {
      int lo_c[D], span[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int a = max(static_cast<int>(floor((c[d] - R - g.lo[d]) / g.edge)), 0);
        const int b = min(static_cast<int>(floor((c[d] + R - g.lo[d]) / g.edge)), static_cast<int>(g.dims[d]) - 1);
        lo_c[d] = a;
        span[d] = b - a + 1;
      }
      warp_visit_samples<D>(g, starts, lo_c, span, [&](std::uint32_t s) {
        const SampleRec rec = sorted[s];
        const double d2 = sqdist<D>(c, rec.x);
        if (d2 > R2) return;
        float rs[D];
#pragma unroll
        for (int d = 0; d < D; ++d) rs[d] = static_cast<float>(rec.x[d] - c[d]);
        if (s != bi && dominated_f<D>(rs, r0, hw, H)) return;
        const int slot = atomicAdd(&s_cnt[warp], 1);
        if (slot < CAP) {
          A.idx[slot] = s;
          A.lab[slot] = rec.label;
#pragma unroll
          for (int d = 0; d < D; ++d) A.rel[std::size_t(slot) * D + d] = rs[d];
        }
      });
    }
    __syncwarp();
    const int ncand = s_cnt[warp];
    if (ncand > CAP) {
      if constexpr (!DENSE) {
        if (lane == 0) dq[atomicAdd(dqn, 1u)] = static_cast<std::uint32_t>(cell);  // heads by the dense pass
      } else {
        for (int f = lane; f < FC; f += 32) heads[cell * FC + f] = kHeadOverflow;
        if (lane == 0) st_over += FC;
      }
      continue;
    }
    // Coarse candidates (a superset of every fine cell's) of one label: every
    // fine cell is UNIFORM with that label (partition interiors).
    if (ncand >= 1) {
      const std::uint32_t lab0 = A.lab[0];
      bool mixed = false;
      for (int j = lane; j < ncand; j += 32) mixed = mixed || A.lab[j] != lab0;
      if (!__any_sync(0xffffffffu, mixed)) {
        for (int f = lane; f < FC; f += 32) heads[cell * FC + f] = lab0 << 8;
        if (lane == 0) st_uniform += FC;
        continue;
      }
    }
    // (c) fine cells, refined into 2^D sub-boxes (depth <= kVltDepth) while a
    //     box's candidate list is longer than kSlots. Kept candidates per
    //     level as index lists in A.kl (level 0 = all coarse candidates).
    VltNode<D>* stk = s_stk[warp];
    int top = 0;
    if (lane == 0) {
      for (int f = FC - 1; f >= 0; --f) {
        int fi[D];
        int rem = f;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          fi[d] = cc[d] * F + rem % F;
          rem /= F;
        }
        VltNode<D> nd;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          nd.lo[d] = g.lo[d] + static_cast<double>(fi[d]) * sg.ef;
          nd.hi[d] = g.lo[d] + static_cast<double>(fi[d] + 1) * sg.ef;
        }
        nd.target = static_cast<unsigned long long>(cell * FC + f);
        nd.level = 1;
        nd.sub = 0;
        stk[top++] = nd;
      }
      s_kn[warp][0] = ncand;
    }
    top = __shfl_sync(0xffffffffu, top, 0);
    __syncwarp();
    while (top > 0) {
      const VltNode<D> nd = stk[top - 1];
      --top;
      __syncwarp();
      const int pl = nd.level - 1;
      const std::uint16_t* plist = A.kl + std::size_t(pl) * CAP;  // unused for level 0 (identity)
      const int np = s_kn[warp][pl];
      std::uint16_t* klist = A.kl + std::size_t(nd.level) * CAP;
      auto cand = [&](int t) -> int { return pl == 0 ? t : static_cast<int>(plist[t]); };
      // box centre/half-widths, and the offset of its centre from the coarse centre
      double fc[D];
      float fhw[D], off[D];
      float fH2 = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        fc[d] = 0.5 * (nd.lo[d] + nd.hi[d]);
        fhw[d] = __double2float_ru(0.5 * (nd.hi[d] - nd.lo[d]) + sg.delta_f);
        fH2 = __fadd_ru(fH2, __fmul_ru(fhw[d], fhw[d]));
        off[d] = static_cast<float>(fc[d] - c[d]);
      }
      const float fH = __fsqrt_ru(fH2);
      // Relative coordinates w.r.t. the box centre are recomputed in binary64
      // for the stored entries; the dominance test uses (coarse-rel - off),
      // whose extra rounding is covered by the 1e-5 margin.
      // the three candidates nearest to the box centre (dominators): per-lane
      // top 3 in one pass, then three warp argmin rounds
      float ld[3] = {INFINITY, INFINITY, INFINITY};
      int lj[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff};
      for (int t = lane; t < np; t += 32) {
        const int j = cand(t);
        float dd = 0.f;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const float u = A.rel[std::size_t(j) * D + d] - off[d];
          dd += u * u;
        }
        // insert (dd, j) into the lane's sorted top 3 (ties: lower j first)
        if (dd < ld[2] || (dd == ld[2] && j < lj[2])) {
          if (dd < ld[1] || (dd == ld[1] && j < lj[1])) {
            ld[2] = ld[1];
            lj[2] = lj[1];
            if (dd < ld[0] || (dd == ld[0] && j < lj[0])) {
              ld[1] = ld[0];
              lj[1] = lj[0];
              ld[0] = dd;
              lj[0] = j;
            } else {
              ld[1] = dd;
              lj[1] = j;
            }
          } else {
            ld[2] = dd;
            lj[2] = j;
          }
        }
      }
      int dom[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        // argmin of (distance, index) over the lanes' heads: distances are
        // >= 0 (or +inf), so their bit patterns order like the values; two
        // warp reductions (min distance, then min index among the ties)
        const unsigned bits = __float_as_uint(ld[0]);
        const unsigned mb = __reduce_min_sync(0xffffffffu, bits);
        const int bjv = static_cast<int>(
            __reduce_min_sync(0xffffffffu, bits == mb ? static_cast<unsigned>(lj[0]) : 0x7fffffffu));
        dom[k] = bjv;
        if (lj[0] == bjv && bjv != 0x7fffffff) {  // the winning lane pops its head
          ld[0] = ld[1];
          lj[0] = lj[1];
          ld[1] = ld[2];
          lj[1] = lj[2];
          ld[2] = INFINITY;
          lj[2] = 0x7fffffff;
        }
      }
      const int bj = dom[0];
      float rt[D];
#pragma unroll
      for (int d = 0; d < D; ++d) rt[d] = A.rel[std::size_t(bj) * D + d] - off[d];
      const std::uint32_t lab0 = A.lab[bj];
      const int dj0 = dom[1] == 0x7fffffff ? bj : dom[1];
      const int dj1 = dom[2] == 0x7fffffff ? bj : dom[2];
      float rt1[D], rt2[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        rt1[d] = A.rel[std::size_t(dj0) * D + d] - off[d];
        rt2[d] = A.rel[std::size_t(dj1) * D + d] - off[d];
      }
      // kept list of this box (dominance against the nearest parent candidates)
      int count = 0, inbox = 0;  // kept candidates; samples inside the box (~ points to expect)
      bool uniform = true;
      for (int t0 = 0; t0 < np; t0 += 32) {
        const int t = t0 + static_cast<int>(lane);
        bool keep = false, ins = false;
        int j = 0;
        if (t < np) {
          j = cand(t);
          float rs[D];
          ins = true;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            rs[d] = A.rel[std::size_t(j) * D + d] - off[d];
            ins = ins && fabsf(rs[d]) <= fhw[d];
          }
          keep = (j == bj) || !(dominated_f<D>(rs, rt, fhw, fH) || dominated_f<D>(rs, rt1, fhw, fH) ||
                                dominated_f<D>(rs, rt2, fhw, fH));
        }
        inbox += __popc(__ballot_sync(0xffffffffu, ins));
        const unsigned word = __ballot_sync(0xffffffffu, keep);
        if (keep) klist[count + __popc(word & ((1u << lane) - 1u))] = static_cast<std::uint16_t>(j);
        if (__ballot_sync(0xffffffffu, keep && A.lab[j] != lab0)) uniform = false;
        count += __popc(word);
      }
      if (lane == 0) s_kn[warp][nd.level] = count;
      __syncwarp();
      std::uint32_t head = kHeadOverflow;
      VltEntry* out = nullptr;
      bool split = false;
      if (uniform) {
        head = lab0 << 8;
      } else if (count <= kSlots && !nd.sub) {
        head = static_cast<std::uint32_t>(count);
        out = slab + nd.target * kSlots;
      } else {
        // split long lists while the depth allows and the sub-head pool has
        // room (moderately long lists stay long: one pass in the queue kernel
        // is cheaper than 2^D sub-boxes)
        if ((count > kVltSplitMin || inbox >= 2) && nd.level <= kVltDepth) {
          unsigned so = 0;
          if (lane == 0) so = atomicAdd(subcount, 1u << D);
          so = __shfl_sync(0xffffffffu, so, 0);
          if (static_cast<unsigned long long>(so) + (1u << D) <= subcap && so < (1u << 24)) {
            head = (so << 8) | kHeadSubBit;
            split = true;
            if (lane == 0) {
              for (int i = (1 << D) - 1; i >= 0; --i) {
                VltNode<D> ch;
#pragma unroll
                for (int d = 0; d < D; ++d) {
                  const bool up = (i >> d) & 1;
                  ch.lo[d] = up ? fc[d] : nd.lo[d];
                  ch.hi[d] = up ? nd.hi[d] : fc[d];
                }
                ch.target = so + static_cast<unsigned>(i);
                ch.level = nd.level + 1;
                ch.sub = 1;
                stk[top + ((1 << D) - 1 - i)] = ch;
              }
            }
          }
        }
        if (!split) {
          unsigned o = 0;
          if (lane == 0) o = atomicAdd(lcount, static_cast<unsigned>(count + 1));
          o = __shfl_sync(0xffffffffu, o, 0);
          if (static_cast<unsigned long long>(o) + count + 1 <= lcap && o < (1u << 28)) {
            head = (o << 4) | (count <= kSlots ? kHeadPool : kHeadLong);
            if (lane == 0) {
              VltEntry h;
              h.r[0] = h.r[1] = h.r[2] = 0.f;
              h.idx = static_cast<std::uint32_t>(count);
              lslab[o] = h;
            }
            out = lslab + o + 1;
          }
        }
      }
      if (out) {
        for (int t = lane; t < count; t += 32) {
          const std::uint32_t si = A.idx[klist[t]];
          VltEntry e;
#pragma unroll
          for (int d = 0; d < 3; ++d) e.r[d] = 0.f;
#pragma unroll
          for (int d = 0; d < D; ++d) e.r[d] = static_cast<float>(sorted[si].x[d] - fc[d]);
          e.idx = si;
          out[t] = e;
        }
      }
      if (lane == 0) {
        if (nd.sub) subheads[nd.target] = head;
        else heads[nd.target] = head;
        const std::uint32_t h = head & 15u;
        if (h == 0) {
          if (!(head & kHeadSubBit)) ++st_uniform;
        } else if (h == kHeadOverflow) {
          ++st_over;
        } else if (h == kHeadLong) {
          ++st_long;
        } else {
          ++st_list;
        }
      }
      if (split) top += 1 << D;
      __syncwarp();
    }
  }
  if (stats && lane == 0) {
    atomicAdd(&stats[0], st_uniform);
    atomicAdd(&stats[1], st_list);
    atomicAdd(&stats[2], st_over);
    atomicAdd(&stats[3], st_long);
  }
}

// K2: table-driven point pass (coordinates streamed once; overflow points
// are queued for k_assign_overflow so they do not diverge the warp).
template <int D>
__global__ void __launch_bounds__(256) k_assign_vlt(const double* __restrict__ xyz, std::uint64_t i_begin,
                                                    std::uint64_t n,
                                                    const SampleGrid<D>* __restrict__ sgp,
                                                    const std::uint32_t* __restrict__ heads,
                                                    const std::uint32_t* __restrict__ subheads,
                                                    const VltEntry* __restrict__ slab,
                                                    const VltEntry* __restrict__ lslab,
                                                    const SampleRec* __restrict__ sorted,
                                                    const std::uint32_t* __restrict__ sorted_labels,
                                                    std::uint32_t* __restrict__ labels, unsigned long long* bbox,
                                                    std::uint32_t* __restrict__ oq, unsigned* __restrict__ oq_count) {
  __shared__ SampleGrid<D> s_sg;
  if (threadIdx.x == 0) s_sg = *sgp;
  __syncthreads();
  const SampleGrid<D>& sg = s_sg;
  constexpr int F = fine_factor<D>();
  constexpr int FC = fine_per_cell<D>();
  double blo[D], bhi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) blo[d] = INFINITY, bhi[d] = -INFINITY;
  // Points whose record is a candidate list wait in a per-warp batch (shared
  // memory) until 32 have gathered; then every lane takes one and the list
  // decision runs with all lanes busy. PointIds are spatially random, so a
  // warp's 32 points mix UNIFORM records (most of them: one lookup) with
  // lists: deciding the lists in place ran the list code for every warp with
  // a quarter of its lanes.
  // {point id, entries pointer lo/hi, count, p[D] (offset from the box centre, binary32)}
  constexpr int BW = 4 + D;
  __shared__ std::uint32_t s_bat[8][BW][64];
  std::uint32_t(&B)[BW][64] = s_bat[threadIdx.x >> 5];
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  unsigned bcount = 0;
  auto decide_list = [&](std::uint64_t i, const VltEntry* ents, std::uint32_t cnt, const float* p) {
    float pp = 0.f;
#pragma unroll
    for (int d = 0; d < D; ++d) pp += p[d] * p[d];
    // binary32 distances with the rigorous bound 4e-6 (|p|^2 + |s|^2): one
    // pass keeps the winner (smallest dd, first on ties) and the two
    // smallest interval lower ends (no per-candidate arrays: registers only)
    auto dist = [&](const float4& e, float* bnd) {
      const float er[3] = {e.x, e.y, e.z};
      float dd = 0.f, ss = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const float t = p[d] - er[d];
        dd += t * t;
        ss += er[d] * er[d];
      }
      *bnd = 4e-6f * (pp + ss) + 1e-30f;
      return dd;
    };
    float bv = INFINITY, bb = 0.f, m1 = INFINITY, m2 = INFINITY;
    int bj = 0, j1 = -1;
    // entries in groups of 4 whose loads are in flight together (one L2
    // latency per group instead of one per entry)
    for (int j0 = 0; j0 < static_cast<int>(cnt); j0 += 4) {
      float4 eg[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        eg[u] = j0 + u < static_cast<int>(cnt) ? __ldg(reinterpret_cast<const float4*>(ents + j0 + u))
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j0 + u >= static_cast<int>(cnt)) break;
        const int j = j0 + u;
        float bnd;
        const float dd = dist(eg[u], &bnd);
        if (dd < bv) {
          bv = dd;
          bb = bnd;
          bj = j;
        }
        const float lo_end = dd - bnd;
        if (lo_end < m1) {
          m2 = m1;
          m1 = lo_end;
          j1 = j;
        } else if (lo_end < m2) {
          m2 = lo_end;
        }
      }
    }
    // decided iff every other candidate is provably farther
    const float lim = bv + bb;
    std::uint32_t lab;
    if ((j1 == bj ? m2 : m1) > lim) {
      lab = __ldg(sorted_labels + ents[bj].idx);
    } else {
      // exact binary64 argmin over the candidates whose interval overlaps
      // the winner's (reference squared_distance, lowest pid on ties)
      double x[D];
#pragma unroll
      for (int d = 0; d < D; ++d) x[d] = xyz[i * D + d];
      double best = INFINITY;
      std::uint32_t bpid = 0xFFFFFFFFu;
      lab = 0;
      for (int j = 0; j < static_cast<int>(cnt); ++j) {
        float bnd;
        const float dd = dist(__ldg(reinterpret_cast<const float4*>(ents + j)), &bnd);
        if (j != bj && dd - bnd > lim) continue;
        const SampleRec rec = sorted[ents[j].idx];
        const double d2 = sqdist<D>(x, rec.x);
        if (d2 < best || (d2 == best && rec.pid < bpid)) {
          best = d2;
          bpid = rec.pid;
          lab = rec.label;
        }
      }
    }
    __stcs(labels + i, lab);
  };
  auto flush_batch = [&](unsigned nproc) {
    __syncwarp();
    if (lane < nproc) {
      const unsigned e = bcount - nproc + lane;
      float p[D];
#pragma unroll
      for (int d = 0; d < D; ++d) p[d] = __uint_as_float(B[4 + d][e]);
      const VltEntry* ents = reinterpret_cast<const VltEntry*>(
          static_cast<std::uintptr_t>(B[1][e]) | (static_cast<std::uintptr_t>(B[2][e]) << 32));
      decide_list(B[0][e], ents, B[3][e], p);
    }
    bcount -= nproc;
    __syncwarp();
  };
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  // (warp-uniform trip count: the lanes of a warp hold consecutive points)
  for (std::uint64_t i0 = i_begin + std::uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); i0 < n; i0 += stride) {
    const std::uint64_t i = i0 + lane;
    bool is_list = false;
    const VltEntry* ents = nullptr;
    std::uint32_t cnt = 0;
    float p[D];
#pragma unroll
    for (int d = 0; d < D; ++d) p[d] = 0.f;
    if (i < n) {
      double x[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        x[d] = __ldcs(xyz + i * D + d);
        blo[d] = fmin(blo[d], x[d]);
        bhi[d] = fmax(bhi[d], x[d]);
      }
      double fcen[D];
      std::uint32_t head = kHeadOverflow;
      long long fid = 0;
      vlt_locate<D>(x, sg, heads, subheads, &head, &fid, fcen);
      cnt = head & 15u;
      if (cnt == 0) {
        __stcs(labels + i, head >> 8);
      } else if (cnt >= kHeadLong) {
        const unsigned slot = atomicAdd(oq_count, 1u);
        oq[slot] = static_cast<std::uint32_t>(i);
      } else {
        is_list = true;
        ents = slab + fid * kSlots;
        if (cnt == kHeadPool) {  // sub-box list in the long slab
          ents = lslab + (head >> 4);
          cnt = ents[0].idx;
          ++ents;
        }
#pragma unroll
        for (int d = 0; d < D; ++d) p[d] = static_cast<float>(x[d] - fcen[d]);
      }
    }
    const unsigned mb = __ballot_sync(0xffffffffu, is_list);
    if (is_list) {
      const unsigned slot = bcount + __popc(mb & lt);
      const std::uintptr_t ep = reinterpret_cast<std::uintptr_t>(ents);
      B[0][slot] = static_cast<std::uint32_t>(i);
      B[1][slot] = static_cast<std::uint32_t>(ep);
      B[2][slot] = static_cast<std::uint32_t>(ep >> 32);
      B[3][slot] = cnt;
#pragma unroll
      for (int d = 0; d < D; ++d) B[4 + d][slot] = __float_as_uint(p[d]);
    }
    bcount += __popc(mb);
    if (bcount >= 32) flush_batch(32);
  }
  if (bcount) flush_batch(bcount);
  bbox_flush<D>(blo, bhi, bbox);
}

// Queued points (long candidate lists and ring searches), one lane per point:
// the queue holds only these, so the lanes of a warp do the same kind of work.
template <int D>
__global__ void __launch_bounds__(128, 8) k_assign_overflow(const double* __restrict__ xyz,
                                                         const SampleGrid<D>* __restrict__ sgp,
                                                         const std::uint32_t* __restrict__ starts,
                                                         const SampleRec* __restrict__ sorted,
                                                         const std::uint32_t* __restrict__ sorted_labels,
                                                         const std::uint32_t* __restrict__ heads,
                                                         const std::uint32_t* __restrict__ subheads,
                                                         const VltEntry* __restrict__ lslab,
                                                         std::uint32_t* __restrict__ labels,
                                                         const std::uint32_t* __restrict__ oq,
                                                         const unsigned* __restrict__ oq_count,
                                                         unsigned* __restrict__ next, unsigned* __restrict__ fin) {
  __shared__ SampleGrid<D> sg;
  if (threadIdx.x == 0) sg = *sgp;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u;
  const unsigned cnt = *oq_count;
  for (;;) {
    const unsigned q0 = claim_batch(next);
    if (q0 >= cnt) break;
    const unsigned q = q0 + lane;
    const bool has = q < cnt;
    std::uint32_t i = 0, head = kHeadOverflow;
    double x[D], fcen[D];
    if (has) {
      i = oq[q];
#pragma unroll
      for (int d = 0; d < D; ++d) x[d] = xyz[std::size_t(i) * D + d];
      long long fid = 0;
      vlt_locate<D>(x, sg, heads, subheads, &head, &fid, fcen);
      if ((head & 15u) != kHeadLong) labels[i] = nearest_label_ring<D>(x, sg.g, sg.margin, starts, sorted);
    }
    if (has && (head & 15u) == kHeadLong) {
      // one lane per point, its whole list: the list path's decision
      // (binary32 distances with the rigorous bound; exact binary64 argmin
      // over the undecided entries only when the bounds overlap)
      const VltEntry* ents = lslab + (head >> 4);
      const int ne = static_cast<int>(ents[0].idx);
      ++ents;
      float p[D], pp = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        p[d] = static_cast<float>(x[d] - fcen[d]);
        pp += p[d] * p[d];
      }
      auto dist = [&](const VltEntry& e, float* bnd) {
        float dd = 0.f, ss = 0.f;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const float t = p[d] - e.r[d];
          dd += t * t;
          ss += e.r[d] * e.r[d];
        }
        *bnd = 4e-6f * (pp + ss) + 1e-30f;
        return dd;
      };
      // one pass: the winner (min dd) and the two smallest lower ends dd - bnd
      // (the smallest one not belonging to the winner decides)
      float bv = INFINITY, bb = 0.f, m1 = INFINITY, m2 = INFINITY;
      int bj = 0, j1 = -1;
      for (int j = 0; j < ne; ++j) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(ents + j));
        VltEntry e;
        e.r[0] = q.x;
        e.r[1] = q.y;
        e.r[2] = q.z;
        float bnd;
        const float dd = dist(e, &bnd);
        if (dd < bv) {
          bv = dd;
          bb = bnd;
          bj = j;
        }
        const float lo_end = dd - bnd;
        if (lo_end < m1) {
          m2 = m1;
          m1 = lo_end;
          j1 = j;
        } else if (lo_end < m2) {
          m2 = lo_end;
        }
      }
      const float lim = bv + bb;
      const bool decided = (j1 == bj ? m2 : m1) > lim;
      std::uint32_t lab;
      if (decided) {
        lab = __ldg(sorted_labels + ents[bj].idx);
      } else {
        double best = INFINITY;
        std::uint32_t bpid = 0xFFFFFFFFu;
        lab = 0;
        for (int j = 0; j < ne; ++j) {
          float bnd;
          const float dd = dist(ents[j], &bnd);
          if (j != bj && dd - bnd > lim) continue;
          const SampleRec rec = sorted[ents[j].idx];
          const double d2 = sqdist<D>(x, rec.x);
          if (d2 < best || (d2 == best && rec.pid < bpid)) {
            best = d2;
            bpid = rec.pid;
            lab = rec.label;
          }
        }
      }
      labels[i] = lab;
    }
  }
  rewind_cursor(next, fin, cnt);
}

__global__ void k_sorted_labels(const SampleRec* __restrict__ sorted, std::uint32_t m, std::uint32_t* __restrict__ out) {
  for (std::uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x)
    out[s] = sorted[s].label;
}

}  // namespace sbdt_gpu
