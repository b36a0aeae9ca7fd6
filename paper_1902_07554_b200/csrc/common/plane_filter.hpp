// Box-vs-halfspace filter for the hull rows (halfspace_box_overlap,
// geometry.cpp:329-345): one binary64 plane per hull facet, evaluated at all
// 2^D corners of a box at once, with a rigorous error bound; the exact
// per-corner orient (predicates.hpp) only runs when the filter cannot decide.
//
// Sign convention (predicates.hpp): orient(f_0, .., f_{D-1}, p) =
// sign(n . (p - f_0)), n = (f_1 - f_0) x (f_2 - f_0) in 3-D, n = perp(f_1 - f_0)
// = (-(f_1 - f_0)_y, (f_1 - f_0)_x) in 2-D. A corner is strictly OUTSIDE when
// its orient is neither 0 nor the inner vertex's sign s_in, i.e. when
// w(p) = -s_in * n . (p - f_0) > 0 (s_in != 0).
//
// Error bound (u = 2^-53): with e~ = fl(f_j - f_0), n~ from e~ by one product
// per term and one difference, N~_d = fl(|t1| + |t2|) the absolute-value sum
// of n~_d's two products (3-D; 2-D: N~_d = |n~_d|), q~_d = fl(p_d - f_0,d):
//   |n~_d - n_d| <= 4.1 u N~_d,
//   |fl(sum_d n~_d q~_d) - n . (p - f_0)| <= 8.2 u sum_d N~_d |q~_d|
// (2.01 u per product term + the n~ error + 2.01 u for the two additions).
// The filter evaluates the separable per-axis extremes of w~ -/+ K N~ |q~|
// over the two corner choices of every axis and sums them; K = 4e-15 (~36 u)
// also covers the rounding of those sums (<= 2.01 u of the absolute sums).
// Underflow: an absolute 1e-280 joins the bound (coordinates whose products
// underflow fall back to the exact corners).
#pragma once

#include <cmath>

#include "predicates.hpp"

namespace sbdt_pred {

template <int D>
struct PlaneFilter {
  double f0[D];  // facet vertex 0
  double w[D];   // -s_in * n~ (outside: w . (p - f0) > 0)
  double k[D];   // K * N~ per axis
  bool ok;       // s_in != 0 and a finite plane
};

constexpr double kPlaneK = 4e-15;
constexpr double kPlaneAbs = 1e-280;

template <int D>
SBDT_HD void plane_filter_init(PlaneFilter<D>& pf, const double* const* facet, int inner_sign) {
  for (int d = 0; d < D; ++d) pf.f0[d] = facet[0][d];
  double n[D], N[D];
  if constexpr (D == 2) {
    const double ex = facet[1][0] - facet[0][0], ey = facet[1][1] - facet[0][1];
    n[0] = -ey;
    n[1] = ex;
    N[0] = std::fabs(ey);
    N[1] = std::fabs(ex);
  } else {
    double e1[3], e2[3];
    for (int d = 0; d < 3; ++d) {
      e1[d] = facet[1][d] - facet[0][d];
      e2[d] = facet[2][d] - facet[0][d];
    }
    for (int d = 0; d < 3; ++d) {
      const int i = (d + 1) % 3, j = (d + 2) % 3;
      const double t1 = e1[i] * e2[j], t2 = e1[j] * e2[i];
      n[d] = t1 - t2;
      N[d] = std::fabs(t1) + std::fabs(t2);
    }
  }
  const double s = -static_cast<double>(inner_sign);
  bool fin = inner_sign != 0;
  for (int d = 0; d < D; ++d) {
    pf.w[d] = s * n[d];
    pf.k[d] = kPlaneK * N[d];
    fin = fin && std::isfinite(n[d]) && std::isfinite(N[d]);
  }
  pf.ok = fin;
}

// 0: no corner strictly outside; 2: every corner strictly outside; 1: some
// corners strictly outside and some not; -1: undecided (exact corners).
template <int D>
SBDT_HD int plane_filter_box(const PlaneFilter<D>& pf, const double* blo, const double* bhi) {
  if (!pf.ok) return -1;
  double min_lo = 0.0, max_hi = 0.0, max_lo = 0.0, min_hi = 0.0;
  for (int d = 0; d < D; ++d) {
    const double ql = blo[d] - pf.f0[d], qh = bhi[d] - pf.f0[d];
    const double tl = pf.w[d] * ql, th = pf.w[d] * qh;
    const double el = pf.k[d] * std::fabs(ql), eh = pf.k[d] * std::fabs(qh);
    const double al = tl - el, ah = th - eh, bl = tl + el, bh = th + eh;
    min_lo += al < ah ? al : ah;
    max_lo += al > ah ? al : ah;
    min_hi += bl < bh ? bl : bh;
    max_hi += bl > bh ? bl : bh;
  }
  if (!(min_lo == min_lo) || !(max_hi == max_hi)) return -1;  // NaN
  if (min_lo > kPlaneAbs) return 2;                 // min_p w(p) > 0
  if (max_hi < -kPlaneAbs) return 0;                // max_p w(p) < 0
  if (max_lo > kPlaneAbs && min_hi < -kPlaneAbs) return 1;  // some w > 0 and some w < 0
  return -1;
}

}  // namespace sbdt_pred
