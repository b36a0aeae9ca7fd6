// CPU check of the hull-row plane filter (csrc/common/plane_filter.hpp)
// against the exact per-corner orient of predicates.hpp: random and
// near-degenerate facets and boxes (corners on / next to the plane, wide
// exponent ranges). Every decided box must match the exact corner count
// class (none / some / all strictly outside). Prints counts; exit 1 on any
// mismatch.  Build: g++ -O2 -std=c++20 -ffp-contract=off -I<csrc/common> ...
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <random>

#include "plane_filter.hpp"
#include "predicates.hpp"

using namespace sbdt_pred;

template <int D>
static int exact_class(const double* const* facet, int s_in, const double* lo, const double* hi) {
  const double* pts[D + 1];
  for (int i = 0; i < D; ++i) pts[i] = facet[i];
  double c[D];
  pts[D] = c;
  int out = 0;
  for (unsigned m = 0; m < (1u << D); ++m) {
    for (int d = 0; d < D; ++d) c[d] = (m >> d) & 1 ? hi[d] : lo[d];
    const int s = D == 2 ? orient2(pts[0], pts[1], pts[2]) : orient3(pts[0], pts[1], pts[2], pts[3]);
    if (s != 0 && s != s_in) ++out;
  }
  return out == 0 ? 0 : (out == (1 << D) ? 2 : 1);
}

template <int D>
static bool run(std::uint64_t seed, long cases, long* decided, long* bad) {
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (long t = 0; t < cases; ++t) {
    const int mode = static_cast<int>(t % 4);
    const double scale = mode == 3 ? std::ldexp(1.0, static_cast<int>(g() % 60) - 30) : 1.0;
    double fx[D][D];
    for (int j = 0; j < D; ++j)
      for (int d = 0; d < D; ++d) fx[j][d] = U(g) * scale;
    const double* facet[D];
    for (int j = 0; j < D; ++j) facet[j] = fx[j];
    const int s_in = (g() & 1) ? 1 : -1;
    double lo[D], hi[D];
    if (mode == 1 || mode == 2) {
      // a box with a corner ON the plane (mode 1: a facet vertex) or within a
      // few ulps of it (mode 2: a point of the facet's affine hull, rounded)
      double p[D];
      if (mode == 1) {
        for (int d = 0; d < D; ++d) p[d] = fx[g() % D][d];
      } else {
        const double w1 = U(g), w2 = U(g);
        for (int d = 0; d < D; ++d)
          p[d] = fx[0][d] + w1 * (fx[1][d] - fx[0][d]) + (D == 3 ? w2 * (fx[D - 1][d] - fx[0][d]) : 0.0);
      }
      for (int d = 0; d < D; ++d) {
        const double w = U(g) * scale * 0.1 * (g() % 3 == 0 ? 1e-9 : 1.0);
        if (g() & 1) lo[d] = p[d], hi[d] = p[d] + w;
        else lo[d] = p[d] - w, hi[d] = p[d];
      }
    } else {
      for (int d = 0; d < D; ++d) {
        const double a = U(g) * scale * 1.5 - 0.25 * scale, w = U(g) * scale * 0.3;
        lo[d] = a;
        hi[d] = a + w;
      }
    }
    PlaneFilter<D> pf;
    plane_filter_init<D>(pf, facet, s_in);
    const int f = plane_filter_box<D>(pf, lo, hi);
    if (f < 0) continue;
    ++*decided;
    const int e = exact_class<D>(facet, s_in, lo, hi);
    if (e != f) {
      if (*bad < 5) std::printf("mismatch D=%d case %ld mode %d: filter %d exact %d\n", D, t, mode, f, e);
      ++*bad;
    }
  }
  return *bad == 0;
}

int main(int argc, char** argv) {
  const long cases = argc > 1 ? std::atol(argv[1]) : 200000;
  long dec2 = 0, bad2 = 0, dec3 = 0, bad3 = 0;
  run<2>(11, cases, &dec2, &bad2);
  run<3>(12, cases, &dec3, &bad3);
  std::printf("{\"cases\": %ld, \"decided2\": %ld, \"bad2\": %ld, \"decided3\": %ld, \"bad3\": %ld}\n", cases, dec2,
              bad2, dec3, bad3);
  return (bad2 || bad3) ? 1 : 0;
}
