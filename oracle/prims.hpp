// TEST INFRASTRUCTURE (oracle) — CPU restatement of the reference's geometry
// primitives on the hot path. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may use anything under oracle/.
//
// Every function restates the cited reference code; compile with
// -ffp-contract=off so binary64 results are bit-identical to the reference's
// and to the GPU's.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>

#include "bigint.hpp"

namespace sbdt_oracle {

using sbdt_bigint::BigInt;

template <int D>
using Vec = std::array<double, D>;

template <int D>
struct Sphere {
  Vec<D> center;
  double radius_squared;
};

template <int D>
struct Box {
  Vec<D> lo, hi;
};

struct DegenerateSimplex : std::runtime_error {
  DegenerateSimplex() : std::runtime_error("degenerate simplex") {}
};

// geometry.hpp:102-110 — left-to-right sum of squared differences.
template <int D>
inline double squared_distance(const double* a, const double* b) {
  double s = 0;
  for (int d = 0; d < D; ++d) {
    const double t = a[d] - b[d];
    s += t * t;
  }
  return s;
}

namespace detail {
constexpr double kEps = 0x1.0p-53;
const double kCcwBound = (3.0 + 16.0 * kEps) * kEps;
const double kO3dBound = (7.0 + 56.0 * kEps) * kEps;
const double kIccBound = (10.0 + 96.0 * kEps) * kEps;
const double kIspBound = (16.0 + 224.0 * kEps) * kEps;

// geometry.cpp:32-56 — common power-of-two scaling to exact integers.
struct Scaler {
  int min_exp = 0;
  template <std::size_t N>
  explicit Scaler(const std::array<double, N>& vals) {
    bool any = false;
    for (double v : vals)
      if (v != 0.0) {
        const int e = std::ilogb(v);
        min_exp = any ? std::min(min_exp, e) : e;
        any = true;
      }
  }
  BigInt operator()(double v) const {
    if (v == 0.0) return BigInt(0);
    const int e = std::ilogb(v);
    BigInt r(static_cast<long long>(std::scalbn(v, 52 - e)));
    r <<= (e - min_exp);
    return r;
  }
};
inline BigInt det2(const BigInt& a, const BigInt& b, const BigInt& c, const BigInt& d) {
  return a * d - b * c;
}
inline BigInt det3(const BigInt m[9]) {
  return m[0] * det2(m[4], m[5], m[7], m[8]) - m[1] * det2(m[3], m[5], m[6], m[8]) +
         m[2] * det2(m[3], m[4], m[6], m[7]);
}
}  // namespace detail

// geometry.cpp:150-170 (+ exact fallback :92-97)
inline int orient2(const double* a, const double* b, const double* c) {
  using namespace detail;
  const double detleft = (a[0] - c[0]) * (b[1] - c[1]);
  const double detright = (a[1] - c[1]) * (b[0] - c[0]);
  const double det = detleft - detright;
  double detsum;
  if (detleft > 0.0) {
    if (detright <= 0.0) return det > 0 ? 1 : (det < 0 ? -1 : 0);
    detsum = detleft + detright;
  } else if (detleft < 0.0) {
    if (detright >= 0.0) return det > 0 ? 1 : (det < 0 ? -1 : 0);
    detsum = -detleft - detright;
  } else {
    return det > 0 ? 1 : (det < 0 ? -1 : 0);
  }
  const double errbound = kCcwBound * detsum;
  if (det >= errbound) return 1;
  if (-det >= errbound) return -1;
  Scaler s(std::array<double, 6>{a[0], a[1], b[0], b[1], c[0], c[1]});
  const BigInt ax = s(a[0]), ay = s(a[1]);
  return det2(s(b[0]) - ax, s(b[1]) - ay, s(c[0]) - ax, s(c[1]) - ay).sign();
}

// geometry.cpp:172-189 (+ exact fallback :99-108); sign det(b-a, c-a, d-a).
inline int orient3(const double* a, const double* b, const double* c, const double* d) {
  using namespace detail;
  const double adx = a[0] - d[0], ady = a[1] - d[1], adz = a[2] - d[2];
  const double bdx = b[0] - d[0], bdy = b[1] - d[1], bdz = b[2] - d[2];
  const double cdx = c[0] - d[0], cdy = c[1] - d[1], cdz = c[2] - d[2];
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double det = adz * (bdxcdy - cdxbdy) + bdz * (cdxady - adxcdy) + cdz * (adxbdy - bdxady);
  const double permanent = (std::fabs(bdxcdy) + std::fabs(cdxbdy)) * std::fabs(adz) +
                           (std::fabs(cdxady) + std::fabs(adxcdy)) * std::fabs(bdz) +
                           (std::fabs(adxbdy) + std::fabs(bdxady)) * std::fabs(cdz);
  const double errbound = kO3dBound * permanent;
  if (det > errbound) return -1;
  if (-det > errbound) return 1;
  Scaler s(std::array<double, 12>{a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]});
  BigInt m[9];
  const double* rows[3] = {b, c, d};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[3 * i + j] = s(rows[i][j]) - s(a[j]);
  return det3(m).sign();
}

template <int D>
inline int orient(const double* const* p) {
  if constexpr (D == 2) return orient2(p[0], p[1], p[2]);
  else return orient3(p[0], p[1], p[2], p[3]);
}

// geometry.cpp:191-212 (+ :110-125)
inline int in_sphere2(const double* a, const double* b, const double* c, const double* q) {
  using namespace detail;
  const double adx = a[0] - q[0], ady = a[1] - q[1];
  const double bdx = b[0] - q[0], bdy = b[1] - q[1];
  const double cdx = c[0] - q[0], cdy = c[1] - q[1];
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double alift = adx * adx + ady * ady;
  const double blift = bdx * bdx + bdy * bdy;
  const double clift = cdx * cdx + cdy * cdy;
  const double det = alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) + clift * (adxbdy - bdxady);
  const double permanent = (std::fabs(bdxcdy) + std::fabs(cdxbdy)) * alift +
                           (std::fabs(cdxady) + std::fabs(adxcdy)) * blift +
                           (std::fabs(adxbdy) + std::fabs(bdxady)) * clift;
  const double errbound = kIccBound * permanent;
  if (det > errbound) return 1;
  if (-det > errbound) return -1;
  Scaler s(std::array<double, 8>{a[0], a[1], b[0], b[1], c[0], c[1], q[0], q[1]});
  const BigInt qx = s(q[0]), qy = s(q[1]);
  BigInt m[9];
  const double* rows[3] = {a, b, c};
  for (int i = 0; i < 3; ++i) {
    const BigInt dx = s(rows[i][0]) - qx, dy = s(rows[i][1]) - qy;
    m[3 * i] = dx;
    m[3 * i + 1] = dy;
    m[3 * i + 2] = dx * dx + dy * dy;
  }
  return det3(m).sign();
}

// geometry.cpp:214-277 (+ :127-146)
inline int in_sphere3(const double* a, const double* b, const double* c, const double* d,
                      const double* q) {
  using namespace detail;
  const double aex = a[0] - q[0], aey = a[1] - q[1], aez = a[2] - q[2];
  const double bex = b[0] - q[0], bey = b[1] - q[1], bez = b[2] - q[2];
  const double cex = c[0] - q[0], cey = c[1] - q[1], cez = c[2] - q[2];
  const double dex = d[0] - q[0], dey = d[1] - q[1], dez = d[2] - q[2];
  const double aexbey = aex * bey, bexaey = bex * aey;
  const double bexcey = bex * cey, cexbey = cex * bey;
  const double cexdey = cex * dey, dexcey = dex * cey;
  const double dexaey = dex * aey, aexdey = aex * dey;
  const double aexcey = aex * cey, cexaey = cex * aey;
  const double bexdey = bex * dey, dexbey = dex * bey;
  const double ab = aexbey - bexaey, bc = bexcey - cexbey, cd = cexdey - dexcey;
  const double da = dexaey - aexdey, ac = aexcey - cexaey, bd = bexdey - dexbey;
  const double abc = aez * bc - bez * ac + cez * ab;
  const double bcd = bez * cd - cez * bd + dez * bc;
  const double cda = cez * da + dez * ac + aez * cd;
  const double dab = dez * ab + aez * bd + bez * da;
  const double alift = aex * aex + aey * aey + aez * aez;
  const double blift = bex * bex + bey * bey + bez * bez;
  const double clift = cex * cex + cey * cey + cez * cez;
  const double dlift = dex * dex + dey * dey + dez * dez;
  const double det = (dlift * abc - clift * dab) + (blift * cda - alift * bcd);
  const double A = std::fabs(aez), B = std::fabs(bez), C = std::fabs(cez), Dz = std::fabs(dez);
  const double p_ab = std::fabs(aexbey) + std::fabs(bexaey), p_bc = std::fabs(bexcey) + std::fabs(cexbey);
  const double p_cd = std::fabs(cexdey) + std::fabs(dexcey), p_da = std::fabs(dexaey) + std::fabs(aexdey);
  const double p_ac = std::fabs(aexcey) + std::fabs(cexaey), p_bd = std::fabs(bexdey) + std::fabs(dexbey);
  const double permanent = (p_cd * B + p_bd * C + p_bc * Dz) * alift + (p_da * C + p_ac * Dz + p_cd * A) * blift +
                           (p_ab * Dz + p_bd * A + p_da * B) * clift + (p_bc * A + p_ac * B + p_ab * C) * dlift;
  const double errbound = kIspBound * permanent;
  if (det > errbound) return -1;
  if (-det > errbound) return 1;
  Scaler s(std::array<double, 15>{a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2],
                                   q[0], q[1], q[2]});
  const BigInt qx = s(q[0]), qy = s(q[1]), qz = s(q[2]);
  BigInt m[16];
  const double* rows[4] = {a, b, c, d};
  for (int i = 0; i < 4; ++i) {
    const BigInt dx = s(rows[i][0]) - qx, dy = s(rows[i][1]) - qy, dz = s(rows[i][2]) - qz;
    m[4 * i] = dx;
    m[4 * i + 1] = dy;
    m[4 * i + 2] = dz;
    m[4 * i + 3] = dx * dx + dy * dy + dz * dz;
  }
  BigInt r = 0;
  for (int j = 0; j < 4; ++j) {
    BigInt minor[9];
    int idx = 0;
    for (int row = 1; row < 4; ++row)
      for (int col = 0; col < 4; ++col)
        if (col != j) minor[idx++] = m[4 * row + col];
    const BigInt term = m[j] * det3(minor);
    if (j % 2 == 0) r += term;
    else r -= term;
  }
  return -r.sign();
}

// geometry.hpp:142-151 — in_sphere on a stored (ascending-id) simplex.
template <int D>
inline int in_sphere_oriented(const double* const* p, int parity, const double* q) {
  const double* a = p[0];
  const double* b = p[1];
  if (parity != 1) std::swap(a, b);
  if constexpr (D == 2) return in_sphere2(a, b, p[2], q);
  else return in_sphere3(a, b, p[2], p[3], q);
}

// geometry.cpp:279-296 — Cramer's rule on the 2x2 bisector system, relative to p0.
inline Sphere<2> circumsphere2(const double* p0, const double* p1, const double* p2) {
  if (orient2(p0, p1, p2) == 0) throw DegenerateSimplex();
  const double ux = p1[0] - p0[0], uy = p1[1] - p0[1];
  const double vx = p2[0] - p0[0], vy = p2[1] - p0[1];
  const double bu = 0.5 * (ux * ux + uy * uy);
  const double bv = 0.5 * (vx * vx + vy * vy);
  const double det = ux * vy - uy * vx;
  const double cx = (bu * vy - bv * uy) / det;
  const double cy = (ux * bv - vx * bu) / det;
  Sphere<2> s;
  s.center = {p0[0] + cx, p0[1] + cy};
  s.radius_squared = cx * cx + cy * cy;
  return s;
}

// geometry.cpp:298-327 — Cramer's rule on the 3x3 bisector system, relative to p0.
inline Sphere<3> circumsphere3(const double* p0, const double* p1, const double* p2, const double* p3) {
  if (orient3(p0, p1, p2, p3) == 0) throw DegenerateSimplex();
  const double* p[4] = {p0, p1, p2, p3};
  double m[3][3], rhs[3];
  for (int i = 0; i < 3; ++i) {
    double n2 = 0;
    for (int d = 0; d < 3; ++d) {
      m[i][d] = p[i + 1][d] - p[0][d];
      n2 += m[i][d] * m[i][d];
    }
    rhs[i] = 0.5 * n2;
  }
  auto det3x3 = [](const double a[3][3]) {
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
           a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
  };
  const double det = det3x3(m);
  double rel[3];
  for (int col = 0; col < 3; ++col) {
    double mc[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) mc[i][j] = (j == col) ? rhs[i] : m[i][j];
    rel[col] = det3x3(mc) / det;
  }
  Sphere<3> s;
  for (int d = 0; d < 3; ++d) s.center[d] = p0[d] + rel[d];
  s.radius_squared = rel[0] * rel[0] + rel[1] * rel[1] + rel[2] * rel[2];
  return s;
}

template <int D>
inline Sphere<D> circumsphere(const double* const* p) {
  if constexpr (D == 2) return circumsphere2(p[0], p[1], p[2]);
  else return circumsphere3(p[0], p[1], p[2], p[3]);
}

// geometry.hpp:175-183
constexpr double kCircumsphereInflation = 1e-10;
template <int D>
inline Sphere<D> inflated(Sphere<D> s) {
  s.radius_squared *= (1.0 + kCircumsphereInflation);
  return s;
}

// geometry.hpp:185-201
template <int D>
inline bool box_sphere_overlap(const Box<D>& box, const Sphere<D>& sphere) {
  double d2 = 0;
  for (int d = 0; d < D; ++d) {
    const double c = sphere.center[d];
    double g = 0;
    if (c < box.lo[d]) g = box.lo[d] - c;
    else if (c > box.hi[d]) g = c - box.hi[d];
    d2 += g * g;
  }
  return d2 <= sphere.radius_squared;
}

// geometry.cpp:329-345 — some box corner strictly on the non-inner side.
template <int D>
inline bool halfspace_box_overlap(const double* const* facet, const double* inner, const Box<D>& box) {
  const double* pts[D + 1];
  for (int i = 0; i < D; ++i) pts[i] = facet[i];
  pts[D] = inner;
  const int inner_sign = orient<D>(pts);
  double corner[D];
  pts[D] = corner;
  for (unsigned c = 0; c < (1u << D); ++c) {
    for (int d = 0; d < D; ++d) corner[d] = (c & (1u << d)) ? box.hi[d] : box.lo[d];
    const int s = orient<D>(pts);
    if (s != 0 && s != inner_sign) return true;
  }
  return false;
}

// Policy object used by the path templates (oracle/path.hpp): the oracle's
// own restated primitives. oracle/ref/ref_glue.cpp instantiates the same
// templates with the reference's compiled primitives to pin this restatement.
template <int D>
struct OwnPrims {
  static Sphere<D> sphere(const double* const* p) { return inflated<D>(circumsphere<D>(p)); }
  static bool box_sphere(const Box<D>& b, const Sphere<D>& s) { return box_sphere_overlap<D>(b, s); }
  static bool halfspace_box(const double* const* f, const double* inner, const Box<D>& b) {
    return halfspace_box_overlap<D>(f, inner, b);
  }
  static int orient_pts(const double* const* p) { return orient<D>(p); }
  static int in_sphere_or(const double* const* p, int parity, const double* q) {
    return in_sphere_oriented<D>(p, parity, q);
  }
  static double sqdist(const double* a, const double* b) { return squared_distance<D>(a, b); }
};

}  // namespace sbdt_oracle
