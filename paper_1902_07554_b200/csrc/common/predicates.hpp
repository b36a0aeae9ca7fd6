// Exact geometric predicates shared by the host setup code (DT builder) and
// the sm_100a kernels.
//
// Semantics follow the reference's predicate contract:
//   orient2/orient3  -> /root/reference/proj/include/sbdt/geometry.hpp:112-121,
//                       /root/reference/proj/src/geometry.cpp:150-189
//   in_sphere2/3     -> geometry.hpp:127-140, geometry.cpp:191-277
//   in_sphere_oriented / tie-broken  -> geometry.hpp:142-166
// Sign conventions: orient3(a,b,c,d) = sign det(b-a, c-a, d-a) (positive for the
// canonical tetrahedron); in_sphere returns +1 strictly inside the
// circumsphere of a positively oriented simplex.
//
// Method: a binary64 evaluation with Shewchuk's static forward-error bounds
// (same constants as geometry.cpp:23-27); when the filter cannot decide, the
// determinant is re-evaluated EXACTLY with floating-point expansion arithmetic
// (Shewchuk 1997: Two-Sum / Two-Product (via an exact fma) / expansion sums).
// This is an independent exact method from the reference's scaled-integer
// fallback (geometry.cpp:32-146); both return the exact sign, so results are
// identical. Translation units including this header must be compiled without
// floating-point contraction (-ffp-contract=off host, -fmad=false device).
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define SBDT_HD __host__ __device__ __forceinline__
#define SBDT_HDN inline __host__ __device__ __noinline__
#else
#define SBDT_HD inline
#define SBDT_HDN inline
#endif

namespace sbdt_pred {

constexpr double kEps = 0x1.0p-53;
constexpr double kCcwBound = (3.0 + 16.0 * kEps) * kEps;
constexpr double kO3dBound = (7.0 + 56.0 * kEps) * kEps;
constexpr double kIccBound = (10.0 + 96.0 * kEps) * kEps;
constexpr double kIspBound = (16.0 + 224.0 * kEps) * kEps;

SBDT_HD double exact_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

// ---- error-free transformations -----------------------------------------
SBDT_HD void two_sum(double a, double b, double& x, double& y) {
  x = a + b;
  const double bv = x - a;
  const double av = x - bv;
  const double br = b - bv;
  const double ar = a - av;
  y = ar + br;
}
SBDT_HD void two_diff(double a, double b, double& x, double& y) {
  x = a - b;
  const double bv = a - x;
  const double av = x + bv;
  const double br = bv - b;
  const double ar = a - av;
  y = ar + br;
}
SBDT_HD void two_product(double a, double b, double& x, double& y) {
  x = a * b;
  y = exact_fma(a, b, -x);
}

// ---- expansion arithmetic (components in increasing magnitude, nonoverlapping)
// h = e + f, zero-eliminated; returns length. h must not alias e or f.
SBDT_HD int expansion_sum(int elen, const double* e, int flen, const double* f, double* h) {
  // Linear merge by magnitude, then a running Two-Sum (Shewchuk's
  // fast_expansion_sum_zeroelim restated).
  if (elen == 0) {
    for (int i = 0; i < flen; ++i) h[i] = f[i];
    return flen;
  }
  if (flen == 0) {
    for (int i = 0; i < elen; ++i) h[i] = e[i];
    return elen;
  }
  double Q, Qnew, hh;
  int ei = 0, fi = 0, hi = 0;
  double enow = e[0], fnow = f[0];
  if ((fnow > enow) == (fnow > -enow)) {
    Q = enow;
    enow = (++ei < elen) ? e[ei] : 0.0;
  } else {
    Q = fnow;
    fnow = (++fi < flen) ? f[fi] : 0.0;
  }
  if (ei < elen && fi < flen) {
    // fast_two_sum for the first merged pair
    if ((fnow > enow) == (fnow > -enow)) {
      Qnew = enow + Q;
      hh = Q - (Qnew - enow);
      enow = (++ei < elen) ? e[ei] : 0.0;
    } else {
      Qnew = fnow + Q;
      hh = Q - (Qnew - fnow);
      fnow = (++fi < flen) ? f[fi] : 0.0;
    }
    Q = Qnew;
    if (hh != 0.0) h[hi++] = hh;
    while (ei < elen && fi < flen) {
      if ((fnow > enow) == (fnow > -enow)) {
        two_sum(Q, enow, Qnew, hh);
        enow = (++ei < elen) ? e[ei] : 0.0;
      } else {
        two_sum(Q, fnow, Qnew, hh);
        fnow = (++fi < flen) ? f[fi] : 0.0;
      }
      Q = Qnew;
      if (hh != 0.0) h[hi++] = hh;
    }
  }
  while (ei < elen) {
    two_sum(Q, enow, Qnew, hh);
    enow = (++ei < elen) ? e[ei] : 0.0;
    Q = Qnew;
    if (hh != 0.0) h[hi++] = hh;
  }
  while (fi < flen) {
    two_sum(Q, fnow, Qnew, hh);
    fnow = (++fi < flen) ? f[fi] : 0.0;
    Q = Qnew;
    if (hh != 0.0) h[hi++] = hh;
  }
  if (Q != 0.0 || hi == 0) h[hi++] = Q;
  return hi;
}

// h = b * e, zero-eliminated; returns length (<= 2*elen). h must not alias e.
SBDT_HD int scale_expansion(int elen, const double* e, double b, double* h) {
  double Q, sum, hh, p1, p0;
  int hi = 0;
  two_product(e[0], b, Q, hh);
  if (hh != 0.0) h[hi++] = hh;
  for (int i = 1; i < elen; ++i) {
    two_product(e[i], b, p1, p0);
    two_sum(Q, p0, sum, hh);
    if (hh != 0.0) h[hi++] = hh;
    // fast_two_sum(p1, sum): |p1| >= |sum| holds here
    Q = p1 + sum;
    hh = sum - (Q - p1);
    if (hh != 0.0) h[hi++] = hh;
  }
  if (Q != 0.0 || hi == 0) h[hi++] = Q;
  return hi;
}

// h = e * f using tmp (size >= 2*elen) and acc scratch (size >= 2*elen*flen);
// result written to h (size >= 2*elen*flen). Returns length.
SBDT_HD int mul_expansion(int elen, const double* e, int flen, const double* f, double* h,
                          double* tmp, double* acc) {
  int hlen = 0;
  for (int j = 0; j < flen; ++j) {
    const int tlen = scale_expansion(elen, e, f[j], tmp);
    const int n = expansion_sum(hlen, h, tlen, tmp, acc);
    for (int i = 0; i < n; ++i) h[i] = acc[i];
    hlen = n;
  }
  return hlen;
}

SBDT_HD int expansion_sign(int len, const double* e) {
  for (int i = len - 1; i >= 0; --i) {
    if (e[i] > 0.0) return 1;
    if (e[i] < 0.0) return -1;
  }
  return 0;
}

SBDT_HD void negate(int len, double* e) {
  for (int i = 0; i < len; ++i) e[i] = -e[i];
}

// ---- exact determinants over 2-term differences ----------------------------
// d[i] = (hi, lo) exact difference.
struct Diff2 {
  double v[2];  // v[0] = low component, v[1] = high component
};
SBDT_HD Diff2 exact_diff(double a, double b) {
  Diff2 d;
  two_diff(a, b, d.v[1], d.v[0]);
  return d;
}
SBDT_HD int diff_len(const Diff2& d, double* out) {
  int n = 0;
  if (d.v[0] != 0.0) out[n++] = d.v[0];
  out[n++] = d.v[1];
  return n;
}

// Exact 2x2 minor  a*d - b*c  with 2-term entries. out size >= 16.
SBDT_HD int minor2(const Diff2& a, const Diff2& b, const Diff2& c, const Diff2& d, double* out) {
  double ea[2], eb[2], ec[2], ed[2];
  const int la = diff_len(a, ea), lb = diff_len(b, eb), lc = diff_len(c, ec), ld = diff_len(d, ed);
  double p[8], q[8], tmp[4], acc[8];
  const int lp = mul_expansion(la, ea, ld, ed, p, tmp, acc);
  const int lq = mul_expansion(lb, eb, lc, ec, q, tmp, acc);
  negate(lq, q);
  return expansion_sum(lp, p, lq, q, out);
}

// Exact orient2 sign (geometry.cpp:150-170 contract): sign of
// (a-c)x (b-c)y - (a-c)y (b-c)x.
SBDT_HDN int orient2_exact(const double* a, const double* b, const double* c) {
  const Diff2 acx = exact_diff(a[0], c[0]), acy = exact_diff(a[1], c[1]);
  const Diff2 bcx = exact_diff(b[0], c[0]), bcy = exact_diff(b[1], c[1]);
  double out[16];
  const int n = minor2(acx, acy, bcx, bcy, out);
  return expansion_sign(n, out);
}

SBDT_HD int orient2(const double* a, const double* b, const double* c) {
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
  return orient2_exact(a, b, c);
}

// Exact 3x3 determinant of rows r0,r1,r2 (2-term entries). out size >= 192.
// scratch size >= 512.
SBDT_HD int det3_exact(const Diff2 r[3][3], double* out, double* scratch) {
  // cofactor expansion along row 0: r00*M00 - r01*M01 + r02*M02
  double* m = scratch;            // 16
  double* term = scratch + 16;    // 64
  double* tmp = scratch + 80;     // 32
  double* acc = scratch + 112;    // 192
  double* acc2 = scratch + 304;   // 192
  int outlen = 0;
  for (int j = 0; j < 3; ++j) {
    const int c1 = (j == 0) ? 1 : 0;
    const int c2 = (j == 2) ? 1 : 2;
    const int ml = minor2(r[1][c1], r[1][c2], r[2][c1], r[2][c2], m);
    double e[2];
    const int el = diff_len(r[0][j], e);
    const int tl = mul_expansion(ml, m, el, e, term, tmp, acc);
    if (j == 1) negate(tl, term);
    const int n = expansion_sum(outlen, out, tl, term, acc2);
    for (int i = 0; i < n; ++i) out[i] = acc2[i];
    outlen = n;
  }
  return outlen;
}

// orient3 = sign det(b-a, c-a, d-a)  (geometry.hpp:112-121 convention).
SBDT_HDN int orient3_exact(const double* a, const double* b, const double* c, const double* d) {
  Diff2 r[3][3];
  for (int k = 0; k < 3; ++k) {
    r[0][k] = exact_diff(b[k], a[k]);
    r[1][k] = exact_diff(c[k], a[k]);
    r[2][k] = exact_diff(d[k], a[k]);
  }
  double out[192];
  double scratch[512];
  const int n = det3_exact(r, out, scratch);
  return expansion_sign(n, out);
}

SBDT_HD int orient3(const double* a, const double* b, const double* c, const double* d) {
  const double adx = a[0] - d[0], ady = a[1] - d[1], adz = a[2] - d[2];
  const double bdx = b[0] - d[0], bdy = b[1] - d[1], bdz = b[2] - d[2];
  const double cdx = c[0] - d[0], cdy = c[1] - d[1], cdz = c[2] - d[2];
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double det = adz * (bdxcdy - cdxbdy) + bdz * (cdxady - adxcdy) + cdz * (adxbdy - bdxady);
  const double permanent = (fabs(bdxcdy) + fabs(cdxbdy)) * fabs(adz) +
                           (fabs(cdxady) + fabs(adxcdy)) * fabs(bdz) +
                           (fabs(adxbdy) + fabs(bdxady)) * fabs(cdz);
  const double errbound = kO3dBound * permanent;
  // det(a-d,b-d,c-d) has the opposite sign of det(b-a,c-a,d-a).
  if (det > errbound) return -1;
  if (-det > errbound) return 1;
  return orient3_exact(a, b, c, d);
}

// ---- in_sphere exact (host + escalation kernels) ---------------------------
// Scratch requirement for in_sphere2_exact: kInSphere2Scratch doubles.
constexpr int kInSphere2Scratch = 8192;
// in_sphere2 = sign det [[p_i - q, |p_i - q|^2]] for the three rows.
SBDT_HDN int in_sphere2_exact_buf(const double* a, const double* b, const double* c,
                                  const double* q, double* buf) {
  const double* pts[3] = {a, b, c};
  Diff2 dx[3], dy[3];
  for (int i = 0; i < 3; ++i) {
    dx[i] = exact_diff(pts[i][0], q[0]);
    dy[i] = exact_diff(pts[i][1], q[1]);
  }
  double* lift = buf;          // 16
  double* minor = buf + 16;    // 16
  double* term = buf + 32;     // 512
  double* tmp = buf + 544;     // 32
  double* acc = buf + 576;     // 2048
  double* res = buf + 2624;    // 1600
  double* res2 = buf + 4224;   // 1600
  double* sq1 = buf + 5824;    // 8
  double* sq2 = buf + 5832;    // 8
  int rlen = 0;
  for (int i = 0; i < 3; ++i) {
    double ex[2], ey[2];
    const int lx = diff_len(dx[i], ex), ly = diff_len(dy[i], ey);
    double t4[4], a8[8];
    const int l1 = mul_expansion(lx, ex, lx, ex, sq1, t4, a8);
    const int l2 = mul_expansion(ly, ey, ly, ey, sq2, t4, a8);
    const int ll = expansion_sum(l1, sq1, l2, sq2, lift);
    const int j = (i + 1) % 3, k = (i + 2) % 3;
    // cyclic cofactor: lift_i * (dx_j*dy_k - dx_k*dy_j)
    const int ml = minor2(dx[j], dy[j], dx[k], dy[k], minor);
    const int tl = mul_expansion(ll, lift, ml, minor, term, tmp, acc);
    const int n = expansion_sum(rlen, res, tl, term, res2);
    for (int t = 0; t < n; ++t) res[t] = res2[t];
    rlen = n;
  }
  return expansion_sign(rlen, res);
}

SBDT_HD int in_sphere2_filtered(const double* a, const double* b, const double* c,
                                const double* q) {
  const double adx = a[0] - q[0], ady = a[1] - q[1];
  const double bdx = b[0] - q[0], bdy = b[1] - q[1];
  const double cdx = c[0] - q[0], cdy = c[1] - q[1];
  const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
  const double cdxady = cdx * ady, adxcdy = adx * cdy;
  const double adxbdy = adx * bdy, bdxady = bdx * ady;
  const double alift = adx * adx + ady * ady;
  const double blift = bdx * bdx + bdy * bdy;
  const double clift = cdx * cdx + cdy * cdy;
  const double det =
      alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) + clift * (adxbdy - bdxady);
  const double permanent = (fabs(bdxcdy) + fabs(cdxbdy)) * alift +
                           (fabs(cdxady) + fabs(adxcdy)) * blift +
                           (fabs(adxbdy) + fabs(bdxady)) * clift;
  const double errbound = kIccBound * permanent;
  if (det > errbound) return 1;
  if (-det > errbound) return -1;
  return 2;  // undecided
}

// in_sphere3 exact: -sign det M, M rows (p_i - q | lift_i)  (geometry.cpp:130-146).
constexpr int kInSphere3Scratch = 131072;
SBDT_HDN int in_sphere3_exact_buf(const double* a, const double* b, const double* c,
                                  const double* d, const double* q, double* buf) {
  const double* pts[4] = {a, b, c, d};
  Diff2 df[4][3];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k) df[i][k] = exact_diff(pts[i][k], q[k]);
  double* lift = buf;           // 24
  double* sq = buf + 32;        // 8
  double* acc8 = buf + 40;      // 24
  double* minor = buf + 64;     // 192
  double* scratch = buf + 256;  // 512
  double* term = buf + 768;     // 9216
  double* tmp = buf + 9984;     // 64
  double* acc = buf + 10048;    // 9216
  double* res = buf + 19264;    // 40000
  double* res2 = buf + 59264;   // 40000
  int rlen = 0;
  for (int i = 0; i < 4; ++i) {
    int ll = 0;
    for (int k = 0; k < 3; ++k) {
      double e[2] = {0.0, 0.0}, t4[4], a8[8];
      const int l = diff_len(df[i][k], e);
      const int sl = mul_expansion(l, e, l, e, sq, t4, a8);
      const int n = expansion_sum(ll, lift, sl, sq, acc8);
      for (int t = 0; t < n; ++t) lift[t] = acc8[t];
      ll = n;
    }
    // minor = det of the other three rows' xyz.
    Diff2 r[3][3];
    int rr = 0;
    for (int j = 0; j < 4; ++j) {
      if (j == i) continue;
      for (int k = 0; k < 3; ++k) r[rr][k] = df[j][k];
      ++rr;
    }
    const int ml = det3_exact(r, minor, scratch);
    const int tl = mul_expansion(ll, lift, ml, minor, term, tmp, acc);
    // Expansion along the lift column (column 3): sign (-1)^(i+3).
    if (((i + 3) & 1) != 0) negate(tl, term);
    const int n = expansion_sum(rlen, res, tl, term, res2);
    for (int t = 0; t < n; ++t) res[t] = res2[t];
    rlen = n;
  }
  return -expansion_sign(rlen, res);
}

SBDT_HD int in_sphere3_filtered(const double* a, const double* b, const double* c,
                                const double* d, const double* q) {
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
  const double ab = aexbey - bexaey;
  const double bc = bexcey - cexbey;
  const double cd = cexdey - dexcey;
  const double da = dexaey - aexdey;
  const double ac = aexcey - cexaey;
  const double bd = bexdey - dexbey;
  const double abc = aez * bc - bez * ac + cez * ab;
  const double bcd = bez * cd - cez * bd + dez * bc;
  const double cda = cez * da + dez * ac + aez * cd;
  const double dab = dez * ab + aez * bd + bez * da;
  const double alift = aex * aex + aey * aey + aez * aez;
  const double blift = bex * bex + bey * bey + bez * bez;
  const double clift = cex * cex + cey * cey + cez * cez;
  const double dlift = dex * dex + dey * dey + dez * dez;
  const double det = (dlift * abc - clift * dab) + (blift * cda - alift * bcd);
  const double aezp = fabs(aez), bezp = fabs(bez), cezp = fabs(cez), dezp = fabs(dez);
  const double aexbeyp = fabs(aexbey), bexaeyp = fabs(bexaey);
  const double bexceyp = fabs(bexcey), cexbeyp = fabs(cexbey);
  const double cexdeyp = fabs(cexdey), dexceyp = fabs(dexcey);
  const double dexaeyp = fabs(dexaey), aexdeyp = fabs(aexdey);
  const double aexceyp = fabs(aexcey), cexaeyp = fabs(cexaey);
  const double bexdeyp = fabs(bexdey), dexbeyp = fabs(dexbey);
  const double permanent =
      ((cexdeyp + dexceyp) * bezp + (dexbeyp + bexdeyp) * cezp + (bexceyp + cexbeyp) * dezp) *
          alift +
      ((dexaeyp + aexdeyp) * cezp + (aexceyp + cexaeyp) * dezp + (cexdeyp + dexceyp) * aezp) *
          blift +
      ((aexbeyp + bexaeyp) * dezp + (bexdeyp + dexbeyp) * aezp + (dexaeyp + aexdeyp) * bezp) *
          clift +
      ((bexceyp + cexbeyp) * aezp + (cexaeyp + aexceyp) * bezp + (aexbeyp + bexaeyp) * cezp) *
          dlift;
  const double errbound = kIspBound * permanent;
  if (det > errbound) return -1;
  if (-det > errbound) return 1;
  return 2;  // undecided
}

}  // namespace sbdt_pred
