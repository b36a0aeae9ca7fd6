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

// ---- wide exponent ranges: scaled big integers ------------------------------
// Expansion arithmetic is exact only while no product underflows or
// overflows. Every component of a degree-g homogeneous determinant of
// coordinate differences is a multiple of 2^(g (emin - 52)) (emin: the smallest
// exponent of a nonzero input) and below 2^(g (emax + 1) + 8), so it is exact
// when those fit binary64 (after an exact power-of-two prescale of all
// inputs, which leaves every sign unchanged). Inputs whose exponents span
// more than that (e.g. 5.0 next to 5e-324) take the reference's own method
// (ExactScaler, geometry.cpp:28-55): every value becomes the integer
// mantissa * 2^(e - emin) and the determinant is evaluated in big integers.

// Power-of-two prescale exponent for a degree-g determinant, or kNoScale.
constexpr int kNoScale = 1 << 30;
SBDT_HD int prescale_exponent(const double* v, int count, int g) {
  int emin = 1 << 20, emax = -(1 << 20);
  for (int i = 0; i < count; ++i) {
    if (v[i] == 0.0) continue;
    const int e = ilogb(v[i]);
    emin = e < emin ? e : emin;
    emax = e > emax ? e : emax;
  }
  if (emax < emin) return 0;  // all zero
  // need g (emin + s - 52) >= -1074 + 53 (a margin: the lowest product bits
  // stay above the subnormal range) and g (emax + s + 1) + 8 <= 1000
  const int lo_need = 52 + (-1021 + g - 1) / g + 1 - emin;  // ceil((-1021) / g), rounded up once more
  const int hi_allow = (1000 - 8) / g - 1 - emax;
  if (lo_need > hi_allow) return kNoScale;
  if (lo_need > 0) return lo_need;
  if (hi_allow < 0) return hi_allow;
  return 0;
}

// Signed-magnitude big integer over 32-bit limbs in caller storage.
struct Big {
  std::uint32_t* d;
  int n;    // limbs in use (no leading zero limb); 0 = zero
  int neg;  // 1 = negative
};

SBDT_HD int big_sign(const Big& a) { return a.n == 0 ? 0 : (a.neg ? -1 : 1); }

SBDT_HD int min_exponent(const double* v, int count) {
  int emin = 1 << 20;
  for (int i = 0; i < count; ++i)
    if (v[i] != 0.0) {
      const int e = ilogb(v[i]);
      emin = e < emin ? e : emin;
    }
  return emin == (1 << 20) ? 0 : emin;
}

// r = v * 2^(52 - emin) as an integer: mantissa(v) << (ilogb(v) - emin).
SBDT_HD void big_scaled(Big& r, double v, int emin) {
  r.n = 0;
  r.neg = v < 0.0;
  if (v == 0.0) return;
  const int e = ilogb(v);
  const std::uint64_t m = static_cast<std::uint64_t>(fabs(scalbn(v, 52 - e)));
  const int shift = e - emin;
  const int w = shift >> 5, b = shift & 31;
  for (int i = 0; i < w; ++i) r.d[i] = 0u;
  const std::uint64_t lo = m << b;                     // bits [b, 64)
  const std::uint64_t hi = b ? (m >> (64 - b)) : 0u;  // the bits shifted out
  r.d[w] = static_cast<std::uint32_t>(lo);
  r.d[w + 1] = static_cast<std::uint32_t>(lo >> 32);
  r.d[w + 2] = static_cast<std::uint32_t>(hi);
  r.n = w + 3;
  while (r.n > 0 && r.d[r.n - 1] == 0u) --r.n;
}

SBDT_HD int big_cmp_mag(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
  return 0;
}

// r = a + (negb ? -b : b); r must not alias a or b.
SBDT_HD void big_add(Big& r, const Big& a, const Big& b, int negb) {
  const int bneg = b.neg ^ negb;
  if (b.n == 0) {
    for (int i = 0; i < a.n; ++i) r.d[i] = a.d[i];
    r.n = a.n, r.neg = a.neg;
    return;
  }
  if (a.n == 0) {
    for (int i = 0; i < b.n; ++i) r.d[i] = b.d[i];
    r.n = b.n, r.neg = bneg;
    return;
  }
  if (a.neg == bneg) {  // magnitudes add
    const int n = a.n > b.n ? a.n : b.n;
    std::uint64_t c = 0;
    for (int i = 0; i < n; ++i) {
      c += std::uint64_t(i < a.n ? a.d[i] : 0u) + (i < b.n ? b.d[i] : 0u);
      r.d[i] = static_cast<std::uint32_t>(c);
      c >>= 32;
    }
    r.n = n;
    if (c) r.d[r.n++] = static_cast<std::uint32_t>(c);
    r.neg = a.neg;
    return;
  }
  const int cmp = big_cmp_mag(a, b);
  if (cmp == 0) {
    r.n = 0, r.neg = 0;
    return;
  }
  const Big& x = cmp > 0 ? a : b;  // larger magnitude
  const Big& y = cmp > 0 ? b : a;
  std::int64_t br = 0;
  for (int i = 0; i < x.n; ++i) {
    std::int64_t t = std::int64_t(x.d[i]) - (i < y.n ? std::int64_t(y.d[i]) : 0) - br;
    br = t < 0;
    r.d[i] = static_cast<std::uint32_t>(t + (br << 32));
  }
  r.n = x.n;
  while (r.n > 0 && r.d[r.n - 1] == 0u) --r.n;
  r.neg = cmp > 0 ? a.neg : bneg;
}

// r = a * b (schoolbook); r must not alias a or b.
SBDT_HD void big_mul(Big& r, const Big& a, const Big& b) {
  if (a.n == 0 || b.n == 0) {
    r.n = 0, r.neg = 0;
    return;
  }
  const int n = a.n + b.n;
  for (int i = 0; i < n; ++i) r.d[i] = 0u;
  for (int i = 0; i < a.n; ++i) {
    std::uint64_t c = 0;
    for (int j = 0; j < b.n; ++j) {
      c += std::uint64_t(a.d[i]) * b.d[j] + r.d[i + j];
      r.d[i + j] = static_cast<std::uint32_t>(c);
      c >>= 32;
    }
    r.d[i + b.n] = static_cast<std::uint32_t>(c);
  }
  r.n = n;
  while (r.n > 0 && r.d[r.n - 1] == 0u) --r.n;
  r.neg = a.neg ^ b.neg;
}

// Limbs of one scaled input: < 2^(1023 + 1074 + 53) (+1 bit for a difference).
constexpr int kBigIn = 70;

// Big determinant helpers over scaled differences. Storage `w` must hold the
// documented number of limbs.
// det2 of big entries (a d - b c) into r; scratch t1, t2 of na+nd / nb+nc limbs.
SBDT_HD void big_det2(Big& r, const Big& a, const Big& b, const Big& c, const Big& d, Big& t1, Big& t2) {
  big_mul(t1, a, d);
  big_mul(t2, b, c);
  big_add(r, t1, t2, 1);
}

// out = det [[m0 m1 m2],[m3 m4 m5],[m6 m7 m8]] (cofactor expansion along row
// 0, as geometry.cpp:63-66), entries of at most E limbs. out holds 3E + 6
// limbs, scratch w 12E + 16 (disjoint).
SBDT_HD void big_det3(Big& out, const Big* m, std::uint32_t* w, int E) {
  Big t1{w, 0, 0}, t2{w + 2 * E + 2, 0, 0}, mi{w + 4 * E + 4, 0, 0};
  Big term{w + 6 * E + 8, 0, 0}, acc2{w + 9 * E + 12, 0, 0};
  out.n = 0, out.neg = 0;
  for (int j = 0; j < 3; ++j) {
    const int c1 = j == 0 ? 1 : 0, c2 = j == 2 ? 1 : 2;
    big_det2(mi, m[3 + c1], m[3 + c2], m[6 + c1], m[6 + c2], t1, t2);
    big_mul(term, m[j], mi);
    big_add(acc2, out, term, j == 1);
    for (int i = 0; i < acc2.n; ++i) out.d[i] = acc2.d[i];
    out.n = acc2.n, out.neg = acc2.neg;
  }
}
constexpr int big_det3_scratch(int E) { return 15 * E + 22; }  // out + w

// orient2 / orient3 on big integers: rows b-a, c-a(, d-a) (the reference's
// orient2_exact / orient3_exact, geometry.cpp:90-107).
SBDT_HDN int orient2_big(const double* a, const double* b, const double* c) {
  const double v[6] = {a[0], a[1], b[0], b[1], c[0], c[1]};
  const int emin = min_exponent(v, 6);
  std::uint32_t w[12 * kBigIn];
  Big x{w, 0, 0}, y{w + kBigIn, 0, 0}, e[4] = {{w + 2 * kBigIn, 0, 0}, {w + 3 * kBigIn, 0, 0},
                                              {w + 4 * kBigIn, 0, 0}, {w + 5 * kBigIn, 0, 0}};
  const double* rows[2] = {b, c};
  for (int i = 0; i < 2; ++i)
    for (int k = 0; k < 2; ++k) {
      big_scaled(x, rows[i][k], emin);
      big_scaled(y, a[k], emin);
      big_add(e[2 * i + k], x, y, 1);
    }
  Big t1{w + 6 * kBigIn, 0, 0}, t2{w + 8 * kBigIn, 0, 0}, r{w + 10 * kBigIn, 0, 0};
  big_det2(r, e[0], e[1], e[2], e[3], t1, t2);
  return big_sign(r);
}

SBDT_HDN int orient3_big(const double* a, const double* b, const double* c, const double* d) {
  const double v[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]};
  const int emin = min_exponent(v, 12);
  std::uint32_t w[11 * kBigIn + big_det3_scratch(kBigIn)];
  Big x{w, 0, 0}, y{w + kBigIn, 0, 0};
  Big m[9];
  for (int i = 0; i < 9; ++i) m[i] = Big{w + (2 + i) * kBigIn, 0, 0};
  const double* rows[3] = {b, c, d};
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) {
      big_scaled(x, rows[i][k], emin);
      big_scaled(y, a[k], emin);
      big_add(m[3 * i + k], x, y, 1);
    }
  Big out{w + 11 * kBigIn, 0, 0};
  big_det3(out, m, w + 11 * kBigIn + 3 * kBigIn + 6, kBigIn);
  return big_sign(out);
}

// Rows (p_i - q, |p_i - q|^2) of the lifted in_sphere matrix, scaled big
// integers (geometry.cpp:109-146 layout), into m (row stride D + 1, entries of
// E = 2 kBigIn + 2 limbs each) using w (2 kBigIn + E limbs) for temporaries.
template <int D>
SBDT_HD void big_lifted_rows(const double* const* p, const double* q, Big* m, std::uint32_t* w, int emin) {
  const int E = 2 * kBigIn + 2;
  Big x{w, 0, 0}, y{w + kBigIn, 0, 0}, sq{w + 2 * kBigIn, 0, 0}, acc{w + 2 * kBigIn + E, 0, 0};
  for (int i = 0; i <= D; ++i) {
    Big& lift = m[i * (D + 1) + D];
    lift.n = 0, lift.neg = 0;
    for (int k = 0; k < D; ++k) {
      big_scaled(x, p[i][k], emin);
      big_scaled(y, q[k], emin);
      Big& dk = m[i * (D + 1) + k];
      big_add(dk, x, y, 1);
      big_mul(sq, dk, dk);
      big_add(acc, lift, sq, 0);
      for (int t = 0; t < acc.n; ++t) lift.d[t] = acc.d[t];
      lift.n = acc.n, lift.neg = acc.neg;
    }
  }
}

// in_sphere2: sign det [[p_i - q, lift_i]] (3 x 3); in_sphere3: -sign of the
// 4 x 4 determinant (geometry.cpp:130-146), cofactor expansion along row 0 as
// the reference's det4. buf: scratch (doubles, reinterpreted as limbs).
SBDT_HDN int in_sphere2_big(const double* a, const double* b, const double* c, const double* q, double* buf) {
  const double v[8] = {a[0], a[1], b[0], b[1], c[0], c[1], q[0], q[1]};
  const int emin = min_exponent(v, 8);
  std::uint32_t* w = reinterpret_cast<std::uint32_t*>(buf);
  const int E = 2 * kBigIn + 2;
  Big m[9];
  for (int i = 0; i < 9; ++i) m[i] = Big{w + i * E, 0, 0};
  const double* p[3] = {a, b, c};
  big_lifted_rows<2>(p, q, m, w + 9 * E, emin);
  Big out{w + 9 * E, 0, 0};
  big_det3(out, m, w + 9 * E + 3 * E + 6, E);
  return big_sign(out);
}

SBDT_HDN int in_sphere3_big(const double* a, const double* b, const double* c, const double* d, const double* q,
                            double* buf) {
  const double v[15] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2], q[0], q[1], q[2]};
  const int emin = min_exponent(v, 15);
  std::uint32_t* w = reinterpret_cast<std::uint32_t*>(buf);
  const int E = 2 * kBigIn + 2;
  Big m[16];
  for (int i = 0; i < 16; ++i) m[i] = Big{w + i * E, 0, 0};
  const double* p[4] = {a, b, c, d};
  std::uint32_t* free0 = w + 16 * E;
  big_lifted_rows<3>(p, q, m, free0, emin);
  // det4 = sum_j (-1)^j m[0][j] det3(minor_j)
  const int E3 = 3 * E + 6;
  Big minor[9];
  Big d3{free0, 0, 0}, term{free0 + E3, 0, 0}, acc{free0 + E3 + E3 + E, 0, 0}, acc2{free0 + 3 * E3 + 2 * E + 4, 0, 0};
  std::uint32_t* wd = free0 + 4 * E3 + 3 * E + 8;
  acc.n = 0, acc.neg = 0;
  for (int j = 0; j < 4; ++j) {
    int idx = 0;
    for (int row = 1; row < 4; ++row)
      for (int col = 0; col < 4; ++col)
        if (col != j) minor[idx++] = m[4 * row + col];
    big_det3(d3, minor, wd, E);
    big_mul(term, m[j], d3);
    big_add(acc2, acc, term, j & 1);
    for (int t = 0; t < acc2.n; ++t) acc.d[t] = acc2.d[t];
    acc.n = acc2.n, acc.neg = acc2.neg;
  }
  return -big_sign(acc);
}

// Exact orient2 sign (geometry.cpp:150-170 contract): sign of
// (a-c)x (b-c)y - (a-c)y (b-c)x.
SBDT_HDN int orient2_expansion(const double* a, const double* b, const double* c) {
  const Diff2 acx = exact_diff(a[0], c[0]), acy = exact_diff(a[1], c[1]);
  const Diff2 bcx = exact_diff(b[0], c[0]), bcy = exact_diff(b[1], c[1]);
  double out[16];
  const int n = minor2(acx, acy, bcx, bcy, out);
  return expansion_sign(n, out);
}

// Exact orient2: expansion arithmetic on prescaled inputs, big integers
// when the inputs' exponent range is too wide for it.
SBDT_HDN int orient2_exact(const double* a, const double* b, const double* c) {
  const double v[6] = {a[0], a[1], b[0], b[1], c[0], c[1]};
  const int s = prescale_exponent(v, 6, 2);
  if (s == kNoScale) return orient2_big(a, b, c);
  if (s == 0) return orient2_expansion(a, b, c);
  double w[6];
  for (int i = 0; i < 6; ++i) w[i] = ldexp(v[i], s);
  return orient2_expansion(w, w + 2, w + 4);
}

// Filter stage only: the sign, or 2 when the binary64 evaluation cannot
// decide it (the caller escalates to orient2_exact).
SBDT_HD int orient2_filtered(const double* a, const double* b, const double* c) {
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
  return 2;
}

SBDT_HD int orient2(const double* a, const double* b, const double* c) {
  const int r = orient2_filtered(a, b, c);
  return r != 2 ? r : orient2_exact(a, b, c);
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
SBDT_HDN int orient3_expansion(const double* a, const double* b, const double* c, const double* d) {
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

SBDT_HDN int orient3_exact(const double* a, const double* b, const double* c, const double* d) {
  const double v[12] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2]};
  const int s = prescale_exponent(v, 12, 3);
  if (s == kNoScale) return orient3_big(a, b, c, d);
  if (s == 0) return orient3_expansion(a, b, c, d);
  double w[12];
  for (int i = 0; i < 12; ++i) w[i] = ldexp(v[i], s);
  return orient3_expansion(w, w + 3, w + 6, w + 9);
}

SBDT_HD int orient3_filtered(const double* a, const double* b, const double* c, const double* d) {
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
  return 2;  // undecided: orient3_exact
}

SBDT_HD int orient3(const double* a, const double* b, const double* c, const double* d) {
  const int r = orient3_filtered(a, b, c, d);
  return r != 2 ? r : orient3_exact(a, b, c, d);
}

// ---- in_sphere exact (host + escalation kernels) ---------------------------
// Scratch requirement for in_sphere2_exact: kInSphere2Scratch doubles.
constexpr int kInSphere2Scratch = 8192;
// in_sphere2 = sign det [[p_i - q, |p_i - q|^2]] for the three rows.
SBDT_HDN int in_sphere2_expansion(const double* a, const double* b, const double* c,
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

// Exact in_sphere2 (degree 4): expansion arithmetic on prescaled inputs, big
// integers for too wide an exponent range. buf: kInSphere2Scratch doubles.
SBDT_HDN int in_sphere2_exact_buf(const double* a, const double* b, const double* c, const double* q, double* buf) {
  const double v[8] = {a[0], a[1], b[0], b[1], c[0], c[1], q[0], q[1]};
  const int s = prescale_exponent(v, 8, 4);
  if (s == kNoScale) return in_sphere2_big(a, b, c, q, buf);
  if (s == 0) return in_sphere2_expansion(a, b, c, q, buf);
  double w[8];
  for (int i = 0; i < 8; ++i) w[i] = ldexp(v[i], s);
  return in_sphere2_expansion(w, w + 2, w + 4, w + 6, buf);
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
SBDT_HDN int in_sphere3_expansion(const double* a, const double* b, const double* c,
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

// Exact in_sphere3 (degree 5), as in_sphere2_exact_buf. buf: kInSphere3Scratch doubles.
SBDT_HDN int in_sphere3_exact_buf(const double* a, const double* b, const double* c, const double* d,
                                 const double* q, double* buf) {
  const double v[15] = {a[0], a[1], a[2], b[0], b[1], b[2], c[0], c[1], c[2], d[0], d[1], d[2], q[0], q[1], q[2]};
  const int s = prescale_exponent(v, 15, 5);
  if (s == kNoScale) return in_sphere3_big(a, b, c, d, q, buf);
  if (s == 0) return in_sphere3_expansion(a, b, c, d, q, buf);
  double w[15];
  for (int i = 0; i < 15; ++i) w[i] = ldexp(v[i], s);
  return in_sphere3_expansion(w, w + 3, w + 6, w + 9, w + 12, buf);
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
