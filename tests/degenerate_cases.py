"""Seeded near-degenerate predicate cases (test helper).

The same scheme as the reference's near-degenerate generator
(/root/reference/proj/tests/support/degenerate_cases.hpp:16-124, restated,
not copied): points placed on a line / plane / circle / sphere in exact
arithmetic, whose binary64 rounding leaves determinants within a few ulps of
zero, plus exactly degenerate integer configurations (collinear / coplanar
lattice points, Pythagorean cocircular and integer cospherical sets) and
large-offset copies (cancellation in the differences). Layout per case:
orient (dim+1) points, in_sphere (dim+1) simplex points then q.
"""
from __future__ import annotations

import numpy as np


def _unit(rng, n, dim):
    v = rng.standard_normal((n, dim))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def orient_cases(dim: int, count: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.empty((count, dim + 1, dim))
    q = count // 4
    # 1) last point on the affine hull of the others (rounded): near zero
    n1 = count - 3 * q
    base = rng.random((n1, dim, dim))
    w = rng.random((n1, dim - 1))
    last = base[:, 0] + sum(w[:, i:i + 1] * (base[:, i + 1] - base[:, 0]) for i in range(dim - 1))
    out[:n1, :dim] = base
    out[:n1, dim] = last
    # 2) the same with a large offset (cancellation) and a random scale
    off = rng.uniform(-1e6, 1e6, (q, 1, dim))
    scale = 2.0 ** rng.integers(-20, 20, (q, 1, 1))
    b2 = rng.random((q, dim, dim)) * scale
    w2 = rng.random((q, dim - 1))
    l2 = b2[:, 0] + sum(w2[:, i:i + 1] * (b2[:, i + 1] - b2[:, 0]) for i in range(dim - 1))
    out[n1:n1 + q, :dim] = b2 + off
    out[n1:n1 + q, dim] = l2 + off[:, 0]
    # 3) exactly degenerate integer configurations: lattice points on a line / plane
    a = rng.integers(-1000, 1000, (q, 1, dim)).astype(np.float64)
    dirs = rng.integers(-20, 20, (q, dim - 1, dim)).astype(np.float64)
    coef = rng.integers(-5, 5, (q, dim + 1, dim - 1)).astype(np.float64)
    out[n1 + q:n1 + 2 * q] = a + np.einsum("qkj,qjd->qkd", coef, dirs)
    # 4) tiny perturbations of exact degeneracies (one ulp-scale nudge)
    c4 = out[n1 + q:n1 + 2 * q].copy()
    c4[:, dim] = np.nextafter(c4[:, dim], c4[:, dim] + rng.choice([-1.0, 1.0], (q, dim)))
    out[n1 + 2 * q:] = c4
    return out


def _integer_sphere_points(dim: int, r2: int) -> np.ndarray:
    m = int(np.floor(np.sqrt(r2))) + 1
    rng_ = np.arange(-m, m + 1)
    grids = np.stack(np.meshgrid(*([rng_] * dim), indexing="ij"), -1).reshape(-1, dim)
    return grids[(grids ** 2).sum(1) == r2].astype(np.float64)


def orient_positive(cases: np.ndarray, orient_fn) -> np.ndarray:
    """The reference's in_sphere2/3 require a positively oriented simplex
    (geometry.cpp:192 asserts it): swap p0, p1 where orient < 0 and drop the
    flat simplices (orient = 0). orient_fn(simplices) -> exact signs."""
    dim = cases.shape[2]
    o = orient_fn(np.ascontiguousarray(cases[:, :dim + 1]))
    out = cases[o != 0].copy()
    neg = o[o != 0] < 0
    out[neg, 0], out[neg, 1] = cases[o != 0][neg, 1], cases[o != 0][neg, 0]
    return out


def in_sphere_cases(dim: int, count: int, seed: int) -> np.ndarray:
    """Raw cases (the simplex orientation is arbitrary; see orient_positive)."""
    rng = np.random.default_rng(seed)
    out = np.empty((count, dim + 2, dim))
    q = count // 4
    n1 = count - 3 * q
    # 1) dim+2 points on a random sphere (rounded): near cospherical
    c = rng.random((n1, 1, dim))
    r = rng.uniform(1e-3, 1.0, (n1, 1, 1))
    out[:n1] = c + r * _unit(rng, n1 * (dim + 2), dim).reshape(n1, dim + 2, dim)
    # 2) the same far from the origin
    off = rng.uniform(-1e5, 1e5, (q, 1, dim))
    r2 = rng.uniform(1e-4, 1.0, (q, 1, 1))
    out[n1:n1 + q] = off + r2 * _unit(rng, q * (dim + 2), dim).reshape(q, dim + 2, dim)
    # 3) exactly cospherical integer points (x^2 + y^2 (+ z^2) = R), translated
    R = 25 if dim == 2 else 27
    S = _integer_sphere_points(dim, R)
    idx = np.stack([rng.choice(len(S), dim + 2, replace=False) for _ in range(q)])
    shift = rng.integers(-100, 100, (q, 1, dim)).astype(np.float64)
    out[n1 + q:n1 + 2 * q] = S[idx] + shift
    # 4) one coordinate of q nudged by an ulp (sign decided far below the filter)
    c4 = out[n1 + q:n1 + 2 * q].copy()
    c4[:, dim + 1, 0] = np.nextafter(c4[:, dim + 1, 0], c4[:, dim + 1, 0] + rng.choice([-1.0, 1.0], q))
    out[n1 + 2 * q:] = c4
    return out


def wide_range_cases(dim: int, npts: int, count: int, seed: int) -> np.ndarray:
    """Coordinates with random signs, mantissas and exponents over the whole
    binary64 range (subnormals and zeros included): the filters' products
    under/overflow and expansion arithmetic alone is not exact; the exact
    stage must fall back to scaled big integers (the reference's ExactScaler)."""
    rng = np.random.default_rng(seed)
    m = rng.random((count, npts, dim)) * 2 - 1
    e = rng.integers(-1074, 1000, (count, npts, dim))
    v = np.ldexp(m, e)
    v[rng.random((count, npts, dim)) < 0.1] = 0.0
    return v
