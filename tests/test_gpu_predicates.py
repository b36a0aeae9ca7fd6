"""Device predicates pinned case by case (SPEC.md acceptance criterion 2:
10^6 near-degenerate orient / in_sphere cases against an exact reference).

The device evaluates exactly what find_border runs internally (predicates.hpp:
binary64 filter with the reference's error constants, geometry.cpp:23-27,
then expansion arithmetic) through the diagnostic C-ABI entry point
sbdt_gpu_predicates. The reference for every case is the reference's own
compiled geometry.cpp (orient2/3 geometry.cpp:150-189, in_sphere2/3
:191-277, exact fallback :32-146) from oracle/_ref, else the restatement
(pinned to it by tests/test_oracle.py)."""
import numpy as np
import pytest

import oracle
from degenerate_cases import in_sphere_cases, orient_cases, orient_positive, wide_range_cases

GOLD = "tests/golden/primitives.npz"


def _orient_ref(simplices):
    return oracle.predicates_batch("orient", simplices)[0]


def _insphere_cases(dim, count, seed):
    return orient_positive(in_sphere_cases(dim, count, seed), _orient_ref)


def test_oracle_matches_reference_near_degenerate():
    """CPU: the restatement (oracle/prims.hpp) equals the reference's compiled
    predicates on the near-degenerate sets (skipped without oracle/_ref)."""
    if oracle.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    for dim in (2, 3):
        P = orient_cases(dim, 20_000, 100 + dim)
        assert np.array_equal(oracle.predicates_batch("orient", P)[0],
                              oracle.predicates_batch("orient", P, use_ref=False)[0])
        Q = _insphere_cases(dim, 20_000, 200 + dim)
        assert np.array_equal(oracle.predicates_batch("in_sphere", Q)[0],
                              oracle.predicates_batch("in_sphere", Q, use_ref=False)[0])


def test_host_predicates_match_reference():
    """CPU: the predicates the kernels compile (csrc/common/predicates.hpp,
    host build) equal the reference's compiled geometry.cpp sign for sign on
    the near-degenerate sets and on whole-binary64-range inputs (subnormals,
    zeros, 1e+300 next to 1e-300: the filters under/overflow and the exact
    stage must use scaled big integers, as the reference's ExactScaler)."""
    from paper_1902_07554_b200 import host
    for dim in (2, 3):
        for P in (orient_cases(dim, 20_000, 500 + dim), wide_range_cases(dim, dim + 1, 20_000, 600 + dim)):
            assert np.array_equal(host.predicates("orient", P), oracle.predicates_batch("orient", P)[0])
        for Q in (_insphere_cases(dim, 20_000, 700 + dim),
                  orient_positive(wide_range_cases(dim, dim + 2, 20_000, 800 + dim), _orient_ref)):
            assert np.array_equal(host.predicates("in_sphere", Q), oracle.predicates_batch("in_sphere", Q)[0])


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
def test_device_predicates_golden(dim, ctx):
    """The golden vectors generated from the reference's compiled code
    (tests/golden/make_golden.py: random + near-degenerate)."""
    z = np.load(GOLD)
    P = z[f"orient{dim}_pts"].reshape(-1, dim + 1, dim)
    got, _ = ctx.predicates("orient", P)
    assert np.array_equal(got, z[f"orient{dim}_out"])
    Q = np.concatenate([z[f"insphere{dim}_pts"].reshape(-1, dim + 1, dim),
                        z[f"insphere{dim}_q"].reshape(-1, 1, dim)], axis=1)
    got, _ = ctx.predicates("in_sphere", Q)
    assert np.array_equal(got, z[f"insphere{dim}_out"])


@pytest.mark.gpu
def test_device_predicates_million_near_degenerate(ctx):
    """~10^6 near-degenerate cases (4 sets of 250k: orient and in_sphere, 2-D
    and 3-D), device vs the reference, sign for sign; the exact stage must
    have run (escalations > 0 in every set)."""
    total, report = 0, {}
    for dim in (2, 3):
        P = orient_cases(dim, 250_000, 300 + dim)
        ref, which = oracle.predicates_batch("orient", P)
        got, esc = ctx.predicates("orient", P)
        assert np.array_equal(got, ref), f"orient{dim}: {np.count_nonzero(got != ref)} signs differ ({which})"
        assert esc > 0
        report[f"orient{dim}"] = (len(P), esc, int(np.count_nonzero(ref == 0)))
        Q = _insphere_cases(dim, 250_000, 400 + dim)
        ref, which = oracle.predicates_batch("in_sphere", Q)
        got, esc = ctx.predicates("in_sphere", Q)
        assert np.array_equal(got, ref), f"in_sphere{dim}: {np.count_nonzero(got != ref)} signs differ ({which})"
        assert esc > 0
        report[f"in_sphere{dim}"] = (len(Q), esc, int(np.count_nonzero(ref == 0)))
        total += len(P) + len(Q)
    assert total >= 990_000
    print("predicate cases (count, escalated, exact zeros):", report)


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
def test_device_predicates_wide_range(dim, ctx):
    """Whole-binary64-range coordinates (subnormals, zeros, huge and tiny
    together): the device's exact stage must switch to scaled big integers
    and still equal the reference's signs."""
    P = wide_range_cases(dim, dim + 1, 50_000, 900 + dim)
    got, esc = ctx.predicates("orient", P)
    assert np.array_equal(got, oracle.predicates_batch("orient", P)[0]) and esc > 0
    Q = orient_positive(wide_range_cases(dim, dim + 2, 50_000, 950 + dim), _orient_ref)
    got, esc = ctx.predicates("in_sphere", Q)
    assert np.array_equal(got, oracle.predicates_batch("in_sphere", Q)[0]) and esc > 0


def _flat_hull_instance():
    """2-D, two parts split by the diagonal; part 0 holds (0,0), (1,1) and a
    point one ulp below (0.5, 0.5): the nearly flat triangle on its hull is
    in its DT (its huge circumcircle holds no part-0 point), its binary32
    sphere cannot be bounded and its binary64 orientation filter cannot
    decide (exact orientation nonzero)."""
    rng = np.random.default_rng(4)
    a = rng.random((4000, 2))
    a = a[a[:, 1] < a[:, 0] - 0.01]
    b = rng.random((4000, 2))
    b = b[b[:, 1] > b[:, 0] + 0.01]
    trip = np.array([[0.0, 0.0], [0.5, np.nextafter(0.5, 0.0)], [1.0, 1.0]])
    pts = np.ascontiguousarray(np.concatenate([trip, a, b]))
    lab = np.concatenate([np.zeros(3 + len(a)), np.ones(len(b))]).astype(np.uint32)
    return pts, lab


def _cocircular_instance():
    """2-D: 9 points exactly on one circle (integer solutions of x^2 + y^2 =
    4225, scaled by 2^-6 and shifted: every difference and product exact);
    3 in part 0, 6 in part 1, all other points outside the circle. The part-0
    triangle on the circle has foreign points exactly ON its circumcircle:
    in_sphere = 0, which the binary64 filter can never decide."""
    m = 66
    g = np.arange(-m, m + 1)
    X, Y = np.meshgrid(g, g)
    on = X ** 2 + Y ** 2 == 4225
    c = np.stack([X[on], Y[on]], 1).astype(np.float64)
    c = c[np.argsort(np.arctan2(c[:, 1], c[:, 0]))] / 64.0 + 2.0
    rng = np.random.default_rng(4)
    r = rng.random((6000, 2)) * 4
    r = r[np.hypot(r[:, 0] - 2, r[:, 1] - 2) > 1.2]
    A = np.concatenate([c[[0, 12, 24]], r[r[:, 0] < 2]])
    B = np.concatenate([c[[3, 7, 16, 20, 28, 33]], r[r[:, 0] >= 2]])
    pts = np.ascontiguousarray(np.concatenate([A, B]))
    lab = np.concatenate([np.zeros(len(A)), np.ones(len(B))]).astype(np.uint32)
    return pts, lab


@pytest.mark.gpu
@pytest.mark.parametrize("case,policy", [("flat_hull", "grid"), ("flat_hull", "exact"), ("cocircular", "exact"),
                                         ("cocircular", "grid")])
def test_find_border_escalates(case, policy, ctx):
    """find_border instances that force the escalation paths INSIDE the
    pipeline (census counters): a binary32 sphere that cannot be bounded ->
    exact orientation row whose binary64 filter fails (orient escalation);
    foreign points exactly on a circumcircle -> in_sphere escalation (exact
    policy). Outputs stay bit-identical to the oracle."""
    from paper_1902_07554_b200 import gpu, host
    pts, lab = _flat_hull_instance() if case == "flat_hull" else _cocircular_instance()
    P = host.build_partials(pts, lab, 2, 7)
    ctx.set_timing(False, census=True)
    try:
        g = gpu.find_border(pts, lab, P, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True, ctx=ctx)
        st = ctx.border_stats()
    finally:
        ctx.set_timing(False)
    o = oracle.find_border(pts, lab, P, policy)
    assert np.array_equal(g.positive, o["positive"]) and np.array_equal(g.border, o["border"])
    assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
    assert np.array_equal(g.border_vertex_ids, o["vertices_border"])
    print(case, policy, {k: st.get(k) for k in ("orient_check_rows", "orient_escalations", "in_sphere_escalations")})
    if case == "flat_hull" and policy == "grid":
        assert st["orient_check_rows"] > 0 and st["orient_escalations"] > 0
    if case == "cocircular" and policy == "exact":
        assert st["in_sphere_escalations"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cocircular", "jittered_lattice"])
def test_escalation_queue_overflow_degrades(case, ctx, monkeypatch):
    """A full escalation queue no longer fails the call: the rows whose
    undecided pairs did not fit are decided again, whole, after the
    escalation (k_border_redo). The queue is shrunk to 4 entries through the
    test hook SBDT_TEST_ESC_CAP; results must still equal the oracle."""
    from paper_1902_07554_b200 import gpu, host
    if case == "cocircular":
        pts, lab = _cocircular_instance()
        P = host.build_partials(pts, lab, 2, 7)
    else:
        side = 12
        g = np.stack(np.meshgrid(*[np.arange(side, dtype=np.float64)] * 3, indexing="ij"), -1).reshape(-1, 3)
        pts = np.ascontiguousarray(g + np.random.default_rng(3).uniform(-1e-9, 1e-9, g.shape))
        lab = np.minimum((pts[:, 0] * 3 // side).astype(np.uint32), 2)
        P = host.build_partials(pts, lab, 3, 7)
    monkeypatch.setenv("SBDT_TEST_ESC_CAP", "4")
    g = gpu.find_border(pts, lab, P, gpu.IntersectionPolicy("exact", 1.0), hull_bfs=True, ctx=ctx)
    monkeypatch.delenv("SBDT_TEST_ESC_CAP")
    o = oracle.find_border(pts, lab, P, "exact")
    assert np.array_equal(g.positive, o["positive"]) and np.array_equal(g.border, o["border"])
    assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
