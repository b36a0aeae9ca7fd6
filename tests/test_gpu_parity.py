"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on
identical seeded inputs, for scaled-down versions of all five BASELINE
configs. Bit-exact for labels, parts, positive/border flags and border-vertex
sets; circumcentres / radii within 1e-12 relative (north_star tolerance)."""
import numpy as np
import pytest

import oracle
from paper_1902_07554_b200 import gpu, host

pytestmark = pytest.mark.gpu

SMALL = {1: dict(n=60_000, k=16, frac=0.01), 2: dict(n=80_000, k=8, frac=0.01), 3: dict(n=80_000, k=8, frac=0.01),
         4: dict(n=120_000, k=16, frac=0.005), 5: dict(n=150_000, k=16, frac=0.002)}

_cache = {}


def instance(cfg):
    if cfg not in _cache:
        inst = host.make_instance(cfg, **SMALL[cfg])
        labels = oracle.assign_kdtree(inst.points, inst.sample_ids, inst.sample_labels)
        host.attach_partials(inst, labels)
        _cache[cfg] = inst
    return _cache[cfg]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_assign_points_bit_exact(cfg, ctx):
    inst = instance(cfg)
    part = gpu.assign_points(inst.points, inst.sample_ids, inst.sample_labels, inst.config["k"], ctx=ctx)
    ref = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels)
    assert np.array_equal(part.labels, ref)
    # Partitioning.parts: ascending ids per part, consistent with labels
    for p in range(inst.config["k"]):
        ids = part.part(p)
        assert np.array_equal(ids, np.nonzero(ref == p)[0].astype(np.uint32))
    np.testing.assert_array_equal(part.bbox[:inst.dim], inst.points.min(axis=0))
    np.testing.assert_array_equal(part.bbox[inst.dim:], inst.points.max(axis=0))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("policy", ["grid", "bbox", "exact"])
def test_find_border_bit_exact(cfg, policy, ctx):
    inst = instance(cfg)
    g = gpu.find_border(inst.points, inst.labels, inst.partials, gpu.IntersectionPolicy(policy, 1.0), hull_bfs=True,
                        spheres=True, ctx=ctx)
    o = oracle.find_border(inst.points, inst.labels, inst.partials, policy, spheres=True)
    assert np.array_equal(g.positive, o["positive"])
    assert np.array_equal(g.border, o["border"])
    assert np.array_equal(g.positive_vertex_ids, o["vertices_positive"])
    assert np.array_equal(g.border_vertex_ids, o["vertices_border"])
    fin = inst.partials.verts[-1] != 0xFFFFFFFF
    a, b = g.spheres[fin], o["spheres"][fin]
    # expected bit-identical; the contract tolerance is 1e-12 relative
    scale = np.maximum(np.abs(b), 1e-300)
    assert np.all(np.abs(a - b) <= 1e-12 * scale)
    assert np.array_equal(a, b)
