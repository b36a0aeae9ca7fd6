"""The C++ drop-in layer (include/sbdt/sample_partition.hpp, border.hpp,
dc_engine.hpp) on the reference's own types: paper_1902_07554_b200/dropin_example
(built by `make` against /root/reference/proj/include, header-only use of
PointSet, Triangulation<D>, Simplex<D>) runs assign_points + build_grid_index
+ find_border + merge exactly as delaunay_dc would, and must agree bit for bit
with the CPU oracle."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_1902_07554_b200 import host

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1902_07554_b200",
                   "dropin_example")


def write_instance(path, inst, part, tb=None):
    """The dropin_example input file (layout in tests/cpp/dropin_example.cpp)."""
    k = part.k
    with open(path, "wb") as f:
        f.write(np.array([inst.dim], np.uint32).tobytes() + np.array([inst.n], np.uint64).tobytes()
                + np.array([len(inst.sample_ids), k], np.uint32).tobytes() + np.array([part.S], np.uint64).tobytes())
        for a in (inst.points, inst.sample_ids, inst.sample_labels, part.offsets, part.verts, part.nbrs, part.parity):
            f.write(np.ascontiguousarray(a).tobytes())
        if tb is not None:
            f.write(np.array([tb.verts.shape[1]], np.uint64).tobytes())
            for a in (tb.verts, tb.nbrs, tb.parity):
                f.write(np.ascontiguousarray(a).tobytes())


@pytest.mark.parametrize("cfg,n,k", [(1, 40_000, 8), (2, 60_000, 8)])
def test_cpp_dropin_matches_oracle(cfg, n, k, tmp_path):
    if not os.path.exists(EXE):
        pytest.skip("dropin_example not built (needs the reference headers at build time)")
    inst = host.make_instance(cfg, n=n, k=k)
    labels = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels)
    part = host.attach_partials(inst, labels)
    dim, S = inst.dim, part.S
    src = tmp_path / "instance.bin"
    with open(src, "wb") as f:
        f.write(np.array([dim], np.uint32).tobytes() + np.array([inst.n], np.uint64).tobytes()
                + np.array([len(inst.sample_ids), k], np.uint32).tobytes() + np.array([S], np.uint64).tobytes())
        for a in (inst.points, inst.sample_ids, inst.sample_labels, part.offsets, part.verts, part.nbrs, part.parity):
            f.write(np.ascontiguousarray(a).tobytes())
        # T_B: the DT of the (BFS) border vertices, for sbdt::merge
        ref = oracle.find_border(inst.points, labels, part, "grid")
        tb = host.triangulate(inst.points, ref["vertices_border"], 7)
        f.write(np.array([tb.verts.shape[1]], np.uint64).tobytes())
        for a in (tb.verts, tb.nbrs, tb.parity):
            f.write(np.ascontiguousarray(a).tobytes())
    dst = tmp_path / "result.bin"
    r = subprocess.run([EXE, str(src), str(dst)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    raw = dst.read_bytes()
    o = 0

    def take(dt, cnt):
        nonlocal o
        a = np.frombuffer(raw, dt, cnt, o)
        o += a.nbytes
        return a

    got_labels = take(np.uint32, inst.n)
    pos, bor = take(np.uint8, S), take(np.uint8, S)
    vpos = take(np.uint32, int(take(np.uint64, 1)[0]))
    vbor = take(np.uint32, int(take(np.uint64, 1)[0]))
    rows = int(take(np.uint64, 1)[0])
    mv = take(np.uint32, (dim + 1) * rows).reshape(dim + 1, rows)
    mn = take(np.uint32, (dim + 1) * rows).reshape(dim + 1, rows)
    mp = take(np.int8, rows)
    assert np.array_equal(got_labels, labels)
    assert np.array_equal(pos, ref["positive"])
    assert np.array_equal(bor, ref["border"])
    assert np.array_equal(vpos, ref["vertices_positive"])
    assert np.array_equal(vbor, ref["vertices_border"])
    ov, on, op, _ = oracle.merge(part, ref["border"], tb, labels)
    assert np.array_equal(mv, ov) and np.array_equal(mn, on) and np.array_equal(mp, op)


@pytest.mark.parametrize("cfg,n,k,level", [(1, 40_000, 8, 3), (2, 60_000, 8, 5)])
def test_cpp_dropin_recursion_level(cfg, n, k, level, tmp_path):
    """A recursion level of delaunay_dc: only the first
    `level` partitions and their points take part, their GridIndex keeps the
    full set's bbox and n (build_grid_index post): the grid is
    the top level's and the other points occupy no cell (SBDT_UNINDEXED)."""
    if not os.path.exists(EXE):
        pytest.skip("dropin_example not built (needs the reference headers at build time)")
    inst = host.make_instance(cfg, n=n, k=k)
    labels = oracle.assign_brute(inst.points, inst.sample_ids, inst.sample_labels)
    part = host.attach_partials(inst, labels)
    src, dst = tmp_path / "instance.bin", tmp_path / "result.bin"
    write_instance(src, inst, part)
    r = subprocess.run([EXE, str(src), str(dst), "--level", str(level)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    SL = int(part.offsets[level])
    raw = dst.read_bytes()
    o = inst.n * 4
    pos = np.frombuffer(raw, np.uint8, SL, o)
    bor = np.frombuffer(raw, np.uint8, SL, o + SL)
    o += 2 * SL
    nv = int(np.frombuffer(raw, np.uint64, 1, o)[0])
    vpos = np.frombuffer(raw, np.uint32, nv, o + 8)
    o += 8 + 4 * nv
    nb = int(np.frombuffer(raw, np.uint64, 1, o)[0])
    vbor = np.frombuffer(raw, np.uint32, nb, o + 8)
    lvl_labels = np.where(labels < level, labels, np.uint32(0xFFFFFFFF)).astype(np.uint32)
    lvl = host.Partials(part.offsets[:level + 1].copy(), np.ascontiguousarray(part.verts[:, :SL]),
                        np.ascontiguousarray(part.nbrs[:, :SL]), part.parity[:SL].copy())
    lo, hi = inst.points.min(axis=0), inst.points.max(axis=0)
    ref = oracle.find_border(inst.points, lvl_labels, lvl, "grid", grid_bbox=(lo, hi), grid_n_total=inst.n)
    assert np.array_equal(pos, ref["positive"]) and np.array_equal(bor, ref["border"])
    assert np.array_equal(vpos, ref["vertices_positive"]) and np.array_equal(vbor, ref["vertices_border"])
    # a grid from the level's own points (bbox, count) gives other flags: the override matters
    sub = inst.points[labels < level]
    own = oracle.find_border(inst.points, lvl_labels, lvl, "grid", grid_bbox=(sub.min(axis=0), sub.max(axis=0)),
                             grid_n_total=len(sub))
    assert not np.array_equal(own["positive"], ref["positive"])
