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
