"""Generates the golden fixtures under tests/golden/ from the REFERENCE's own
compiled code (oracle/_ref/libsbdt_ref.so: /root/reference/proj/src/geometry.cpp,
triangulation.cpp, F4-patched sequential_dt.cpp compiled by path).

  python tests/golden/make_golden.py      (needs oracle/_ref, i.e. this container)

primitives.npz : orient / in_sphere / circumsphere / box_sphere_overlap /
                 halfspace_box_overlap on random and near-degenerate inputs
                 (points on a line/circle/sphere perturbed by a few ulps, the
                 scheme of proj/tests/support/degenerate_cases.hpp).
dt_canon.npz   : canonical forms of the reference's triangulate_seq on small sets.
path_cfg*.npz  : small seeded instances of the five configs with the
                 reference-primitive instantiation of the path (assign labels,
                 positive / BFS-border flags and border-vertex sets for the
                 bbox, grid and exact policies).
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1902_07554_b200 import host  # noqa: E402

P = oracle._p


def near_degenerate(rng, dim, kind, count):
    out_pts, out_q = [], []
    for _ in range(count):
        if kind == "orient":
            a, b = rng.random(dim), rng.random(dim)
            if dim == 2:
                t = 4 * rng.random() - 2
                p = a + t * (b - a)
                pts = [a, b, p]
            else:
                v = rng.random(3)
                s, t = 4 * rng.random() - 2, 4 * rng.random() - 2
                p = a + s * (b - a) + t * (v - a)
                pts = [a, b, v, p]
            pts = [np.array(x, dtype=np.float64) for x in pts]
            for _k in range(2):
                pts[-1] = np.nextafter(pts[-1], rng.choice([-np.inf, np.inf], size=dim))
            out_pts.append(np.concatenate(pts))
        else:  # in_sphere: D+2 points on a common circle/sphere, +-1 ulp
            c = rng.random(dim)
            r = 0.1 + rng.random()
            pts = []
            for _j in range(dim + 2):
                d = rng.normal(size=dim)
                d /= np.linalg.norm(d)
                p = c + r * d
                p = np.nextafter(p, rng.choice([-np.inf, np.inf], size=dim))
                pts.append(p)
            out_pts.append(np.concatenate(pts[:dim + 1]))
            out_q.append(pts[dim + 1])
    return np.array(out_pts), (np.array(out_q) if out_q else None)


def primitives(R):
    rng = np.random.default_rng(1902)
    res = {}
    for dim in (2, 3):
        # orient: random + near-degenerate
        rnd = rng.random((1000, (dim + 1) * dim))
        deg, _ = near_degenerate(rng, dim, "orient", 2000)
        pts = np.ascontiguousarray(np.vstack([rnd, deg]))
        res[f"orient{dim}_pts"] = pts
        res[f"orient{dim}_out"] = np.array([R.ref_orient(dim, P(np.ascontiguousarray(p), C.c_double)) for p in pts],
                                           np.int8)
        # in_sphere on positively oriented simplices
        deg, q = near_degenerate(rng, dim, "insphere", 1500)
        rq = rng.random((1000, dim)) * 1.2 - 0.1
        rp = rng.random((1000, (dim + 1) * dim))
        allp, allq = np.vstack([rp, deg]), np.vstack([rq, q])
        keep_p, keep_q, outs = [], [], []
        for p, qq in zip(allp, allq):
            p = np.ascontiguousarray(p)
            o = R.ref_orient(dim, P(p, C.c_double))
            if o == 0:
                continue
            if o < 0:
                p = p.copy()
                p[:dim], p[dim:2 * dim] = p[dim:2 * dim].copy(), p[:dim].copy()
            qq = np.ascontiguousarray(qq)
            keep_p.append(p)
            keep_q.append(qq)
            outs.append(R.ref_in_sphere(dim, P(p, C.c_double), P(qq, C.c_double)))
        res[f"insphere{dim}_pts"], res[f"insphere{dim}_q"] = np.array(keep_p), np.array(keep_q)
        res[f"insphere{dim}_out"] = np.array(outs, np.int8)
        # circumsphere (+ degenerate throw -> status 1)
        cs = np.ascontiguousarray(rng.random((800, (dim + 1) * dim)))
        a = rng.random(dim)
        b = rng.random(dim)
        line = np.concatenate([a, b] + [a + t * (b - a) for t in (2.0,)] + ([a + 0.5 * (b - a)] if dim == 3 else []))
        cs = np.vstack([cs, line])
        outc, st = np.zeros((len(cs), dim + 1)), np.zeros(len(cs), np.int8)
        for i, p in enumerate(cs):
            o = np.zeros(dim + 1)
            st[i] = R.ref_circumsphere(dim, P(np.ascontiguousarray(p), C.c_double), P(o, C.c_double))
            outc[i] = o
        res[f"circum{dim}_pts"], res[f"circum{dim}_out"], res[f"circum{dim}_status"] = cs, outc, st
        # box_sphere_overlap
        lo = rng.random((1500, dim)) * 4 - 2
        hi = lo + rng.random((1500, dim)) * 2
        cc = rng.random((1500, dim)) * 4 - 2
        r2 = rng.random(1500) * 2
        res[f"boxsphere{dim}"] = np.hstack([lo, hi, cc, r2[:, None]])
        res[f"boxsphere{dim}_out"] = np.array(
            [R.ref_box_sphere(dim, P(np.ascontiguousarray(l), C.c_double), P(np.ascontiguousarray(h), C.c_double),
                              P(np.ascontiguousarray(c), C.c_double), float(r)) for l, h, c, r in zip(lo, hi, cc, r2)],
            np.int8)
        # halfspace_box_overlap
        fac = rng.random((1000, dim * dim))
        inn = rng.random((1000, dim))
        lo = rng.random((1000, dim)) * 2 - 0.5
        hi = lo + rng.random((1000, dim)) * 0.5
        outs = []
        for f, i_, l, h in zip(fac, inn, lo, hi):
            pts = np.concatenate([f, i_])
            if R.ref_orient(dim, P(np.ascontiguousarray(pts), C.c_double)) == 0:
                outs.append(-1)
                continue
            outs.append(R.ref_halfspace_box(dim, P(np.ascontiguousarray(f), C.c_double),
                                            P(np.ascontiguousarray(i_), C.c_double),
                                            P(np.ascontiguousarray(l), C.c_double),
                                            P(np.ascontiguousarray(h), C.c_double)))
        res[f"halfspace{dim}"] = np.hstack([fac, inn, lo, hi])
        res[f"halfspace{dim}_out"] = np.array(outs, np.int8)
    res["inflate_probe"] = np.array([R.ref_inflate(x) for x in (1.0, 0.75, 2.0, 1e-20, 3.3)])
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **res)


def ref_tri(R, pts, ids, seed):
    pts = np.ascontiguousarray(pts)
    ids = np.ascontiguousarray(ids, np.uint32)
    h = R.ref_triangulate(pts.shape[1], P(pts, C.c_double), len(pts), P(ids, C.c_uint32), len(ids), seed)
    S = R.ref_tri_count(h)
    v = np.empty((pts.shape[1] + 1, S), np.uint32)
    R.ref_tri_export(h, P(v, C.c_uint32), None, None)
    R.ref_tri_free(h)
    fin = v[:, v[-1] != 0xFFFFFFFF]
    return np.unique(np.sort(fin.T, axis=1), axis=0)


def dt_canon(R):
    res = {}
    for dim in (2, 3):
        for i, (dist, n) in enumerate((("uniform", 300), ("uniform", 2000), ("normal", 1500))):
            pts = host.generate(dist, dim, n, 40 + i)
            res[f"d{dim}_{i}_pts"] = pts
            res[f"d{dim}_{i}_canon"] = ref_tri(R, pts, np.arange(n, dtype=np.uint32), 7)
    pts = host.generate("bubbles", 3, 3000, 44)
    res["bubbles_pts"], res["bubbles_canon"] = pts, ref_tri(R, pts, np.arange(3000, dtype=np.uint32), 7)
    pts = host.generate("lines", 2, 3000, 45, params=(10, 1e-4))
    res["lines_pts"], res["lines_canon"] = pts, ref_tri(R, pts, np.arange(3000, dtype=np.uint32), 7)
    np.savez_compressed(os.path.join(HERE, "dt_canon.npz"), **res)


SMALL = {1: dict(n=4000, k=4, frac=0.02), 2: dict(n=5000, k=4, frac=0.02), 3: dict(n=5000, k=4, frac=0.02),
         4: dict(n=6000, k=4, frac=0.02), 5: dict(n=6000, k=4, frac=0.02)}


def path(R):
    for cfg, kw in SMALL.items():
        inst = host.make_instance(cfg, **kw)
        pts = np.ascontiguousarray(inst.points)
        lab = np.empty(inst.n, np.uint32)
        R.ref_assign_brute(inst.dim, P(pts, C.c_double), inst.n, P(inst.sample_ids, C.c_uint32),
                           len(inst.sample_ids), P(inst.sample_labels, C.c_uint32), P(lab, C.c_uint32))
        part = host.attach_partials(inst, lab)
        out = dict(points=pts, sample_ids=inst.sample_ids, sample_labels=inst.sample_labels, labels=lab,
                   offsets=part.offsets, verts=part.verts, nbrs=part.nbrs, parity=part.parity)
        for pol, code in (("bbox", 0), ("grid", 1), ("exact", 2)):
            pos, bor = np.empty(part.S, np.uint8), np.empty(part.S, np.uint8)
            vp, vb = np.empty(inst.n, np.uint32), np.empty(inst.n, np.uint32)
            np_, nb_ = C.c_uint64(), C.c_uint64()
            R.ref_find_border(inst.dim, P(pts, C.c_double), inst.n, P(lab, C.c_uint32), part.k,
                              P(part.offsets, C.c_uint64), P(part.verts, C.c_uint32), P(part.nbrs, C.c_uint32),
                              P(part.parity, C.c_int8), code, 1.0, P(pos, C.c_uint8), P(bor, C.c_uint8),
                              P(vp, C.c_uint32), C.byref(np_), P(vb, C.c_uint32), C.byref(nb_))
            out[f"{pol}_positive"] = np.packbits(pos)
            out[f"{pol}_border"] = np.packbits(bor)
            out[f"{pol}_vpos"] = vp[:np_.value].copy()
            out[f"{pol}_vbfs"] = vb[:nb_.value].copy()
        np.savez_compressed(os.path.join(HERE, f"path_cfg{cfg}.npz"), **out)


if __name__ == "__main__":
    R = oracle.ref_lib()
    if R is None:
        raise SystemExit("oracle/_ref/libsbdt_ref.so missing (build it with `make -C oracle` where /root/reference exists)")
    primitives(R)
    dt_canon(R)
    path(R)
    print("golden fixtures written to", HERE)
