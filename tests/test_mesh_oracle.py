"""Pins of the oracle's triangle-mesh signed distance (NEXT-4, reading R-24),
CPU only.

What fixes the expected values:
  * a 12-triangle box mesh has exactly the box SDF (closed form, SG_BOX);
  * an icosphere is inscribed in its sphere: |f_mesh - f_sphere| <= h, the
    largest face-plane depth below the sphere (computed from the vertices),
    and the signs agree wherever |f_sphere| > h;
  * re-ordering triangles (and rotating each triangle's vertex order) leaves
    f unchanged to rounding;
  * whole pipeline: a box-mesh grid has the box-primitive grid's tables.
"""
import numpy as np

import workloads as W

BOX_C, BOX_B = (0.5, 0.48, 0.52), (0.2, 0.15, 0.25)


def _box_sdf(x, c=BOX_C, b=BOX_B):
    q = np.abs(x - np.asarray(c)) - np.asarray(b)
    out = np.linalg.norm(np.maximum(q, 0.0), axis=1)
    return out + np.minimum(q.max(1), 0.0)


def _near_box_points(rng, n):
    # random points plus points near faces, edges and corners
    x = rng.uniform(0, 1, (n, 3))
    c, b = np.asarray(BOX_C), np.asarray(BOX_B)
    s = rng.choice([-1.0, 1.0], (n, 3))
    y = c + s * b * rng.choice([1.0, 1.0 + 1e-3, 1.0 - 1e-3, 0.5], (n, 3))
    return np.concatenate([x, y + rng.normal(0, 0.01, (n, 3))])


def test_box_mesh_is_box_sdf(oracle_lib):
    w = W.mesh_workload("boxm", W.box_mesh(BOX_C, BOX_B), 16)
    o = oracle_lib.Oracle(w)
    x = _near_box_points(np.random.default_rng(3), 20000)
    f, ex = o.sdf(x), _box_sdf(x)
    np.testing.assert_allclose(f, ex, rtol=0, atol=1e-12)
    sure = np.abs(ex) > 1e-12
    np.testing.assert_array_equal(f[sure] < 0, ex[sure] < 0)


def test_icosphere_within_sagitta(oracle_lib):
    c, r = np.array([0.5, 0.5, 0.5]), 0.3
    m = W.icosphere(3, tuple(c), r, rot=0.4)
    V = np.array(m.verts).reshape(-1, 3)
    T = np.array(m.tris).reshape(-1, 3)
    a, b, cc = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    n = np.cross(b - a, cc - a)
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    h = r - np.min(np.abs(((a - c) * n).sum(1)))  # deepest face plane below the sphere
    assert 0 < h < 0.01
    o = oracle_lib.Oracle(W.mesh_workload("ico", m, 16))
    x = np.random.default_rng(4).uniform(0.05, 0.95, (20000, 3))
    f, fs = o.sdf(x), np.linalg.norm(x - c, axis=1) - r
    assert np.max(np.abs(f - fs)) <= h + 1e-12
    sure = np.abs(fs) > h
    np.testing.assert_array_equal(f[sure] < 0, fs[sure] < 0)


def test_triangle_order_invariance(oracle_lib):
    m = W.icosphere(2, rot=0.7)
    T = np.array(m.tris).reshape(-1, 3)
    rng = np.random.default_rng(5)
    T2 = np.roll(T[rng.permutation(len(T))], 1, axis=1)
    m2 = W.Mesh(m.verts, tuple(int(i) for i in T2.ravel()))
    x = rng.uniform(0, 1, (5000, 3))
    f1 = oracle_lib.Oracle(W.mesh_workload("a", m, 8)).sdf(x)
    f2 = oracle_lib.Oracle(W.mesh_workload("b", m2, 8)).sdf(x)
    np.testing.assert_allclose(f1, f2, rtol=0, atol=1e-14)
    sure = np.abs(f1) > 1e-12
    np.testing.assert_array_equal(f1[sure] < 0, f2[sure] < 0)


def test_box_mesh_grid_tables_equal_box_primitive(oracle_lib):
    n = 20
    wp = W.Workload("boxp", (n, n, n), 1.0 / n, dtype="f64",
                    prims=(W.Prim(W.BOX, BOX_C + BOX_B),))
    op = oracle_lib.Oracle(wp)
    tp = op.build_tables()
    assert tp.near_ties == 0
    om = oracle_lib.Oracle(W.mesh_workload("boxm", W.box_mesh(BOX_C, BOX_B), n))
    tm = om.build_tables()
    np.testing.assert_array_equal(tm.bg, tp.bg)
    np.testing.assert_array_equal(tm.nb, tp.nb)
    np.testing.assert_allclose(om.phi_dense(), op.phi_dense(), rtol=0, atol=1e-12)


def test_stl_round_trip(tmp_path, oracle_lib):
    """STL (the paper's input) in and out: a box mesh written as binary
    STL (fp32 coordinates) and as ASCII reads back to the same closed mesh,
    whose SDF is still the box closed form."""
    c, b = (0.5, 0.5, 0.5), (0.25, 0.125, 0.375)  # fp32-exact corners
    m = W.box_mesh(c, b)
    p = tmp_path / "box.stl"
    W.write_stl(str(p), m)
    r = W.read_stl(str(p))
    assert r.n_tris == 12 and r.n_verts == 8
    V = np.array(r.verts).reshape(-1, 3)
    T = np.array(r.tris).reshape(-1, 3)
    tri = V[T]
    nrm = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
    assert np.all((nrm * (tri.mean(1) - np.asarray(c))).sum(1) > 0)  # outward
    asc = tmp_path / "box_ascii.stl"
    with open(asc, "w") as fh:
        fh.write("solid box\n")
        for t in tri:
            fh.write(" facet normal 0 0 0\n  outer loop\n")
            for v in t:
                fh.write(f"   vertex {float(v[0])!r} {float(v[1])!r} {float(v[2])!r}\n")
            fh.write("  endloop\n endfacet\n")
        fh.write("endsolid box\n")
    r2 = W.read_stl(str(asc))
    assert r2 == r
    o = oracle_lib.Oracle(W.mesh_workload("stl", r, 8))
    x = np.random.default_rng(6).uniform(0, 1, (5000, 3))
    np.testing.assert_allclose(o.sdf(x), _box_sdf(x, c, b), rtol=0, atol=1e-12)
