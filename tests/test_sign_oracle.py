"""Pins of the oracle's sign-consistency correction (NEXT-3, P:528-535,
reading R-22) and of the SG_LEAK post-operation, CPU only.

What fixes the expected values:
  * closed-form containment of spheres / tori: after the correction every
    data point and every cell has the sign of the exact (non-leaky) SDF;
  * scipy's taxicab distance transform: a synchronous flood from the trusted
    set needs exactly max-distance sweeps (6-connected BFS in a box = L1);
  * invariants: |phi| unchanged, trusted signs unchanged, a watertight input
    is a fixed point.
"""
import numpy as np
import pytest
from scipy.ndimage import distance_transform_cdt

import workloads as W

SPHERE = W.Workload("S24", (24, 24, 24), 1.0 / 24, dtype="f64",
                    prims=(W.Prim(W.SPHERE, (0.5, 0.5, 0.5, 0.3)),))
TORUS = W.Workload("T24", (24, 24, 24), 1.0 / 24, dtype="f64",
                   prims=(W.Prim(W.TORUS_Y, (0.5, 0.5, 0.5, 0.3, 0.1)),))


def _true_sdf(w, x):
    """Closed-form SDF of the (single) non-leak primitive of w."""
    p = w.prims[0]
    c = np.asarray(p.p[:3])
    if p.kind == W.SPHERE:
        return np.linalg.norm(x - c, axis=-1) - p.p[3]
    if p.kind == W.TORUS_Y:
        e = x - c
        t = np.hypot(e[..., 0], e[..., 2]) - p.p[3]
        return np.hypot(t, e[..., 1]) - p.p[4]
    raise ValueError(p.kind)


def _points(w):
    mx, my, mz = (4 * n for n in w.n)
    dx = w.cell / 4
    iz, iy, ix = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    return np.stack([w.lower[0] + (ix + 0.5) * dx, w.lower[1] + (iy + 0.5) * dx,
                     w.lower[2] + (iz + 0.5) * dx], -1)


def _centres(w):
    nx, ny, nz = w.n
    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return np.stack([w.lower[0] + (cx + 0.5) * w.cell, w.lower[1] + (cy + 0.5) * w.cell,
                     w.lower[2] + (cz + 0.5) * w.cell], -1)


def _active_points(w, bg):
    nx, ny, nz = w.n
    act = (bg.reshape(nz, ny, nx) >= 2)
    return act.repeat(4, 0).repeat(4, 1).repeat(4, 2)


def test_leak_postop_closed_form(oracle_lib):
    """f_leaky = -f inside a ball where |f| >= margin, else f (sg.h SG_LEAK)."""
    w = W.leaky(SPHERE)
    o, o0 = oracle_lib.Oracle(w), oracle_lib.Oracle(SPHERE)
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (20000, 3))
    f = _true_sdf(SPHERE, x)
    inside = np.zeros(len(x), bool)
    for b in W.LEAK_BALLS:
        inside |= ((x - np.asarray(b[:3])) ** 2).sum(1) < b[3] ** 2
    flip = inside & (np.abs(f) >= w.cell)
    got = o.sdf(x)
    np.testing.assert_allclose(got, np.where(flip, -f, f), atol=1e-12)
    np.testing.assert_array_equal(np.abs(got), np.abs(o0.sdf(x)))
    assert flip.sum() > 500


@pytest.mark.parametrize("base", [SPHERE, TORUS], ids=["sphere", "torus"])
def test_sign_correct_recovers_closed_form(oracle_lib, base):
    w = W.leaky(base)
    o = oracle_lib.Oracle(w)
    t = o.build_tables()
    phi0 = o.phi_dense()
    truth = _true_sdf(base, _points(w))
    act = _active_points(w, t.bg)
    wrong_before = act & ((phi0 < 0) != (truth < 0)) & (np.abs(truth) > 1e-12)
    assert wrong_before.sum() > 100, "the leak must corrupt the input"
    bg, nb, cell_neg, phi, sweeps = o.sign_correct(phi0)
    # magnitudes untouched, signs = exact containment at every active point
    np.testing.assert_array_equal(np.abs(phi), np.abs(phi0))
    ok = act & (np.abs(truth) > 1e-12)
    np.testing.assert_array_equal((phi < 0)[ok], (truth < 0)[ok])
    # trusted points (|phi| < dx) keep their sign
    tr = act & (np.abs(phi0) < o.dx)
    np.testing.assert_array_equal(np.signbit(phi[tr]), np.signbit(phi0[tr]))
    # every cell: sign of the exact SDF at its centre
    fc = _true_sdf(base, _centres(w)).ravel()
    np.testing.assert_array_equal(cell_neg.astype(bool), fc < 0)
    # inactive table entries and singular neighbour entries: exact signs, i.e.
    # the watertight build's tables
    o0 = oracle_lib.Oracle(base)
    t0 = o0.build_tables()
    np.testing.assert_array_equal(bg, t0.bg)
    np.testing.assert_array_equal(nb, t0.nb)
    # inactive points carry the far constant of the exact sign
    np.testing.assert_array_equal(phi[~act], o0.phi_dense()[~act])
    assert sweeps[0] > 0 and sweeps[1] > 0


@pytest.mark.parametrize("base", [SPHERE, TORUS], ids=["sphere", "torus"])
def test_sweep_counts_equal_taxicab_distance(oracle_lib, base):
    """A synchronous flood from the trusted set signs a site in the sweep equal
    to its 6-connected BFS distance, which in a box is the L1 distance."""
    w = W.leaky(base)
    o = oracle_lib.Oracle(w)
    t = o.build_tables()
    phi0 = o.phi_dense()
    _, _, _, _, sweeps = o.sign_correct(phi0)
    nx, ny, nz = w.n
    core = (t.cat.reshape(nz, ny, nx) == 3)
    assert sweeps[0] == int(distance_transform_cdt(~core, metric="taxicab").max())
    act = _active_points(w, t.bg)
    src = ~act | (np.abs(phi0) < o.dx)  # trusted points, inactive points
    pad = np.pad(src, 1, constant_values=True)  # out-of-domain points are signed (R-6)
    d = distance_transform_cdt(~pad, metric="taxicab")[1:-1, 1:-1, 1:-1]
    assert sweeps[1] == int(d[act & ~src].max())


def test_sweep_cap(oracle_lib):
    w = W.leaky(SPHERE)
    o = oracle_lib.Oracle(w)
    o.build_tables()
    phi0 = o.phi_dense()
    *_, full = o.sign_correct(phi0)
    *_, capped = o.sign_correct(phi0, max_sweeps=2)
    assert capped == (min(2, full[0]), min(2, full[1]))


@pytest.mark.parametrize("base", [SPHERE, TORUS], ids=["sphere", "torus"])
def test_watertight_is_fixed_point(oracle_lib, base):
    o = oracle_lib.Oracle(base)
    t = o.build_tables()
    phi0 = o.phi_dense()
    bg, nb, cell_neg, phi, _ = o.sign_correct(phi0)
    np.testing.assert_array_equal(phi, phi0)
    np.testing.assert_array_equal(bg, t.bg)
    np.testing.assert_array_equal(nb, t.nb)
