"""The box-window oracle (oracle/sg_oracle.c or_grid.win_lo/win_n) is the
whole-domain oracle restricted to a box (CPU only).

C3 / C5 cannot be checked on the whole dense grid (69 GB / 550 GB per fp64
field), so their GPU parity tests use the oracle on a box of background cells
("a z-window of W bg planes plus a margin of ceil(n_iter/4) + 1
planes each side ... the window interior is exact").  This pins that claim:
on grids small enough for the whole-domain oracle, every O6-O10 value of the
window oracle at depth > (sweeps + stencil radius) from the box faces is
bit-identical to the whole-domain value.
"""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O


def _sub(a, lo, hi, lead=0):
    """dense box [4 lo, 4 hi) of a whole-domain dense array (z, y, x last)."""
    sl = tuple(slice(4 * lo[k], 4 * hi[k]) for k in (2, 1, 0))
    return a[(slice(None),) * lead + sl]


def _inner(a, d, lead=0):
    sl = tuple(slice(d, -d) for _ in range(3))
    return a[(slice(None),) * lead + sl]


@pytest.mark.parametrize("w,lo,hi,sweeps", [
    (W.config("C1"), (2, 3, 1), (14, 13, 15), 6),
    (W.random_scene(3, 24, dtype="f64"), (5, 0, 4), (20, 24, 16), 8),
    (W.random_scene(6, 17, dtype="f64"), (0, 2, 3), (17, 15, 12), 5),
])
def test_window_equals_whole_domain_interior(w, lo, hi, sweeps):
    full = O.Oracle(w)
    t = full.build_tables()
    win = O.Oracle(w, (lo, hi))
    win.tables = t
    phi = full.phi_dense()
    pw = win.phi_dense()
    # O6 is pointwise: the whole box equals
    assert np.array_equal(pw, _sub(phi, lo, hi))
    p_full = full.reinit(phi, sweeps)
    p_win = win.reinit(pw, sweeps)
    d = sweeps + 1
    assert np.array_equal(_inner(p_win, d), _inner(_sub(p_full, lo, hi), d))
    g_full, n_full = full.gradient(p_full)
    g_win, n_win = win.gradient(p_win)
    K_full, G_full = full.kernel_integrals(p_full, w.h_ratio)
    K_win, G_win = win.kernel_integrals(p_win, w.h_ratio)
    e = d + 3  # + kernel radius (2 at h = 1.3 dx) and the gradient's 1
    assert np.array_equal(_inner(g_win, e, 1), _inner(_sub(g_full, lo, hi, 1), e, 1))
    assert np.array_equal(_inner(n_win, e, 1), _inner(_sub(n_full, lo, hi, 1), e, 1))
    assert np.array_equal(_inner(K_win, e), _inner(_sub(K_full, lo, hi), e))
    assert np.array_equal(_inner(G_win, e, 1), _inner(_sub(G_full, lo, hi, 1), e, 1))
    # probe of points deep inside the box
    rng = np.random.default_rng(5)
    dx = w.cell / 4
    a = np.array([w.lower[k] + (4 * lo[k] + e + 1) * dx for k in range(3)])
    b = np.array([w.lower[k] + (4 * hi[k] - e - 1) * dx for k in range(3)])
    pos = rng.uniform(a, b, size=(3000, 3))
    r_full = full.probe(p_full, g_full, pos)
    r_win = win.probe(p_win, g_win, pos)
    assert np.array_equal(r_full[0], r_win[0]) and np.array_equal(r_full[1], r_win[1])


def test_box_to_packages_layout():
    """The layout helper gives the canonical package order of
    or_gather_packages for every active cell of the box."""
    w = W.config("C1")
    o = O.Oracle(w)
    t = o.build_tables()
    phi = o.reinit(o.phi_dense(), 2)
    lo, hi = (1, 2, 3), (15, 11, 16)
    pk = O.box_to_packages(_sub(phi, lo, hi))
    ref = o.to_packages(phi, 0.0, 0.0)
    bgb = t.bg.reshape(w.n[2], w.n[1], w.n[0])[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
    act = bgb >= 2
    assert act.sum() > 100
    assert np.array_equal(pk[act], ref[bgb[act]])
    g, _ = o.gradient(phi)
    pk3 = O.box_to_packages(_sub(g, lo, hi, 1))
    assert pk3.shape[0] == 3
    ref3 = np.stack([o.to_packages(g[c], 0.0, 0.0) for c in range(3)], 0)
    assert np.array_equal(pk3[:, act], ref3[:, bgb[act]])


def test_window_rejects_whole_domain_only_ops():
    w = W.config("C1")
    win = O.Oracle(w, ((0, 0, 0), (8, 8, 8)))
    with pytest.raises(AssertionError):
        win.to_packages(np.zeros((32, 32, 32)), 0.0, 0.0)
