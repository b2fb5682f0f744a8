"""Pins of the oracle's small-feature cleaning (NEXT-3, reading
R-23 = SPEC S:476-484 stand-in, threshold 0.4 of the kernel sum S), CPU only.

What fixes the expected values (SPEC S:482-484 examples, closed geometry):
  * a planar slab has K = S/2 on its surface (pinned in test_oracle_pins):
    nothing is raised, the call is a fixed point;
  * a wall thinner than h is removed: every point of it ends outside;
  * a wall 4h thick and the slab keep their interior signs;
  * idempotence: a second call raises nothing.
"""
import numpy as np

import workloads as W

N = 24


def _pos(w):
    mx, my, mz = (4 * n for n in w.n)
    dx = w.cell / 4
    z, y, x = np.meshgrid(*[w.lower[k] + (np.arange(m) + 0.5) * dx
                            for k, m in ((2, mz), (1, my), (0, mx))], indexing="ij")
    return x, y, z


def test_planar_slab_is_fixed_point(oracle_lib):
    w = W.Workload("slab", (N, N, N), 1.0 / N, dtype="f64",
                   prims=(W.Prim(W.BOX, (0.5, 0.5, 0.3, 1.0, 1.0, 0.1)),))
    o = oracle_lib.Oracle(w)
    phi0 = o.phi_dense()
    phi, rounds, mods = o.clean(phi0)
    assert rounds == 0 and mods[0] == 0
    np.testing.assert_array_equal(phi, phi0)


def test_thin_wall_removed_thick_wall_and_slab_kept(oracle_lib):
    w = W.fins(N)
    o = oracle_lib.Oracle(w)
    phi0 = o.phi_dense()
    x, y, z = _pos(w)
    h = w.h_ratio * w.dx
    # away from the x faces of the domain, where the walls leave the domain
    # and the far-field neighbours of R-6 distort the reinitialisation
    mid = np.abs(x - 0.5) < 0.3
    thin = mid & (np.abs(y - 0.3) < 0.25 * h) & (z > 0.42) & (z < 0.58)
    thick = mid & (np.abs(y - 0.7) < 1.5 * w.dx) & (z > 0.45) & (z < 0.55)
    slab = mid & (z > 0.25) & (z < 0.35)
    air = mid & (np.abs(y - 0.5) < 0.05) & (z > 0.45)
    assert (phi0[thin] < 0).sum() > 50, "the thin wall must be resolved before cleaning"
    assert (phi0[thick] < 0).all() and (phi0[slab] < 0).all()
    phi, rounds, mods = o.clean(phi0)
    assert rounds >= 1 and mods[0] > 0
    assert (phi[thin] > 0).all(), "thin wall not removed"
    assert (phi[thick] < 0).all(), "thick wall damaged"
    assert (phi[slab] < 0).all() and (phi[air] > 0).all()


def test_idempotent_once_converged(oracle_lib):
    """Slab + thin wall: the first call converges (a round raises nothing), so
    a second call is a fixed point.  (Convex edges sharper than the kernel
    support, like the top of the 4h wall, erode by about one data point per
    round instead, so that scene is bounded by max_rounds.)"""
    w = W.fins(N)
    w = w.with_(name="FINthin", prims=w.prims[:2])
    o = oracle_lib.Oracle(w)
    phi, rounds, mods = o.clean(o.phi_dense())
    assert 1 <= rounds < 5 and mods[rounds] == 0
    phi2, rounds2, mods2 = o.clean(phi)
    assert rounds2 == 0 and mods2[0] == 0
    np.testing.assert_array_equal(phi2, phi)
