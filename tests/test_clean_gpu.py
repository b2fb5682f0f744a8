"""GPU parity of the small-feature cleaning (NEXT-3, reading R-23).

fp64: the raised-point counts per round are exact against the oracle (the
decision K < threshold S is taken in fp64 on both sides) and phi agrees to
rounding after every round's reinitialisation.  fp32: the decisions are the
kernel's; the geometric outcome (thin wall removed, thick wall and slab kept,
idempotence once converged) is checked on the GPU result itself.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sgm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_11473_b200 import build
    build.build()
    from paper_2512_11473_b200 import sg
    return sg


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


def dense(g, w):
    """Scatter the active packages of the GPU phi into a dense (Mz, My, Mx)
    array (NaN at inactive points)."""
    nx, ny, nz = w.n
    phi = g.view("phi").cpu().numpy().astype(np.float64)
    cell = g.view("meta_cell").cpu().numpy().view(np.uint32)[2:].astype(np.int64)
    out = np.full((4 * nz, 4 * ny, 4 * nx), np.nan)
    cx, cy, cz = cell % nx, (cell // nx) % ny, cell // (nx * ny)
    k, j, i = np.meshgrid(np.arange(4), np.arange(4), np.arange(4), indexing="ij")
    zz = (4 * cz)[:, None] + k.ravel()[None, :]
    yy = (4 * cy)[:, None] + j.ravel()[None, :]
    xx = (4 * cx)[:, None] + i.ravel()[None, :]
    out[zz, yy, xx] = phi[2:]
    return out


def masks(w):
    mx, my, mz = (4 * n for n in w.n)
    dx = w.dx
    z, y, x = np.meshgrid(*[(np.arange(m) + 0.5) * dx for m in (mz, my, mx)], indexing="ij")
    h = w.h_ratio * dx
    mid = np.abs(x - 0.5) < 0.3
    return {"thin": mid & (np.abs(y - 0.3) < 0.25 * h) & (z > 0.42) & (z < 0.58),
            "thick": mid & (np.abs(y - 0.7) < 1.5 * dx) & (z > 0.45) & (z < 0.55),
            "slab": mid & (z > 0.25) & (z < 0.35)}


def test_clean_fp64_matches_oracle(sgm, O):
    w = W.fins(24, dtype="f64")
    o = O.Oracle(w)
    g = sgm.Grid(w)
    phi_o, r_o, m_o = o.clean(o.phi_dense(), threshold=0.4)
    r, m = g.clean(threshold=0.4)
    assert (r, m) == (r_o, m_o)
    got = g.view("phi").cpu().numpy()
    exp = o.to_packages(phi_o, -o.far, o.far)
    err = np.max(np.abs(got - exp))
    assert err <= 1e-9 * w.dx, f"max err {err / w.dx:.3e} dx"


def test_clean_fp32_geometry(sgm):
    w = W.fins(24, dtype="f32")
    g = sgm.Grid(w)
    d0 = dense(g, w)
    mk = masks(w)
    assert np.sum(d0[mk["thin"]] < 0) > 50
    r, m = g.clean(threshold=0.4)
    assert r >= 1 and m[0] > 0
    d = dense(g, w)
    # inactive points (NaN) lie in the far field of their cell's sign
    assert not np.any(d[mk["thin"]] <= 0), "thin wall not removed"
    assert not np.any(d[mk["thick"]] >= 0), "thick wall damaged"
    assert not np.any(d[mk["slab"]] >= 0), "slab damaged"


def test_clean_fp32_idempotent_once_converged(sgm):
    w = W.fins(24, dtype="f32")
    w = w.with_(name="FINthin", prims=w.prims[:2])
    g = sgm.Grid(w)
    r, m = g.clean(threshold=0.4)
    assert 1 <= r < 5 and m[r] == 0
    before = g.view("phi").cpu().numpy().copy()
    r2, m2 = g.clean(threshold=0.4)
    assert r2 == 0 and m2[0] == 0
    assert np.array_equal(g.view("phi").cpu().numpy(), before)


def test_clean_planar_slab_fixed_point(sgm):
    w = W.Workload("slab", (24, 24, 24), 1.0 / 24, dtype="f32",
                   prims=(W.Prim(W.BOX, (0.5, 0.5, 0.3, 1.0, 1.0, 0.1)),))
    g = sgm.Grid(w)
    before = g.view("phi").cpu().numpy().copy()
    assert g.clean(threshold=0.4) == (0, [0, 0, 0, 0, 0])
    assert np.array_equal(g.view("phi").cpu().numpy(), before)


def test_clean_argument_errors(sgm):
    w = W.config("C1")
    g = sgm.Grid(w, slab=(0, 8, 2))
    with pytest.raises(sgm.SgError):
        g.clean()
    g2 = sgm.Grid(w)
    with pytest.raises(sgm.SgError):
        g2.clean(threshold=1.5)
    with pytest.raises(sgm.SgError):
        g2.clean(h_ratio=3.0)
