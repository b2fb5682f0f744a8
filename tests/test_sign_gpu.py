"""GPU parity of the sign-consistency correction (NEXT-3, R-22)
and of the SG_LEAK post-operation in the build.

Integer / sign work: bit-exact against the oracle (tables, cell signs, phi
bits, sweep counts).  The trust decision |phi| < tau is taken in the grid
dtype on both sides: for fp32 grids the oracle receives phi and tau rounded
to float32.  At full size (C2, C3) the corrected leaky grid must equal the
watertight grid bit for bit (closed-form truth of the analytic SDF).
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


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def cell_bits(g, w):
    a = u32(g.view("cell_neg"))
    nzt, ny, nw = a.shape
    bits = (a[..., None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(nzt, ny, nw * 32)[:, :, : w.n[0]].astype(bool).ravel()


def phi_bits_equal(got, exp):
    if got.dtype == np.float32:  # far constants etc. as the grid stores them
        exp = exp.astype(np.float32).astype(np.float64)
    got = np.asarray(got, dtype=np.float64)
    assert got.shape == exp.shape
    bad = np.flatnonzero((got != exp) | (np.signbit(got) != np.signbit(exp)))
    assert bad.size == 0, f"{bad.size} values differ, first {bad[:5]}"


SPHERE24 = W.Workload("S24", (24, 24, 24), 1.0 / 24, dtype="f64",
                      prims=(W.Prim(W.SPHERE, (0.5, 0.5, 0.5, 0.3)),))
TORUS24 = W.Workload("T24", (24, 24, 24), 1.0 / 24, dtype="f32",
                     prims=(W.Prim(W.TORUS_Y, (0.5, 0.5, 0.5, 0.3, 0.1)),))
PRISM40 = W.config("C2").with_(name="C2s", n=(40, 40, 40), cell=1.0 / 40)

CASES = {
    "C1L-f64": W.leaky(W.config("C1")),
    "C1L-f32": W.leaky(W.config("C1").with_(dtype="f32")),
    "S24L-f64": W.leaky(SPHERE24),
    "T24L-f32": W.leaky(TORUS24),
    "C2sL-f32": W.leaky(PRISM40),
}


def _pair(sgm, O, w, max_sweeps=0):
    o = O.Oracle(w)
    t = o.build_tables()
    g = sgm.Grid(w)
    # the leaky build itself: tables bit-exact (SG_LEAK in K1/K3/K4)
    assert np.array_equal(u32(g.view("bg")), t.bg)
    assert np.array_equal(u32(g.view("nb")), t.nb)
    phi0 = o.phi_dense()
    if w.dtype == "f32":
        phi_in = phi0.astype(np.float32).astype(np.float64)
        tau = float(np.float32(w.dx))
    else:
        phi_in, tau = phi0, w.dx
    far = o.far
    phi_bits_equal(g.view("phi").cpu().numpy(), o.to_packages(phi_in, -far, far))
    sw = g.sign_correct(tau, max_sweeps)
    bg, nb, cn, phi, osw = o.sign_correct(phi_in, tau, max_sweeps)
    assert sw == osw
    assert np.array_equal(u32(g.view("bg")), bg)
    assert np.array_equal(u32(g.view("nb")), nb)
    # the face table the sweeps read follows the corrected neighbour table
    face = u32(g.view("face"))
    assert np.array_equal(face[:, :6], nb[:, [12, 14, 10, 16, 4, 22]])
    assert np.array_equal(cell_bits(g, w), cn.astype(bool))
    phi_bits_equal(g.view("phi").cpu().numpy(), o.to_packages(phi, -far, far))
    return g, sw


@pytest.mark.parametrize("case", list(CASES))
def test_sign_correct_bit_exact(sgm, O, case):
    g, sw = _pair(sgm, O, CASES[case])
    assert sw[0] > 0 and sw[1] > 0


@pytest.mark.parametrize("cap", [1, 3])
def test_sign_correct_sweep_cap(sgm, O, cap):
    _pair(sgm, O, CASES["S24L-f64"], max_sweeps=cap)


def _grid_state(g):
    return (u32(g.view("bg")).copy(), u32(g.view("nb")).copy(), g.view("phi").cpu().numpy(),
            u32(g.view("cell_neg")).copy(), u32(g.view("face")).copy())


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_full_size_leaky_equals_watertight(sgm, name):
    """C2 / C3 at full size: the corrected leaky grid is the watertight grid,
    bit for bit (every leak-flipped sign restored, nothing else touched)."""
    w = W.config(name)
    ref = _grid_state(sgm.Grid(w))
    g = sgm.Grid(W.leaky(w))
    before = g.view("phi").cpu().numpy()
    assert np.count_nonzero(np.signbit(before) != np.signbit(ref[2])) > 1000
    sw = g.sign_correct()
    got = _grid_state(g)
    assert np.array_equal(got[0], ref[0])
    assert np.array_equal(got[1], ref[1])
    phi_bits_equal(got[2], ref[2].astype(np.float64))
    assert np.array_equal(got[3], ref[3])
    assert np.array_equal(got[4], ref[4])  # face table
    assert sw[0] > 0 and sw[1] > 0
    del g


def test_watertight_fixed_point_c2(sgm):
    w = W.config("C2")
    g = sgm.Grid(w)
    ref = _grid_state(g)
    g.sign_correct()
    got = _grid_state(g)
    for a, b in zip(got, ref):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_sign_correct_rejects_slab_grid(sgm):
    w = W.config("C1")
    g = sgm.Grid(w, slab=(0, 8, 2))
    with pytest.raises(sgm.SgError):
        g.sign_correct()
    with pytest.raises(sgm.SgError):
        g.sign_correct(tau=-1.0)


@pytest.mark.parametrize("base,levels", [("C2", 2), ("C3", 1)])
def test_multires_leaky_chain_equals_watertight(sgm, base, levels):
    """P:528-535 across layers: correct the coarsest leaky layer over all
    cells, refine, correct each refined layer over its evaluated cells only;
    the finest layer equals the watertight direct build bit for bit."""
    w0 = W.config(base)
    f = 2 ** levels
    wc = w0.with_(n=tuple(k // f for k in w0.n), cell=w0.cell * f)
    leaky = W.leaky(wc)
    g = sgm.Grid(leaky)
    sw = g.sign_correct()
    for _ in range(levels):
        g = g.refined()
        sw_fine = g.sign_correct()
        assert sw_fine[0] <= 2 * sw[0]
    ref = _grid_state(sgm.Grid(w0))
    got = _grid_state(g)
    assert np.array_equal(got[0], ref[0])
    assert np.array_equal(got[1], ref[1])
    phi_bits_equal(got[2], ref[2].astype(np.float64))
    assert np.array_equal(got[3], ref[3])
