"""GPU parity at the bench sizes C3 (2048^3 effective) and C5 (4096^3) on box
windows (SURVEY 8(d) "How the oracle is timed beside it": the dense grid does
not fit -- 69 GB / 550 GB per fp64 field -- so the oracle runs on a box of
background cells plus a margin; tests/test_oracle_window.py pins that the box
interior is the whole-domain oracle bit for bit).

Per window (inner box I of background cells, oracle box B = I + 7 cells per
side; 7 cells = 28 points >= 20 sweeps + 3 stencil points + 1):
  * the 20-sweep drift of the GPU's own reinit against 20 oracle sweeps from
    the same init (flag at 20 x 1e-5 dx);
  * one sweep from the oracle's 10-sweep state, uploaded to the GPU;
  * gradient, normal, K and G from the oracle's 20-sweep state uploaded to the
    GPU (fused K6+K7 kernel, the bench's call);
  * the probe (phi and grad phi) at random positions in I on that state.
Oracle inputs never come from the GPU: the oracle's state (rounded to fp32)
is uploaded into the packages of I + 1 cell, and every comparison is inside
I, at least one cell (4 points) from any value the GPU did not receive.
Tolerances: DESIGN.md section 4.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

MARGIN = 7  # cells


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


_TABLES = {}


def tables(O, name):
    if name not in _TABLES:
        _TABLES.clear()  # one full-size table set at a time (C5: ~7 GB host)
        _TABLES[name] = O.Oracle(W.config(name)).build_tables()
    return _TABLES[name]


# inner boxes (background cells): surfaces, an edge / corner kink, thin walls
WINDOWS = {
    "C3-torus": ("C3", (448, 248, 252), (464, 264, 260)),   # torus tube, outer side
    "C3-corner": ("C3", (300, 300, 456), (316, 316, 464)),  # box corner (0.6, 0.6, 0.9)
    "C5-shell": ("C5", (504, 504, 824), (520, 520, 834)),   # big shell, outer wall at top
    "C5-small": ("C5", (190, 136, 136), (206, 152, 144)),   # small shell walls at (0.14,)*3
}


class Win:
    def __init__(self, O, name):
        cfg, lo, hi = WINDOWS[name]
        self.w = w = W.config(cfg)
        self.t = tables(O, cfg)
        self.lo, self.hi = lo, hi
        self.blo = tuple(max(0, lo[k] - MARGIN) for k in range(3))
        self.bhi = tuple(min(w.n[k], hi[k] + MARGIN) for k in range(3))
        self.o = O.Oracle(w, (self.blo, self.bhi))
        self.o.tables = self.t
        self.O = O
        self.dx = w.cell / 4
        bg3 = self.t.bg.reshape(w.n[2], w.n[1], w.n[0])
        self.bgb = bg3[self.blo[2]:self.bhi[2], self.blo[1]:self.bhi[1], self.blo[0]:self.bhi[0]]

    def region(self, grow):
        """(mask over the box cells, package ids) of I grown by `grow` cells."""
        m = np.zeros(self.bgb.shape, bool)
        sl = tuple(slice(self.lo[k] - grow - self.blo[k], self.hi[k] + grow - self.blo[k])
                   for k in (2, 1, 0))
        m[sl] = True
        m &= self.bgb >= 2
        return m, self.bgb[m].astype(np.int64)

    def upload(self, g, dense_f32):
        m, ids = self.region(1)
        vals = self.O.box_to_packages(dense_f32)[m]
        g.view("phi")[torch.from_numpy(ids).cuda()] = torch.from_numpy(
            np.ascontiguousarray(vals, dtype=np.float32)).cuda()


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("name", list(WINDOWS))
def test_window_reinit(sgm, O, name):
    win = Win(O, name)
    w, o, dx = win.w, win.o, win.dx
    m, ids = win.region(0)
    assert ids.size > 100, "window must contain band packages"
    phi0 = o.phi_dense()
    # (1) 20-sweep drift of the GPU's own iterate
    g = sgm.Grid(w)
    g.reinit(20)
    gid = torch.from_numpy(ids).cuda()
    got = g.view("phi")[gid].cpu().numpy().astype(np.float64)
    p20 = o.reinit(phi0, 20)
    exp = O.box_to_packages(p20)[m]
    drift = np.max(np.abs(got - exp)) / dx
    assert drift <= 20 * 1e-5, f"{name}: 20-sweep drift {drift:.3e} dx"
    # (2) one sweep from the oracle's 10-sweep state
    p10 = f32(o.reinit(phi0, 10))
    g2 = sgm.Grid(w)
    win.upload(g2, p10)
    g2.reinit(1)
    got1 = g2.view("phi")[gid].cpu().numpy().astype(np.float64)
    exp1 = O.box_to_packages(o.reinit_step(p10))[m]
    err = np.max(np.abs(got1 - exp1)) / dx
    assert err <= 1e-5, f"{name}: one sweep {err:.3e} dx"


@pytest.mark.parametrize("name", list(WINDOWS))
def test_window_gradient_kernel_probe(sgm, O, name):
    win = Win(O, name)
    w, o, dx = win.w, win.o, win.dx
    m, ids = win.region(0)
    gid = torch.from_numpy(ids).cuda()
    p20 = f32(o.reinit(o.phi_dense(), 20))
    g = sgm.Grid(w)
    win.upload(g, p20)
    g.gradient(sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT, h_ratio=w.h_ratio)
    grad, normal = o.gradient(p20)
    K, G = o.kernel_integrals(p20, w.h_ratio)
    eg = O.box_to_packages(grad)[:, m].transpose(1, 0, 2)   # [pkg][3][64]
    en = O.box_to_packages(normal)[:, m].transpose(1, 0, 2)
    eK = O.box_to_packages(K)[m]
    eG = O.box_to_packages(G)[:, m].transpose(1, 0, 2)
    g4 = g.view("grad")[gid].cpu().numpy().astype(np.float64)      # [pkg][64][4]
    gg = g4[:, :, 1:].transpose(0, 2, 1)
    gn = g.view("normal")[gid].cpu().numpy().astype(np.float64)
    gK = g.view("kint")[gid].cpu().numpy().astype(np.float64)
    gG = g.view("gkint")[gid].cpu().numpy().astype(np.float64)
    assert np.array_equal(g4[:, :, 0], f32(O.box_to_packages(p20)[m]))
    tol = 1e-5
    assert np.max(np.abs(gg - eg) / np.maximum(1.0, np.abs(eg))) <= tol
    big = np.broadcast_to(np.linalg.norm(eg, axis=1, keepdims=True) >= 0.5, en.shape)
    assert np.max(np.abs(gn - en)[big]) <= tol
    assert np.max(np.abs(gK - eK)) <= tol
    h = w.h_ratio * dx
    assert np.max(np.abs(gG - eG) / (np.maximum(1.0, h * np.abs(eG)) / h)) <= tol
    S = g.info["kernel_sum"]
    assert ((eK > 1e-3 * S) & (eK < (1 - 1e-3) * S)).sum() > 1000  # the smoothing band
    # probe at random positions of I (fp32), on the uploaded state
    rng = np.random.default_rng(7)
    a = np.array([w.lower[k] + win.lo[k] * w.cell for k in range(3)])
    b = np.array([w.lower[k] + win.hi[k] * w.cell for k in range(3)])
    pos = rng.uniform(a, b, size=(200000, 3)).astype(np.float32)
    gphi, ggrad = g.probe(torch.from_numpy(pos).cuda())
    ephi, egrad, eoob = o.probe(p20, f32(grad), pos)
    assert eoob == 0
    band = np.abs(ephi) < o.far
    assert band.mean() > 0.05, "window must put probes in the band"
    assert np.max(np.abs(gphi.cpu().numpy().astype(np.float64) - ephi)) <= 1e-5 * dx
    eg3 = egrad
    gg3 = ggrad.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(gg3 - eg3) / np.maximum(1.0, np.abs(eg3))) <= tol


@pytest.mark.parametrize("name", ["C5-shell", "C5-small"])
def test_window_probe_c5_particles(sgm, O, name):
    """The C5 particle recipe (lattice points inside the shell walls,
    workloads.shell_lattice_particles) restricted to the window: probe of the
    uploaded 20-sweep state against the oracle."""
    win = Win(O, name)
    w, o, dx = win.w, win.o, win.dx
    p20 = f32(o.reinit(o.phi_dense(), 20))
    g = sgm.Grid(w)
    win.upload(g, p20)
    g.gradient(sgm.SG_GRAD, h_ratio=w.h_ratio)
    grad, _ = o.gradient(p20)
    box = (tuple(4 * v for v in win.lo), tuple(4 * v for v in win.hi))
    pos = W.shell_lattice_particles(w, box=box, device="cuda")
    assert pos.shape[0] > 5000
    gphi, ggrad = g.probe(pos)
    pos_np = pos.cpu().numpy()
    ephi, egrad, eoob = o.probe(p20, f32(grad), pos_np)
    assert eoob == 0
    # the wall middle (> l_c from both surfaces) is inactive: about half the
    # wall particles are band particles
    assert (np.abs(ephi) < o.far).mean() > 0.3
    assert np.max(np.abs(gphi.cpu().numpy().astype(np.float64) - ephi)) <= 1e-5 * dx
    gg = ggrad.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(gg - egrad) / np.maximum(1.0, np.abs(egrad))) <= 1e-5
