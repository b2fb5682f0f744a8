"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Tables (background, meta, neighbours, plane ranges) must be bit-exact.
Fields use the tolerances of DESIGN.md "Tolerances" (north_star: 1e-5 dx per
reinit iteration in fp32, 1e-12 relative in fp64).  Oracle inputs never come
from the GPU: multi-step comparisons feed the ORACLE's state into the GPU.
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


def np_dtype(w):
    return np.float64 if w.dtype == "f64" else np.float32


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def phi_tol(w):
    return 1e-5 * w.dx if w.dtype == "f32" else None


def assert_phi_close(w, got, exp, what=""):
    got = np.asarray(got, dtype=np.float64)
    if w.dtype == "f32":
        err = np.max(np.abs(got - exp)) if got.size else 0.0
        assert err <= 1e-5 * w.dx, f"{what}: max err {err / w.dx:.3e} dx"
    else:
        scale = np.maximum(np.abs(exp), w.dx)
        err = np.max(np.abs(got - exp) / scale) if got.size else 0.0
        assert err <= 1e-12, f"{what}: max rel err {err:.3e}"


FACE_SLOTS = [12, 14, 10, 16, 4, 22]  # -x, +x, -y, +y, -z, +z (ox + 3 oy + 9 oz)


def assert_face_table(g):
    """The compact face table the 7-point sweeps read is the neighbour table's
    six face slots (plus two zero pads), for every package."""
    face, nb = u32(g.view("face")), u32(g.view("nb"))
    assert face.shape == (nb.shape[0], 8)
    assert np.array_equal(face[:, :6], nb[:, FACE_SLOTS])
    assert not face[:, 6:].any()


def tables_equal(sgm, O, w):
    o = O.Oracle(w)
    t = o.build_tables()
    g = sgm.Grid(w)
    info = g.info
    assert info["n_pkg"] == t.n_pkg
    assert info["n_core"] == int(np.count_nonzero(t.cat == 3))
    assert info["n_inner"] == int(np.count_nonzero(t.cat == 2))
    assert np.array_equal(u32(g.view("bg")), t.bg)
    assert np.array_equal(u32(g.view("meta_cell")), t.meta_cell)
    assert np.array_equal(g.view("meta_cat").cpu().numpy(), t.meta_cat)
    assert np.array_equal(u32(g.view("nb")), t.nb)
    assert_face_table(g)
    pf = g.view("plane_first").cpu().numpy()
    exp_pf = 2 + np.concatenate([[0], np.cumsum(t.plane_count)])
    assert np.array_equal(pf, exp_pf)
    return o, t, g


# ------------------------------------------------------------------ tables --

@pytest.mark.parametrize("name", ["C1", "C2"])
def test_tables_bit_exact_configs(sgm, O, name):
    tables_equal(sgm, O, W.config(name))


@pytest.mark.parametrize("seed,n", [(0, 8), (1, 13), (2, 16), (3, 24), (4, 9), (5, 20), (6, 17), (7, 31)])
def test_tables_bit_exact_random_scenes(sgm, O, seed, n):
    tables_equal(sgm, O, W.random_scene(seed, n, dtype="f64" if seed % 2 else "f32"))


def test_tables_nonuniform_grid_and_offset(sgm, O):
    w = W.Workload("aniso", (23, 9, 14), 0.05, lower=(-0.3, 0.1, -0.2), dtype="f32",
                   prims=(W.Prim(W.TORUS_Z, (0.25, 0.32, 0.15, 0.25, 0.08)),
                          W.Prim(W.SPHERE, (0.7, 0.3, 0.4, 0.12))))
    tables_equal(sgm, O, w)


def test_band_touching_domain_boundary(sgm, O):
    # sphere reaching outside the domain: out-of-domain neighbours by sign (R-6)
    w = W.Workload("edge", (12, 12, 12), 1 / 12, dtype="f64",
                   prims=(W.Prim(W.SPHERE, (0.1, 0.5, 0.5, 0.35)),))
    o, t, g = tables_equal(sgm, O, w)
    assert (t.nb[2:] <= 1).any()
    # fields too
    phi0 = o.phi_dense()
    gp = g.view("phi").cpu().numpy()
    assert_phi_close(w, gp, o.to_packages(phi0, -o.far, o.far), "init")
    g.reinit(1)
    assert_phi_close(w, g.view("phi").cpu().numpy(),
                     o.to_packages(o.reinit_step(phi0), -o.far, o.far), "reinit")


def test_empty_band_and_single_cell(sgm, O):
    # geometry entirely outside the domain: no packages, all far field
    w = W.Workload("empty", (8, 8, 8), 1 / 8, dtype="f32",
                   prims=(W.Prim(W.SPHERE, (5.0, 5.0, 5.0, 0.3)),))
    o, t, g = tables_equal(sgm, O, w)
    assert g.info["n_pkg"] == 2
    g.reinit(3).gradient(sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT)
    pos = torch.tensor([[0.5, 0.5, 0.5], [0.1, 0.2, 0.3]], dtype=torch.float32, device="cuda")
    phi, grad = g.probe(pos)
    assert torch.all(phi == o.far) and torch.all(grad == 0)
    # n = 1 background cell
    w1 = W.Workload("one", (1, 1, 1), 0.5, dtype="f64", prims=(W.Prim(W.SPHERE, (0.25, 0.25, 0.25, 0.2)),))
    o1, t1, g1 = tables_equal(sgm, O, w1)
    assert g1.info["n_pkg"] == 3
    g1.reinit(1)
    assert_phi_close(w1, g1.view("phi").cpu().numpy(),
                     o1.to_packages(o1.reinit_step(o1.phi_dense()), -o1.far, o1.far))


def test_argument_errors(sgm):
    w = W.config("C1")
    d, geom, keep = sgm.make_desc(w)
    d.pkg = 3
    with pytest.raises(sgm.SgError) as e:
        sgm.sg_build(d, geom)
    assert e.value.status == sgm.SG_ERR_ARG
    g = sgm.Grid(w)
    with pytest.raises(sgm.SgError):
        g.reinit(1, cfl=0.7)
    with pytest.raises(sgm.SgError):
        g.gradient(sgm.SG_KINT, h_ratio=3.0)
    pos = torch.zeros((4, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(sgm.SgError) as e:
        g.probe(pos, want_grad=True)  # no gradient yet
    assert e.value.status == sgm.SG_ERR_STATE


# ------------------------------------------------------------------ fields --

@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C1", 2.0), ("C2", 1.0)])
def test_phi_init(sgm, O, name, scale):
    w = W.config(name).with_(init_scale=scale)
    o = O.Oracle(w)
    o.build_tables()
    exp = o.to_packages(o.phi_dense(), -o.far, o.far)
    g = sgm.Grid(w)
    got = g.view("phi").cpu().numpy()
    # fp64 SDF with identical operation order on both sides, then RN to dtype
    assert np.array_equal(got, exp.astype(np_dtype(w)))


TORUS_Y_BOX = W.Workload("TYB24", (24, 24, 24), 1.0 / 24, dtype="f32",
                         prims=(W.Prim(W.TORUS_Y, (0.5, 0.5, 0.5, 0.3, 0.08)),
                                W.Prim(W.BOX, (0.5, 0.5, 0.5, 0.1, 0.1, 0.4))))


@pytest.mark.parametrize("seed,n,dtype", [(s, n, d) for s, n in [(0, 13), (1, 16), (2, 20), (3, 24),
                                                                  (6, 17), (9, 21), (12, 19)]
                                          for d in ("f64", "f32")] + [(-1, 24, "f32")])
def test_phi_init_random_scenes(sgm, O, seed, n, dtype):
    """Initial phi bit-exact on unions of every primitive kind (the y-column
    evaluation for tori about y, the z-column one otherwise, the per-package
    primitive mask)."""
    w = TORUS_Y_BOX if seed < 0 else W.random_scene(seed, n, dtype=dtype)
    o = O.Oracle(w)
    o.build_tables()
    exp = o.to_packages(o.phi_dense(), -o.far, o.far)
    g = sgm.Grid(w)
    assert np.array_equal(g.view("phi").cpu().numpy(), exp.astype(np_dtype(w)))


def _upload(g, w, pk):
    g.view("phi").copy_(torch.from_numpy(pk.astype(np_dtype(w))))


@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C1", 2.0), ("C2", 1.0), ("C2", 2.0)])
def test_reinit_per_iteration(sgm, O, name, scale):
    """One sweep from the same input state, at k = 0 and k = 10 oracle
    iterations (the oracle state rounded to dtype is uploaded to the GPU)."""
    w = W.config(name).with_(init_scale=scale)
    o = O.Oracle(w)
    o.build_tables()
    g = sgm.Grid(w)
    phi = o.phi_dense()
    dt = np_dtype(w)
    for k in (0, 10):
        if k:
            phi = o.reinit(phi, k)
        phi_in = phi.astype(dt).astype(np.float64)  # exactly the GPU's input
        _upload(g, w, o.to_packages(phi_in, -o.far, o.far))
        exp = o.to_packages(o.reinit_step(phi_in), -o.far, o.far)
        g.reinit(1)
        assert_phi_close(w, g.view("phi").cpu().numpy(), exp, f"{name} step {k}")


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_reinit_drift_20(sgm, O, name):
    """20 GPU sweeps vs 20 oracle sweeps from the same init: flag if the
    drift exceeds 20 x the per-step tolerance."""
    w = W.config(name)
    o = O.Oracle(w)
    o.build_tables()
    g = sgm.Grid(w)
    g.reinit(20)
    exp = o.to_packages(o.reinit(o.phi_dense(), 20), -o.far, o.far)
    got = g.view("phi").cpu().numpy().astype(np.float64)
    if w.dtype == "f32":
        assert np.max(np.abs(got - exp)) <= 20 * 1e-5 * w.dx
    else:
        assert np.max(np.abs(got - exp) / np.maximum(np.abs(exp), w.dx)) <= 20 * 1e-12


def _vec_pk(o, dense3):
    return np.stack([o.to_packages(dense3[c], 0.0, 0.0) for c in range(3)], axis=1)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_gradient_normal_kernel(sgm, O, name):
    w = W.config(name)
    o = O.Oracle(w)
    o.build_tables()
    phi = o.reinit(o.phi_dense(), 5).astype(np_dtype(w)).astype(np.float64)
    g = sgm.Grid(w)
    _upload(g, w, o.to_packages(phi, -o.far, o.far))
    g.gradient(sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT, h_ratio=w.h_ratio)
    grad, normal = o.gradient(phi)
    eg, en = _vec_pk(o, grad), _vec_pk(o, normal)
    g4 = g.view("grad").cpu().numpy().astype(np.float64)  # [n_pkg][64][(phi, gx, gy, gz)]
    assert np.array_equal(g4[:, :, 0], g.view("phi").cpu().numpy().astype(np.float64))
    gg = g4[:, :, 1:].transpose(0, 2, 1)
    gn = g.view("normal").cpu().numpy().astype(np.float64)
    tol = 1e-5 if w.dtype == "f32" else 1e-12
    assert np.max(np.abs(gg - eg) / np.maximum(1.0, np.abs(eg))) <= tol
    m = np.linalg.norm(eg, axis=1, keepdims=True) >= 0.5
    mm = np.broadcast_to(m, en.shape)
    assert np.max(np.abs(gn - en)[mm]) <= tol
    K, G = o.kernel_integrals(phi, w.h_ratio)
    S = O.kernel_taps(w.h_ratio, o.dx)[1].sum()
    eK = o.to_packages(K, S, 0.0)  # singular packages: S / 0 (R-16)
    eG = _vec_pk(o, G)
    gK = g.view("kint").cpu().numpy().astype(np.float64)
    gG = g.view("gkint").cpu().numpy().astype(np.float64)
    assert abs(g.info["kernel_sum"] - S) < 1e-12
    assert np.max(np.abs(gK - eK)) <= tol
    h = w.h_ratio * w.dx
    assert np.max(np.abs(gG - eG) / (np.maximum(1.0, h * np.abs(eG)) / h)) <= tol


@pytest.mark.parametrize("h_ratio", [0.5, 1.0, 1.3, 1.45, 1.7])
def test_kernel_integral_h_ratios(sgm, O, h_ratio):
    """K7 at every staged radius R = ceil(2 h_ratio) - 1 (0..3), including
    R = 2 with (1.45) and without (1.3) the |o|^2 = 8 taps in the support."""
    w = W.config("C1")
    o = O.Oracle(w)
    o.build_tables()
    phi = o.reinit(o.phi_dense(), 3)
    g = sgm.Grid(w)
    _upload(g, w, o.to_packages(phi, -o.far, o.far))
    g.gradient(sgm.SG_KINT, h_ratio=h_ratio)
    K, G = o.kernel_integrals(phi, h_ratio)
    S = O.kernel_taps(h_ratio, o.dx)[1].sum()
    assert abs(g.info["kernel_sum"] - S) < 1e-12
    gK = g.view("kint").cpu().numpy()
    gG = g.view("gkint").cpu().numpy()
    assert np.max(np.abs(gK - o.to_packages(K, S, 0.0))) <= 1e-12
    h = h_ratio * w.dx
    eG = _vec_pk(o, G)
    assert np.max(np.abs(gG - eG) / (np.maximum(1.0, h * np.abs(eG)) / h)) <= 1e-12


@pytest.mark.parametrize("name,h_ratio", [("C1", 1.3), ("C1", 0.5), ("C2", 1.3), ("C2", 1.6),
                                          ("C2", 0.9)])
def test_fused_gradient_kernel_equals_separate(sgm, name, h_ratio):
    """SG_GRAD|SG_NORMAL|SG_KINT in one call runs K6 warps beside K7 warps in
    one kernel; it must give the bits of the separate K6 and K7 calls."""
    w = W.config(name)
    a = sgm.Grid(w).reinit(3)
    b = sgm.Grid(w).reinit(3)
    a.gradient(sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT, h_ratio=h_ratio)
    b.gradient(sgm.SG_GRAD | sgm.SG_NORMAL, h_ratio=h_ratio)
    b.gradient(sgm.SG_KINT, h_ratio=h_ratio)
    for f in ("grad", "normal", "kint", "gkint"):
        assert torch.equal(a.view(f), b.view(f)), f


# ------------------------------------------------------------------- probe --

def _probe_compare(sgm, O, w, pos_np, phi_iters=3):
    o = O.Oracle(w)
    o.build_tables()
    phi = o.reinit(o.phi_dense(), phi_iters).astype(np_dtype(w)).astype(np.float64)
    g = sgm.Grid(w)
    _upload(g, w, o.to_packages(phi, -o.far, o.far))
    g.gradient(sgm.SG_GRAD)
    grad, _ = o.gradient(phi)
    grad = grad.astype(np_dtype(w)).astype(np.float64)  # the GPU stores grad in dtype
    # the oracle interpolates the same dtype-rounded grad the GPU stores
    pos = torch.from_numpy(pos_np).cuda()
    oob = torch.zeros(1, dtype=torch.int64, device="cuda")
    gphi, ggrad = g.probe(pos, oob=oob)
    ephi, egrad, eoob = o.probe(phi, grad, pos_np)
    gphi = gphi.cpu().numpy().astype(np.float64)
    ggrad = ggrad.cpu().numpy().astype(np.float64)
    assert int(oob.item()) == eoob
    assert_phi_close(w, gphi, ephi, "probe phi")
    tol = 1e-5 if w.dtype == "f32" else 1e-12
    assert np.max(np.abs(ggrad - egrad) / np.maximum(1.0, np.abs(egrad))) <= tol
    return g, o, pos, gphi, ggrad


def test_probe_c1_lattice_and_random(sgm, O):
    w = W.config("C1")
    lat = W.lattice_particles(w, dtype=np.float64)
    rnd = W.random_positions(w, 20000, seed=3)
    bad = np.array([[-0.1, 0.5, 0.5], [0.5, 1.0, 0.5], [np.nan, 0.5, 0.5], [0.5, 0.5, 1.5]])
    faces = rnd[:2000].copy()
    faces[:, 0] = np.round(faces[:, 0] / w.cell) * w.cell  # exactly on package faces
    pos = np.concatenate([lat, rnd, bad, faces])
    g, o, tpos, gphi, ggrad = _probe_compare(sgm, O, w, pos)
    # host-buffer path (C-ABI with host pointers) is bitwise the device path
    hpos = tpos.cpu().pin_memory()
    hphi, hgrad = g.probe(hpos)
    assert np.array_equal(hphi.numpy(), gphi) and np.array_equal(hgrad.numpy(), ggrad)
    pphi, pgrad = g.probe(tpos.cpu())  # pageable
    assert np.array_equal(pphi.numpy(), gphi)
    # the host path's kernels wait for work still queued on the caller's
    # stream (its uploads do not): new fields queued right before the call
    g.reinit(5).gradient(sgm.SG_GRAD)
    hphi2, hgrad2 = g.probe(hpos)
    dphi2, dgrad2 = g.probe(tpos)
    assert not np.array_equal(hphi2.numpy(), hphi.numpy())
    assert np.array_equal(hphi2.numpy(), dphi2.cpu().numpy())
    assert np.array_equal(hgrad2.numpy(), dgrad2.cpu().numpy())


def test_probe_c4_particles_on_c2(sgm, O):
    """C4: ~19.45 M lattice particles (jittered, sorted) on the C2 grid."""
    w = W.config("C2")
    pos = W.lattice_particles(w, seed=0)
    g, o, tpos, gphi, ggrad = _probe_compare(sgm, O, w, pos)
    assert pos.shape[0] == 19454436
    far = np.abs(gphi) == np.float32(o.far)
    frac_band = 1.0 - far.mean()
    assert 0.15 < frac_band < 0.23  # ~18.9 % in active cells
    # host buffers (the e2e path: 16 pipelined chunks on two staging streams,
    # uploads overlapping the caller's stream) give the device path's bits
    hphi, hgrad = g.probe(tpos.cpu().pin_memory())
    assert np.array_equal(hphi.numpy(), gphi) and np.array_equal(hgrad.numpy(), ggrad)


def test_probe_empty_and_zero(sgm, O):
    w = W.config("C1")
    g = sgm.Grid(w)
    pos = torch.empty((0, 3), dtype=torch.float64, device="cuda")
    phi, grad = g.probe(pos, want_grad=False)
    assert phi.numel() == 0


# ----------------------------------------------------------- Table 1 ops ---

@pytest.mark.parametrize("name", ["C1", "C2"])
def test_table1_sequential_and_laplacian(sgm, O, name):
    """Table-1 workloads (NEXT-1) against the oracle on the same
    input phi: sequential add (phi + value at active points) and the 7-point
    Laplacian at active points."""
    w = W.config(name)
    o = O.Oracle(w)
    o.build_tables()
    phi = o.reinit(o.phi_dense(), 2).astype(np_dtype(w)).astype(np.float64)
    g = sgm.Grid(w)
    _upload(g, w, o.to_packages(phi, -o.far, o.far))
    g.table1(1)  # stencil -> phi_next (active packages)
    lap = g.view("phi_next").cpu().numpy().astype(np.float64)[2:]
    elap = o.to_packages(o.table1(phi, 1), 0.0, 0.0)[2:]
    # (sum - 6 phi) / dx^2 of values |phi| <= 16 dx: a few roundings of 16 dx
    # relative to dx^2 -> tolerance 1e-5 / dx (fp32) / 1e-12 / dx (fp64)
    tol = (1e-5 if w.dtype == "f32" else 1e-12) * 16 / w.dx
    assert np.max(np.abs(lap - elap)) <= tol
    g.table1(0, 0.25)  # sequential, in place
    seq = g.view("phi").cpu().numpy().astype(np.float64)
    eseq = o.to_packages(o.table1(phi, 0, 0.25), -o.far, o.far)
    ulp = np.spacing(np.abs(eseq).astype(np_dtype(w))).astype(np.float64)
    assert np.all(np.abs(seq - eseq) <= ulp)


# ----------------------------------------------------- full size, sampled --

def test_c3_full_size_sampled(sgm, O):
    """C3 (2048^3 effective): tables bit-exact in full; phi init and the first
    reinit sweep at sampled points against the oracle's pointwise forms."""
    w = W.config("C3")
    o, t, g = tables_equal(sgm, O, w)
    phi = g.view("phi")
    rng = np.random.default_rng(11)
    ids = rng.integers(2, t.n_pkg, 3000)
    ds = rng.integers(0, 64, 3000)
    cells = t.meta_cell[ids].astype(np.int64)
    cx, cy, cz = cells % 512, (cells // 512) % 512, cells // (512 * 512)
    ix, iy, iz = 4 * cx + (ds & 3), 4 * cy + ((ds >> 2) & 3), 4 * cz + (ds >> 4)
    got0 = phi.cpu().numpy()[ids, ds]
    exp0 = np.array([o.phi_point(a, b, c) for a, b, c in zip(ix, iy, iz)])
    assert np.array_equal(got0, exp0.astype(np.float32))
    g.reinit(1)
    got1 = g.view("phi").cpu().numpy()[ids, ds].astype(np.float64)
    exp1 = np.array([o.reinit_point_from_init(a, b, c, w.cfl) for a, b, c in zip(ix, iy, iz)])
    # the GPU's input is the fp32-rounded init; the pointwise oracle uses the
    # fp64 init: allow the input rounding (0.5 ulp of |phi| <= 16 dx) on top
    assert np.max(np.abs(got1 - exp1)) <= 1e-5 * w.dx + 2 * 16 * w.dx * 2**-24


def test_c5_full_size(sgm, O):
    """C5 (4096^3 effective, ~10^9 active data points): the whole background
    table, meta and neighbour table bit-exact against the oracle; phi init and
    the first reinit sweep at sampled data points."""
    w = W.config("C5")
    o = O.Oracle(w)
    t = o.build_tables()
    assert t.n_pkg - 2 == 15166440  # SURVEY App. A (tests/golden/tagging_counts.json)
    g = sgm.Grid(w)
    info = g.info
    assert info["n_pkg"] == t.n_pkg
    assert np.array_equal(g.view("plane_first").cpu().numpy(),
                          2 + np.concatenate([[0], np.cumsum(t.plane_count)]))
    assert np.array_equal(u32(g.view("bg")), t.bg)
    assert np.array_equal(u32(g.view("meta_cell")), t.meta_cell)
    assert np.array_equal(u32(g.view("nb")), t.nb)
    rng = np.random.default_rng(13)
    ids = rng.integers(2, t.n_pkg, 2000)
    ds = rng.integers(0, 64, 2000)
    cells = t.meta_cell[ids].astype(np.int64)
    n = w.n[0]
    cx, cy, cz = cells % n, (cells // n) % n, cells // (n * n)
    ix, iy, iz = 4 * cx + (ds & 3), 4 * cy + ((ds >> 2) & 3), 4 * cz + (ds >> 4)
    got0 = g.view("phi")[torch.from_numpy(ids).cuda(), torch.from_numpy(ds).cuda()].cpu().numpy()
    exp0 = np.array([o.phi_point(a, b, c) for a, b, c in zip(ix, iy, iz)])
    assert np.array_equal(got0, exp0.astype(np.float32))
    g.reinit(1)
    got1 = g.view("phi")[torch.from_numpy(ids).cuda(), torch.from_numpy(ds).cuda()].cpu().numpy()
    exp1 = np.array([o.reinit_point_from_init(a, b, c, w.cfl) for a, b, c in zip(ix, iy, iz)])
    assert np.max(np.abs(got1.astype(np.float64) - exp1)) <= 1e-5 * w.dx + 2 * 16 * w.dx * 2**-24


def test_probe_offset_grid_fp32(sgm, O):
    """fp32 probe on a grid with a non-zero lower corner and a non-dyadic
    cell size (the general fp64 index path of the kernel)."""
    w = W.Workload("aniso", (23, 9, 14), 0.05, lower=(-0.3, 0.1, -0.2), dtype="f32",
                   prims=(W.Prim(W.TORUS_Z, (0.25, 0.32, 0.15, 0.25, 0.08)),
                          W.Prim(W.SPHERE, (0.7, 0.3, 0.4, 0.12))))
    rng = np.random.default_rng(21)
    lo = np.array(w.lower)
    hi = lo + np.array(w.n) * w.cell
    pos = rng.uniform(lo - 0.01, hi + 0.01, size=(50000, 3)).astype(np.float32)
    _probe_compare(sgm, O, w, pos, phi_iters=2)


def test_probe_shuffled_c4_matches_lattice(sgm, O):
    """The probe is a pure per-particle function: a seeded permutation of the
    C4 particles gives the permuted results bit for bit."""
    w = W.config("C2")
    g = sgm.Grid(w)
    g.reinit(3).gradient(sgm.SG_GRAD)
    pos = W.lattice_particles(w, seed=0)
    perm = np.random.default_rng(1).permutation(pos.shape[0])
    a_phi, a_grad = g.probe(torch.from_numpy(pos).cuda())
    b_phi, b_grad = g.probe(torch.from_numpy(pos[perm]).cuda())
    p = torch.from_numpy(perm).cuda()
    assert torch.equal(a_phi[p], b_phi) and torch.equal(a_grad[p], b_grad)


def test_tables_with_forced_tag_cull(O):
    """The Lipschitz-culled tagging kernel (default only for >= 2^25 cells) on
    small scenes with partial words and boundary-touching bands, in a fresh
    process with SG_TAG_CULL=1: tables bit-exact."""
    import subprocess
    import sys
    code = (
        "import numpy as np, workloads as W\n"
        "from oracle.oracle import Oracle\n"
        "from paper_2512_11473_b200 import sg\n"
        "for seed, n in [(0, 8), (1, 13), (3, 24), (5, 20), (7, 31), (9, 40)]:\n"
        "    w = W.random_scene(seed, n)\n"
        "    t = Oracle(w).build_tables(); g = sg.Grid(w)\n"
        "    assert np.array_equal(g.view('bg').cpu().numpy().view(np.uint32), t.bg), (seed, n)\n"
        "    assert np.array_equal(g.view('nb').cpu().numpy().view(np.uint32), t.nb), (seed, n)\n"
        "w = W.Workload('aniso', (45, 19, 14), 0.05, lower=(-0.3, 0.1, -0.2), prims=(W.Prim(W.TORUS_Z, (0.25, 0.32, 0.15, 0.25, 0.08)),))\n"
        "t = Oracle(w).build_tables(); g = sg.Grid(w)\n"
        "assert np.array_equal(g.view('bg').cpu().numpy().view(np.uint32), t.bg)\n"
        "print('ok')\n")
    import os
    env = dict(os.environ, SG_TAG_CULL="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


# -------------------------------------------------- NEXT-2: relaxation ----

def _relax_setup(sgm, O, w, iters=2):
    o = O.Oracle(w)
    o.build_tables()
    phi = o.reinit(o.phi_dense(), iters).astype(np_dtype(w)).astype(np.float64)
    g = sgm.Grid(w)
    _upload(g, w, o.to_packages(phi, -o.far, o.far))
    g.gradient(sgm.SG_GRAD | sgm.SG_KINT, w.h_ratio)
    grad, _ = o.gradient(phi)
    _, G = o.kernel_integrals(phi, w.h_ratio)
    # the GPU stores grad / G in dtype: the oracle interpolates the same values
    dt = np_dtype(w)
    return o, g, phi, grad.astype(dt).astype(np.float64), G.astype(dt).astype(np.float64)


def test_relax_c1_fp64(sgm, O):
    """Three relaxation steps of the C1 lattice particles (dp = dx) against the
    brute-force oracle (reading R-21)."""
    w = W.config("C1")
    o, g, phi, grad, G = _relax_setup(sgm, O, w)
    pos = W.lattice_particles(w, dtype=np.float64)
    exp = o.relax(phi, grad, G, pos, dp=w.dx, steps=3)
    t = torch.from_numpy(pos.copy()).cuda()
    g.relax(t, dp=w.dx, steps=3)
    got = t.cpu().numpy()
    assert np.max(np.abs(got - exp)) <= 1e-10 * w.dx
    moved = np.linalg.norm(got - pos, axis=1)
    assert moved.max() > 0.01 * w.dx  # it does something
    # containment after bounding: every particle inside (phi <= 0);
    # the projection along the interpolated normal lands near -off dp
    gp, _ = g.probe(torch.from_numpy(got).cuda(), want_grad=False)
    assert float(gp.max()) <= 0.0
    assert float(gp.max()) <= -0.4 * w.dx


def test_relax_c2_subset_fp32(sgm, O):
    """fp32: a 20k-particle subset of C4 near the prism's edge and top face."""
    w = W.config("C2")
    o, g, phi, grad, G = _relax_setup(sgm, O, w)
    pos = W.lattice_particles(w, seed=0)
    sel = (np.abs(pos[:, 0] - 0.5) < 0.03) & (np.abs(pos[:, 1] - 0.3) < 0.03) & (pos[:, 2] > 0.8)
    pos = np.ascontiguousarray(pos[sel][:20000])
    assert pos.shape[0] > 2000
    exp = o.relax(phi, grad, G, pos.astype(np.float64), dp=w.dx, steps=1)
    t = torch.from_numpy(pos.copy()).cuda()
    g.relax(t, dp=w.dx, steps=1)
    got = t.cpu().numpy().astype(np.float64)
    tol = 4 * np.spacing(np.float32(1.0)) + 1e-5 * w.dx
    assert np.max(np.abs(got - exp)) <= tol


def test_probe_unaligned_buffers(sgm, O):
    """Buffers that are not 16 B aligned take the scalar staging path: the
    results equal those of an aligned copy bit for bit."""
    w = W.config("C2")
    g = sgm.Grid(w)
    g.reinit(2).gradient(sgm.SG_GRAD)
    pos = torch.from_numpy(W.lattice_particles(w, seed=3)[:300001]).cuda()
    big = torch.empty((pos.shape[0] + 1, 3), dtype=pos.dtype, device="cuda")
    big[1:] = pos
    un = big[1:]  # 12 B offset
    assert un.data_ptr() % 16 != 0
    a_phi, a_grad = g.probe(pos)
    b_phi = torch.empty(pos.shape[0] + 1, dtype=pos.dtype, device="cuda")[1:]
    b_grad = torch.empty((pos.shape[0] + 1, 3), dtype=pos.dtype, device="cuda")[1:]
    sgm.sg_probe(g.handle, pos.shape[0], un.data_ptr(), b_phi.data_ptr(), b_grad.data_ptr())
    assert torch.equal(a_phi, b_phi) and torch.equal(a_grad, b_grad)


# ------------------------------------------------ edge cases (round 2) ----

LOWFACE = W.Workload("lowface", (16, 16, 16), 1.0 / 16, dtype="f32",
                     prims=(W.Prim(W.SPHERE, (0.1, 0.45, 0.55, 0.2)),))


def _lowface_positions(w, n=40000, seed=4):
    """Positions with x in [0, dx/4) (the fp32 fast path's u = x/dx - 1/2 is
    rounded there) inside the band near the lower x face, plus x = 0 exactly
    and tiny x."""
    rng = np.random.default_rng(seed)
    dx = w.cell / 4
    pos = np.empty((n, 3))
    pos[:, 0] = rng.uniform(0.0, 0.25 * dx, n)
    pos[:, 1] = rng.uniform(0.3, 0.6, n)
    pos[:, 2] = rng.uniform(0.4, 0.7, n)
    pos[:50, 0] = 0.0
    pos[50:100, 0] = np.ldexp(1.0, -rng.integers(20, 120, 50))
    return pos.astype(np.float32)


def test_probe_lower_face_fp32(sgm, O):
    """fp32 dyadic grid whose band touches the lower x face (out-of-domain
    neighbours by sign, R-6), particles at x < dx/4: against the oracle, and
    the exact fp32 index path against the fp64 index path bit for bit (the
    latter in a fresh process with SG_PROBE_IDX32=0)."""
    w = LOWFACE
    pos = _lowface_positions(w)
    g, o, tpos, gphi, ggrad = _probe_compare(sgm, O, w, pos, phi_iters=2)
    assert (np.abs(gphi) < o.far).mean() > 0.5  # in the band
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import tempfile
    tmp = os.path.join(tempfile.mkdtemp(), "lowface_idx64.npz")
    code = (
        "import numpy as np, torch, sys\n"
        "sys.path.insert(0, 'tests')\n"
        "from test_parity_gpu import LOWFACE, _lowface_positions\n"
        "from paper_2512_11473_b200 import sg\n"
        "g = sg.Grid(LOWFACE); g.reinit(2).gradient(sg.SG_GRAD)\n"
        "p, gr = g.probe(torch.from_numpy(_lowface_positions(LOWFACE)).cuda())\n"
        f"np.savez({tmp!r}, phi=p.cpu().numpy(), grad=gr.cpu().numpy())\n")
    env = dict(os.environ, SG_PROBE_IDX32="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    ref = np.load(tmp)
    g2 = sgm.Grid(w)
    g2.reinit(2).gradient(sgm.SG_GRAD)
    a_phi, a_grad = g2.probe(tpos)
    assert np.array_equal(a_phi.cpu().numpy(), ref["phi"])
    assert np.array_equal(a_grad.cpu().numpy(), ref["grad"])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_reinit_phi_exactly_zero(sgm, O, dtype):
    """O7's stationary case: an active point with phi = 0 exactly stays 0 and
    its neighbours update as the definition says."""
    w = W.config("C1").with_(dtype=dtype)
    o = O.Oracle(w)
    t = o.build_tables()
    phi = o.reinit(o.phi_dense(), 3).astype(np_dtype(w)).astype(np.float64)
    rng = np.random.default_rng(2)
    band = np.argwhere(np.abs(phi) < 1.5 * w.dx)
    pick = band[rng.choice(band.shape[0], 200, replace=False)]
    phi[pick[:, 0], pick[:, 1], pick[:, 2]] = 0.0
    g = sgm.Grid(w)
    _upload(g, w, o.to_packages(phi, -o.far, o.far))
    g.reinit(1)
    got = g.view("phi").cpu().numpy().astype(np.float64)
    exp = o.to_packages(o.reinit_step(phi), -o.far, o.far)
    assert_phi_close(w, got, exp, "phi = 0 step")
    cells = (pick[:, 2] // 4) + w.n[0] * ((pick[:, 1] // 4) + w.n[1] * (pick[:, 0] // 4))
    ids = t.bg[cells]
    ds = (pick[:, 2] % 4) + 4 * (pick[:, 1] % 4) + 16 * (pick[:, 0] % 4)
    assert np.all(got[ids, ds] == 0.0)


def test_table1_add_invalidates_derived_fields(sgm):
    """sg_table1 op 0 changes phi in place: grad / normal / K / G are stale
    afterwards (probing grad is a state error until sg_gradient runs again)."""
    w = W.config("C1")
    g = sgm.Grid(w)
    g.reinit(2).gradient(sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT)
    assert g.info["has_grad"] and g.info["has_kint"]
    g.table1(0, 0.5 * w.dx)
    info = g.info
    assert not info["has_grad"] and not info["has_normal"] and not info["has_kint"]
    pos = torch.tensor([[0.5, 0.5, 0.21]], dtype=torch.float64, device="cuda")
    with pytest.raises(sgm.SgError) as e:
        g.probe(pos, want_grad=True)
    assert e.value.status == sgm.SG_ERR_STATE
    phi, _ = g.probe(pos, want_grad=False)
    g.gradient(sgm.SG_GRAD)
    phi2, _ = g.probe(pos)
    assert torch.equal(phi, phi2)


def test_probe_chunk_queue_order_bitwise(sgm):
    """The probe's in-order chunk queue (used for long particle streams such
    as C5's) gives the static order's results bit for bit (C4 on C2, forced
    with SG_PROBE_QUEUE=1 in a fresh process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for q in ("0", "1"):
        import tempfile
        tmp = os.path.join(tempfile.mkdtemp(), f"probe_queue{q}.npz")
        code = ("import numpy as np, torch, workloads as W\n"
                "from paper_2512_11473_b200 import sg\n"
                "w = W.config('C2'); g = sg.Grid(w); g.reinit(3).gradient(sg.SG_GRAD)\n"
                "pos = W.particles(w, device='cuda')\n"
                "oob = torch.zeros(1, dtype=torch.int64, device='cuda')\n"
                "p, gr = g.probe(pos, oob=oob)\n"
                f"np.savez({tmp!r}, phi=p.cpu().numpy(), grad=gr.cpu().numpy(), oob=oob.cpu().numpy())\n")
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                           timeout=300, env=dict(os.environ, SG_PROBE_QUEUE=q))
        assert r.returncode == 0, r.stderr[-2000:]
        out[q] = np.load(tmp)
    for k in ("phi", "grad", "oob"):
        assert np.array_equal(out["0"][k], out["1"][k]), k


def test_repeated_build_with_size_hint(sgm, O):
    """A second build of the same (desc, geometry) sizes its arena and
    launches from the first build's counts (no mid-build host wait); its
    tables and initial phi must equal the first build's and the oracle's."""
    for name in ("C1", "C2"):
        w = W.config(name)
        t = O.Oracle(w).build_tables()
        a = sgm.Grid(w)
        b = sgm.Grid(w)  # hinted
        for g in (a, b):
            assert np.array_equal(u32(g.view("bg")), t.bg)
            assert np.array_equal(u32(g.view("nb")), t.nb)
            assert np.array_equal(u32(g.view("meta_cell")), t.meta_cell)
        assert a.info["n_core"] == b.info["n_core"] and a.info["n_pkg"] == b.info["n_pkg"]
        assert torch.equal(a.view("phi"), b.view("phi"))


@pytest.mark.parametrize("skew", ["-7", "5"])
def test_build_hint_mismatch_rebuilds(skew):
    """A size hint that is wrong (too small: the compaction's meta writes
    must stay inside the smaller arena; too large) is detected once the
    build's work is queued and the grid is rebuilt without it: tables equal
    the oracle's.  Fresh process with SG_BUILD_HINT_SKEW (the hint of every
    repeated build is off by that many packages)."""
    import os
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    code = (
        "import numpy as np, torch, workloads as W\n"
        "from oracle.oracle import Oracle\n"
        "from paper_2512_11473_b200 import sg\n"
        "for name in ('C1', 'C2'):\n"
        "    w = W.config(name); t = Oracle(w).build_tables()\n"
        "    for rep in range(3):\n"
        "        g = sg.Grid(w)\n"
        "        assert np.array_equal(g.view('bg').cpu().numpy().view(np.uint32), t.bg), (name, rep)\n"
        "        assert np.array_equal(g.view('nb').cpu().numpy().view(np.uint32), t.nb), (name, rep)\n"
        "        assert np.array_equal(g.view('meta_cell').cpu().numpy().view(np.uint32), t.meta_cell)\n"
        "        assert g.info['n_pkg'] == t.n_pkg\n"
        "torch.cuda.synchronize()\n"
        "print('ok')\n")
    env = dict(os.environ, SG_BUILD_HINT_SKEW=skew)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
