"""z-slab partition on ONE GPU through the explicit-slab entry point: P slab
grids built with sg_build(slab) in one process from the library's plan
(sg_slab_plan), halos refreshed by device copies between their views over
the plan's halo ranges (the ranges the library's own exchange uses; the
partitioned grids with their in-library exchange are tests/test_comm_gpu.py).  The P-slab result must be BITWISE equal to
the 1-GPU grid (Jacobi sweeps are order independent): tables, phi after 20
sweeps, grad/normal/kernel integrals and probes."""
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


def _owner_mask(pos, w, p):
    """particles whose containing background plane rank p owns"""
    cz = torch.floor((pos[:, 2].double() - w.lower[2]) / w.cell)
    return (cz >= p.z_lo) & (cz < p.z_hi)


def _check_plan_ranges(p, g):
    """the plan's halo ranges are whole stored planes of the built grid"""
    pf = [int(v) for v in g.view("plane_first").cpu().numpy()]

    def rng(z):
        return (pf[z - p.zs_lo], pf[z - p.zs_lo + 1])
    none = (0, 0)
    assert p.n_pkg == g.info["n_pkg"] == pf[-1]
    assert (p.own_lo, p.own_hi) == (g.info["own_lo"], g.info["own_hi"])
    assert p.send_lo == (rng(p.z_lo) if p.rank > 0 else none)
    assert p.recv_lo == (rng(p.z_lo - 1) if p.rank > 0 else none)
    assert p.send_hi == (rng(p.z_hi - 1) if p.rank < p.world - 1 else none)
    assert p.recv_hi == (rng(p.z_hi) if p.rank < p.world - 1 else none)


def _exchange_local(grids, halos, name, per):
    P = len(grids)
    views = [g.view(name).reshape(-1) for g in grids]
    for r in range(P):
        h = halos[r]
        if r > 0:  # my ghost-below <- (r-1)'s last owned plane
            a, b = h.recv_lo
            c, d = halos[r - 1].send_hi
            assert b - a == d - c
            views[r][a * per:b * per].copy_(views[r - 1][c * per:d * per])
        if r < P - 1:
            a, b = h.recv_hi
            c, d = halos[r + 1].send_lo
            assert b - a == d - c
            views[r][a * per:b * per].copy_(views[r + 1][c * per:d * per])


@pytest.mark.parametrize("name,P", [("C1", 2), ("C1", 3), ("C2", 4), ("C2", 8)])
def test_slabs_bitwise_equal_one_gpu(sgm, name, P):
    from paper_2512_11473_b200 import slab
    w = W.config(name)
    full = sgm.Grid(w)
    desc, geom, keep = sgm.make_desc(w)
    nz = w.n[2]
    counts = torch.zeros(nz, dtype=torch.int64, device="cuda")
    sgm.sg_plane_counts(desc, geom, 0, nz, counts.data_ptr())
    counts = counts.cpu().numpy()
    pf_full = full.view("plane_first").cpu().numpy()
    assert np.array_equal(np.diff(pf_full), counts)
    plans = [slab.plan(counts, P, r) for r in range(P)]
    grids = [sgm.Grid(w, slab=(p.z_lo, p.z_hi, p.id_base)) for p in plans]
    for p, g in zip(plans, grids):
        _check_plan_ranges(p, g)
    halos = plans
    fnb = full.view("nb").cpu().numpy().view(np.uint32)
    fmeta = full.view("meta_cell").cpu().numpy().view(np.uint32)
    for p, g in zip(plans, grids):
        info = g.info
        gl = np.arange(2, info["n_pkg"]) - 2 + p.id_base
        assert np.array_equal(g.view("meta_cell").cpu().numpy().view(np.uint32)[2:], fmeta[gl])
        # neighbour rows of owned packages: local ids map to the global ones
        nb = g.view("nb").cpu().numpy().view(np.uint32).astype(np.int64)
        own = slice(info["own_lo"], info["own_hi"])
        loc = nb[own]
        glob = np.where(loc >= 2, loc - 2 + p.id_base, loc)
        assert np.array_equal(glob, fnb[info["own_lo"] - 2 + p.id_base:info["own_hi"] - 2 + p.id_base])
    iters = 20
    full.reinit(iters, w.cfl)
    for _ in range(iters):
        for g in grids:
            g.reinit(1, w.cfl)
        _exchange_local(grids, halos, "phi", 64)
    fields = sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT
    full.gradient(fields, w.h_ratio)
    for g in grids:
        g.gradient(fields, w.h_ratio)
    _exchange_local(grids, halos, "grad", 256)
    for name_ in ("phi", "grad", "normal", "kint", "gkint"):
        fv = full.view(name_)
        for p, g in zip(plans, grids):
            info = g.info
            a, b = info["own_lo"], info["own_hi"]
            ga, gb = a - 2 + p.id_base, b - 2 + p.id_base
            assert torch.equal(g.view(name_)[a:b], fv[ga:gb]), (name_, p.rank)
    # probes binned to their owner slab
    dt = np.float32 if w.dtype == "f32" else np.float64
    pos = torch.from_numpy(W.random_positions(w, 200000, seed=5, dtype=dt)).cuda()
    fphi, fgrad = full.probe(pos)
    got_phi = torch.full_like(fphi, float("nan"))
    got_grad = torch.full_like(fgrad, float("nan"))
    for p, g in zip(plans, grids):
        m = _owner_mask(pos, w, p)
        ph, gr = g.probe(pos[m].contiguous())
        got_phi[m] = ph
        got_grad[m] = gr
    assert torch.equal(got_phi, fphi) and torch.equal(got_grad, fgrad)


def _slab_setup(sgm, w, P):
    from paper_2512_11473_b200 import slab
    desc, geom, keep = sgm.make_desc(w)
    nz = w.n[2]
    counts = torch.zeros(nz, dtype=torch.int64, device="cuda")
    sgm.sg_plane_counts(desc, geom, 0, nz, counts.data_ptr())
    counts = counts.cpu().numpy()
    plans = [slab.plan(counts, P, r) for r in range(P)]
    grids = [sgm.Grid(w, slab=(p.z_lo, p.z_hi, p.id_base)) for p in plans]
    return plans, grids, plans


def _owned_equal(full, plans, grids, name):
    fv = full.view(name)
    ok = True
    for p, g in zip(plans, grids):
        info = g.info
        a, b = info["own_lo"], info["own_hi"]
        ok = ok and torch.equal(g.view(name)[a:b], fv[a - 2 + p.id_base:b - 2 + p.id_base])
    return ok


@pytest.mark.parametrize("name,P", [("C1", 2), ("C2", 4)])
def test_ghost_reuse_four_sweeps_per_exchange(sgm, name, P):
    """SURVEY 8(e) ghost reuse: sweeping owned + ghost packages (sg_reinit_halo)
    keeps the owned packages exact for up to 4 sweeps per exchange (ghost
    depth 4 points): bitwise equal to the 1-GPU grid."""
    w = W.config(name)
    iters = 20
    full = sgm.Grid(w)
    full.reinit(iters, w.cfl)
    for k, expect in ((4, True), (3, True)):
        plans, grids, halos = _slab_setup(sgm, w, P)
        done = 0
        while done < iters:
            m = min(k, iters - done)
            for g in grids:
                sgm.sg_reinit_halo(g.handle, m, w.cfl)
            _exchange_local(grids, halos, "phi", 64)
            done += m
        assert _owned_equal(full, plans, grids, "phi") == expect, (k, expect)
