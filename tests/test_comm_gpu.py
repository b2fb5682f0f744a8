"""Partitioned grids on ONE GPU through the library's own multi-GPU data plane
(include/sg.h sg_build_ex + sg_comm_create_local): P ranks, one host thread
each, exchange through the in-process communicator with the NCCL
communicator's semantics.  Every step of the partitioned path runs in libsg:
the plane-count all-gather and the plan, the ghost exchange every 4 sweeps
overlapped with the interior sweep, the (phi, grad) ghost exchange after
sg_gradient, and the probe's K9 binning + all-to-all with results in the
caller's order.  The result must be BITWISE the 1-GPU grid's (SURVEY 8(c.5):
"any quantity, P GPUs vs 1 GPU: bitwise")."""
import threading

import numpy as np
import pytest

import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sgm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2512_11473_b200 import build
    build.build()
    from paper_2512_11473_b200 import sg
    return sg


def run_ranks(P, body):
    """body(rank, comm, stream) on P threads over one local comm group;
    returns the per-rank results (re-raises the first failure)."""
    from paper_2512_11473_b200 import sg
    comms = sg.Comm.local(P)
    out, err = [None] * P, []
    dev = torch.cuda.current_device()

    def run(r):
        try:
            torch.cuda.set_device(dev)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = body(r, comms[r], st)
            st.synchronize()
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "a rank is stuck in a collective"
    for c in comms:
        c.close()
    if err:
        raise err[0]
    return out


def shares(n, P):
    return [(n * r // P, n * (r + 1) // P) for r in range(P)]


@pytest.mark.parametrize("name,P,iters", [("C1", 2, 20), ("C1", 3, 7), ("C2", 4, 20),
                                          ("C2", 8, 20), ("C2", 2, 1)])
def test_partitioned_bitwise_equal_one_gpu(sgm, name, P, iters):
    w = W.config(name)
    fields = sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT
    dt = np.float32 if w.dtype == "f32" else np.float64
    pos_np = W.random_positions(w, 300000, seed=9, dtype=dt)
    # a few outside the domain and NaN: they stay with the caller's rank
    pos_np[:7] = np.array([[-0.1, 0.5, 0.5], [0.5, 1.2, 0.5], [np.nan, 0.5, 0.5],
                           [0.5, 0.5, -0.01], [0.5, 0.5, 1.0], [2.0, 2.0, 2.0], [0.3, 0.3, 1.5]])
    full = sgm.Grid(w)
    full.reinit(iters, w.cfl).gradient(fields, w.h_ratio)
    pos = torch.from_numpy(pos_np).cuda()
    foob = torch.zeros(1, dtype=torch.int64, device="cuda")
    fphi, fgrad = full.probe(pos, oob=foob)
    sh = shares(pos_np.shape[0], P)

    def body(r, comm, st):
        g = sgm.Grid(w, comm=comm, stream=st)
        info0 = g.info
        g.reinit(iters, w.cfl, stream=st)
        g.gradient(fields, w.h_ratio, stream=st)
        a, b = sh[r]
        mine = pos[a:b].contiguous()
        oob = torch.zeros(1, dtype=torch.int64, device="cuda")
        phi, grad = g.probe(mine, oob=oob, stream=st)
        st.synchronize()
        res = {"info": info0, "phi": phi.clone(), "grad": grad.clone(), "oob": int(oob.item())}
        lo, hi = info0["own_lo"], info0["own_hi"]
        for f in ("phi", "grad", "normal", "kint", "gkint", "nb", "meta_cell"):
            res[f + "_own"] = g.view(f)[lo:hi].clone()
        # ghost planes of phi and (phi, grad) hold the neighbours' values
        res["phi_all"] = g.view("phi").clone()
        res["grad_all"] = g.view("grad").clone()
        g.close()
        return res

    out = run_ranks(P, body)
    # the owned id ranges tile the global range; tables map to global ids
    spans = []
    for r, res in enumerate(out):
        info = res["info"]
        assert info["rank"] == r and info["nranks"] == P
        base = info["id_base"]
        ga, gb = info["own_lo"] - 2 + base, info["own_hi"] - 2 + base
        spans.append((ga, gb))
        for f in ("phi", "grad", "normal", "kint", "gkint"):
            assert torch.equal(res[f + "_own"], full.view(f)[ga:gb]), (f, r)
        assert torch.equal(res["meta_cell_own"], full.view("meta_cell")[ga:gb])
        nb = res["nb_own"].cpu().numpy().view(np.uint32).astype(np.int64)
        glob = np.where(nb >= 2, nb - 2 + base, nb)
        assert np.array_equal(glob, full.view("nb")[ga:gb].cpu().numpy().view(np.uint32))
        # every stored package (owned + ghost) equals the global one
        n_loc = info["n_pkg"]
        g_ids = torch.arange(2, n_loc, device="cuda") - 2 + base
        assert torch.equal(res["phi_all"][2:], full.view("phi")[g_ids])
        assert torch.equal(res["grad_all"][2:], full.view("grad")[g_ids])
    assert spans[0][0] == 2 and spans[-1][1] == full.info["n_pkg"]
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    # probes: results in the caller's order, bitwise; OOB counted once
    got_phi = torch.cat([res["phi"] for res in out])
    got_grad = torch.cat([res["grad"] for res in out])
    assert torch.equal(got_phi, fphi) and torch.equal(got_grad, fgrad)
    assert sum(res["oob"] for res in out) == int(foob.item()) == 7


def test_partitioned_probe_uneven_shares(sgm):
    """Ranks with no particles at all, one rank holding everything, host
    buffers: the collective probe still returns every result in order."""
    w = W.config("C2")
    P = 3
    full = sgm.Grid(w)
    full.reinit(4, w.cfl).gradient(sgm.SG_GRAD, w.h_ratio)
    pos_np = W.lattice_particles(w, seed=0)[::7].copy()
    pos = torch.from_numpy(pos_np).cuda()
    fphi, fgrad = full.probe(pos)
    n = pos_np.shape[0]
    cuts = [(0, 0), (0, n), (n, n)]  # rank 1 holds all

    def body(r, comm, st):
        g = sgm.Grid(w, comm=comm, stream=st)
        g.reinit(4, w.cfl, stream=st).gradient(sgm.SG_GRAD, w.h_ratio, stream=st)
        a, b = cuts[r]
        d = g.probe(pos[a:b].contiguous(), stream=st)
        h = g.probe(pos[a:b].cpu().contiguous(), stream=st)  # host path
        st.synchronize()
        g.close()
        return d, h

    out = run_ranks(P, body)
    phi = torch.cat([o[0][0] for o in out])
    grad = torch.cat([o[0][1] for o in out])
    assert torch.equal(phi, fphi) and torch.equal(grad, fgrad)
    hphi = torch.cat([o[1][0] for o in out])
    assert torch.equal(hphi, fphi.cpu())


def test_partitioned_single_rank_and_allocator(sgm):
    """P = 1 partition = the plain grid; a grid on PyTorch's caching allocator
    (sg_allocator) holds its memory there and gives the same bits."""
    w = W.config("C2")
    full = sgm.Grid(w).reinit(20, w.cfl).gradient(sgm.SG_GRAD | sgm.SG_KINT, w.h_ratio)

    def body(r, comm, st):
        g = sgm.Grid(w, comm=comm, stream=st).reinit(20, w.cfl, stream=st)
        g.gradient(sgm.SG_GRAD | sgm.SG_KINT, w.h_ratio, stream=st)
        st.synchronize()
        res = (g.view("phi").clone(), g.view("grad").clone(), g.view("kint").clone())
        g.close()
        return res

    (phi, grad, K), = run_ranks(1, body)
    assert torch.equal(phi, full.view("phi")) and torch.equal(grad, full.view("grad"))
    assert torch.equal(K, full.view("kint"))
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    alloc = sgm.TorchAllocator()
    g = sgm.Grid(w, allocator=alloc).reinit(20, w.cfl).gradient(sgm.SG_GRAD | sgm.SG_KINT,
                                                                w.h_ratio)
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - before
    assert held >= g.info["device_bytes"] > 0
    assert torch.equal(g.view("phi"), full.view("phi"))
    assert torch.equal(g.view("kint"), full.view("kint"))
    g.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == before


def test_nccl_communicator_one_rank(sgm):
    """The NCCL backend (dlopen of the libnccl.so.2 PyTorch loaded): a
    one-rank communicator builds and runs a grid like the plain one."""
    import ctypes as C
    uid = sgm.Comm.unique_id()
    assert len(uid) == sgm.SG_COMM_ID_BYTES
    out = C.c_void_p()
    buf = (C.c_char * sgm.SG_COMM_ID_BYTES).from_buffer_copy(uid)
    sgm._check(sgm.lib().sg_comm_create(buf, 0, 1, C.byref(out)))
    comm = sgm.Comm(out.value)
    assert (comm.rank, comm.nranks, comm.kind) == (0, 1, sgm.SG_COMM_NCCL)
    comm.check()  # no asynchronous NCCL error
    w = W.config("C1")
    g = sgm.Grid(w, comm=comm).reinit(5, w.cfl)
    ref = sgm.Grid(w).reinit(5, w.cfl)
    assert torch.equal(g.view("phi"), ref.view("phi"))
    g.close()
    comm.close()


@pytest.mark.parametrize("seed,n,P,iters", [(1, 24, 2, 6), (3, 20, 3, 9), (5, 31, 5, 4), (7, 17, 4, 13),
                                            (9, 40, 3, 20)])
def test_partitioned_random_scenes(sgm, seed, n, P, iters):
    """Random unions (some bands touching the domain boundary, fp32 / fp64),
    P ranks with uneven particle shares and out-of-domain positions: every
    owned field and every probe result equals the 1-GPU grid's bits."""
    w = W.random_scene(seed, n, dtype="f64" if seed % 4 == 1 else "f32")
    fields = sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT
    dt = np.float32 if w.dtype == "f32" else np.float64
    pos_np = W.random_positions(w, 50000, seed=seed, dtype=dt)
    pos_np[::997] = -1.0  # out of the domain
    full = sgm.Grid(w)
    full.reinit(iters, w.cfl).gradient(fields, w.h_ratio)
    pos = torch.from_numpy(pos_np).cuda()
    fphi, fgrad = full.probe(pos)
    rng = np.random.default_rng(seed)
    cuts = np.sort(rng.integers(0, pos_np.shape[0], P - 1))
    sh = list(zip([0, *cuts], [*cuts, pos_np.shape[0]]))

    def body(r, comm, st):
        g = sgm.Grid(w, comm=comm, stream=st)
        g.reinit(iters, w.cfl, stream=st).gradient(fields, w.h_ratio, stream=st)
        a, b = sh[r]
        phi, grad = g.probe(pos[a:b].contiguous(), stream=st)
        st.synchronize()
        info = g.info
        lo, hi = info["own_lo"], info["own_hi"]
        own = {f: g.view(f)[lo:hi].clone() for f in ("phi", "grad", "normal", "kint", "gkint")}
        g.close()
        return info, own, phi.clone(), grad.clone()

    out = run_ranks(P, body)
    for info, own, _, _ in out:
        ga, gb = info["own_lo"] - 2 + info["id_base"], info["own_hi"] - 2 + info["id_base"]
        for f, v in own.items():
            assert torch.equal(v, full.view(f)[ga:gb]), f
    assert torch.equal(torch.cat([o[2] for o in out]), fphi)
    assert torch.equal(torch.cat([o[3] for o in out]), fgrad)
