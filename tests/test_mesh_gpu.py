"""GPU parity of the triangle-mesh geometry (NEXT-4, reading R-24).

Tables (background, meta, neighbours) bit-exact against the oracle's
brute-force mesh SDF; initial phi bit-exact (fp64 evaluation in the same
operation order, rounded to the grid dtype).  The device evaluates distances
from per-cell triangle bins and floods the signs of the cells beyond the bin
radius; the oracle evaluates every cell exactly -- equal tables are the check
that both agree.
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


CASES = {
    "ico3-16-f64": W.mesh_workload("ico3", W.icosphere(3, rot=0.4), 16, "f64"),
    "ico3-24-f32": W.mesh_workload("ico3", W.icosphere(3, rot=0.4), 24, "f32"),
    "ico4-40-f32": W.mesh_workload("ico4", W.icosphere(4, (0.52, 0.47, 0.5), 0.33, rot=1.1), 40,
                                   "f32"),
    "box-20-f64": W.mesh_workload("boxm", W.box_mesh((0.5, 0.48, 0.52), (0.2, 0.15, 0.25)), 20,
                                  "f64"),
    "ico2-off-f64": W.mesh_workload("ico2", W.icosphere(2, (0.3, 0.6, 0.45), 0.2, rot=2.0), 16,
                                    "f64").with_(lower=(-0.05, 0.02, -0.01)),
}


@pytest.mark.parametrize("case", list(CASES))
def test_mesh_tables_and_phi_bit_exact(sgm, O, case):
    w = CASES[case]
    o = O.Oracle(w)
    t = o.build_tables()
    g = sgm.Grid(w)
    info = g.info
    assert info["n_pkg"] == t.n_pkg
    assert np.array_equal(u32(g.view("bg")), t.bg)
    assert np.array_equal(u32(g.view("meta_cell")), t.meta_cell)
    assert np.array_equal(u32(g.view("nb")), t.nb)
    exp = o.to_packages(o.phi_dense(), -o.far, o.far)
    got = g.view("phi").cpu().numpy()
    if got.dtype == np.float32:
        exp = exp.astype(np.float32)
    assert np.array_equal(got, exp)
    # the downstream path runs unchanged on a mesh grid
    g.reinit(2).gradient(sgm.SG_GRAD | sgm.SG_NORMAL | sgm.SG_KINT)
    phi, grad = g.probe(torch.rand(1000, 3, dtype=torch.float64 if w.dtype == "f64"
                                   else torch.float32, device="cuda"))
    assert torch.isfinite(phi).all() and torch.isfinite(grad).all()


def test_mesh_argument_errors(sgm):
    w = CASES["ico3-16-f64"]
    with pytest.raises(sgm.SgError):  # mesh + primitives
        sgm.Grid(w.with_(prims=(W.Prim(W.SPHERE, (0.5, 0.5, 0.5, 0.2)),)))
    bad = W.Mesh(w.mesh.verts, (0, 1, 10 ** 6) + w.mesh.tris[3:])
    with pytest.raises(sgm.SgError):  # index out of range
        sgm.Grid(w.with_(mesh=bad))
    with pytest.raises(sgm.SgError):  # slab grid
        sgm.Grid(w, slab=(0, 8, 2))
