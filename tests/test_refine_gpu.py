"""GPU checks of the multi-resolution layer build (NEXT-4, P:473-489,
P:499-504; include/sg.h sg_build_refined).

A layer refined from its parent must equal the direct build at the finer
resolution bit for bit (tables, tagging bitmasks, initial phi): a fine core
cell always lies under a core parent, and a non-core parent cell has one sign
over its whole cell.  The direct builds are themselves oracle-checked
(test_parity_gpu, test_mesh_gpu); the refined mesh layer is also compared
with the oracle directly.
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


def u8(t):
    return t.cpu().numpy().view(np.uint8)


def state(g):
    return {k: u8(g.view(k)) for k in ("bg", "meta_cell", "meta_cat", "nb", "phi", "cell_core",
                                        "cell_neg")}


def assert_same(a, b):
    for k in a:
        assert a[k].shape == b[k].shape and np.array_equal(a[k], b[k]), k


def fine(w, levels):
    f = 2 ** levels
    return w.with_(n=tuple(f * k for k in w.n), cell=w.cell / f)


CHAINS = {
    "C1-f64": (W.config("C1"), 1),
    "prism-32-to-128": (W.config("C2").with_(n=(32, 32, 32), cell=1 / 32), 2),
    "torusbox-64-to-128": (W.config("C3").with_(n=(64, 64, 64), cell=1 / 64), 1),
    "random-scene": (W.random_scene(3, 12, dtype="f32"), 2),
    "ico4-mesh": (W.mesh_workload("ico4", W.icosphere(4, rot=0.4), 16, "f32"), 2),
    "box-mesh": (W.mesh_workload("boxm", W.box_mesh((0.5, 0.48, 0.52), (0.2, 0.15, 0.25)), 12,
                                 "f64"), 2),
}


@pytest.mark.parametrize("case", list(CHAINS))
def test_refined_layer_equals_direct_build(sgm, case):
    w, levels = CHAINS[case]
    g = sgm.Grid(w)
    for lv in range(1, levels + 1):
        g = g.refined()
        assert_same(state(g), state(sgm.Grid(fine(w, lv))))


def test_refined_mesh_layer_matches_oracle(sgm):
    from oracle import oracle as O
    O.build()
    w = W.mesh_workload("ico3", W.icosphere(3, rot=0.4), 16, "f64")
    g = sgm.Grid(w).refined()
    o = O.Oracle(fine(w, 1))
    t = o.build_tables()
    assert np.array_equal(g.view("bg").cpu().numpy().view(np.uint32), t.bg)
    assert np.array_equal(g.view("nb").cpu().numpy().view(np.uint32), t.nb)
    exp = o.to_packages(o.phi_dense(), -o.far, o.far)
    assert np.array_equal(g.view("phi").cpu().numpy(), exp)


def test_refined_rejects_slab_parent(sgm):
    g = sgm.Grid(W.config("C1"), slab=(0, 8, 2))
    with pytest.raises(sgm.SgError):
        g.refined()
