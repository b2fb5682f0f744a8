"""Two-sweep reinitialisation tiles (sg_tsweep.cu) against the single sweep.

The tile path is opt-in (SG_TSWEEP=1; measured slower than the single-sweep
chain, profiles/README.md).  With it, sg_reinit(grid, iters) on an fp32
whole-domain grid runs iters // 2 launches
of the two-sweep tile kernel (plus one single sweep for odd iters); the
arithmetic per point is the single sweep's (sg_godunov.cuh), so the result
must equal iters calls of sg_reinit(grid, 1) -- which always run the single
sweep k_sweep -- BIT FOR BIT, on every grid shape the plan has to handle
(ragged tiles, halved chunks, bands touching the domain faces, anisotropic
and offset grids, grids too small for one full tile).  The oracle tolerance
tests of test_parity_gpu.py / test_window_gpu.py go through the same
sg_reinit(iters) calls and pin the values against the paper's definition.
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
    import os
    os.environ["SG_TSWEEP"] = "1"  # opt-in path (read by the library at every call)
    from paper_2512_11473_b200 import build
    build.build()
    from paper_2512_11473_b200 import sg
    return sg


@pytest.fixture(scope="module", autouse=True)
def _restore_env():
    yield
    import os
    os.environ.pop("SG_TSWEEP", None)


def _chain_vs_tiles(sgm, w, iters):
    a = sgm.Grid(w)
    b = sgm.Grid(w)
    n0 = sgm.sg_launch_count()
    a.reinit(iters)  # the first call also builds the tile plan
    launches = sgm.sg_launch_count() - n0
    for _ in range(iters):
        b.reinit(1)
    if iters >= 2:  # a second call reuses the plan: count the sweep launches only
        n0 = sgm.sg_launch_count()
        a.reinit(iters)
        launches = sgm.sg_launch_count() - n0
        for _ in range(iters):
            b.reinit(1)
    torch.cuda.synchronize()
    pa, pb = a.view("phi"), b.view("phi")
    assert pa.shape == pb.shape
    same = torch.equal(pa.view(torch.int32), pb.view(torch.int32))
    if not same:
        d = (pa.double() - pb.double()).abs()
        i = int(torch.argmax(d.reshape(-1)))
        pytest.fail(f"{w.name} iters={iters}: tiles differ from the sweep chain; max |d| "
                    f"{float(d.max()):.3e} at flat index {i} (package {i // 64})")
    return launches


@pytest.mark.parametrize("iters", [2, 3, 20])
def test_c2_bitwise(sgm, iters):
    w = W.config("C2")
    launches = _chain_vs_tiles(sgm, w, iters)
    assert launches == iters // 2 + iters % 2, "the two-sweep path did not run"


@pytest.mark.parametrize("seed,n", [(0, 8), (1, 13), (3, 24), (5, 20), (7, 31), (9, 40), (11, 64)])
def test_random_scenes_bitwise(sgm, seed, n):
    w = W.random_scene(seed, n, dtype="f32")
    _chain_vs_tiles(sgm, w, 6)


def test_c1_fp32_and_scaled_init_bitwise(sgm):
    for scale in (1.0, 2.0):
        w = W.config("C1").with_(dtype="f32", init_scale=scale)
        _chain_vs_tiles(sgm, w, 4)


def test_anisotropic_offset_grid_bitwise(sgm):
    w = W.Workload("aniso", (45, 19, 14), 0.05, lower=(-0.3, 0.1, -0.2), dtype="f32",
                   prims=(W.Prim(W.TORUS_Z, (0.25, 0.32, 0.15, 0.25, 0.08)),))
    _chain_vs_tiles(sgm, w, 5)


def test_thick_band_halved_tiles_bitwise(sgm):
    """A scene whose band fills whole blocks of cells (many chunks exceed a
    tile's slots and are halved): the fins workload at a coarse spacing."""
    w = W.fins(24, dtype="f32", thin=1.5, thick=6.0)
    _chain_vs_tiles(sgm, w, 4)


def test_c3_full_size_bitwise(sgm):
    w = W.config("C3")
    _chain_vs_tiles(sgm, w, 4)


def test_fp64_keeps_single_sweeps(sgm):
    w = W.config("C1")  # fp64: the tile kernel is fp32-only
    g = sgm.Grid(w)
    n0 = sgm.sg_launch_count()
    g.reinit(4)
    assert sgm.sg_launch_count() - n0 == 4


def test_plan_rebuilt_after_sign_correction(sgm):
    """sg_sign_correct rewrites the face table's singular references: the
    next reinit must use a fresh tile plan (compare with the sweep chain on a
    second grid that went through the same calls)."""
    w = W.leaky(W.config("C2"))
    grids = [sgm.Grid(w), sgm.Grid(w)]
    grids[0].reinit(2)  # builds the plan of grid 0 before the tables change
    for _ in range(2):
        grids[1].reinit(1)
    for g in grids:
        g.sign_correct()
    grids[0].reinit(6)
    for _ in range(6):
        grids[1].reinit(1)
    torch.cuda.synchronize()
    assert torch.equal(grids[0].view("phi").view(torch.int32), grids[1].view("phi").view(torch.int32))
