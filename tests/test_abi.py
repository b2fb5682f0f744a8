"""C-ABI checks that need no GPU: the library loads, exports every function
include/sg.h declares, the ctypes mirrors match the C struct layouts, and the
host-only partition helper behaves (no device compute calls here)."""
import ctypes as C
import itertools
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sg.h")


@pytest.fixture(scope="module")
def sg():
    from paper_2512_11473_b200 import build, sg as S
    build.build()
    return S


def _declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:sg_status|void|const char\*|int32_t|uint64_t)\s+(sg_\w+)\s*\(",
                                 txt, flags=re.M)))


def test_exports_every_declared_symbol(sg):
    names = _declared_functions()
    assert len(names) >= 14
    L = C.CDLL(sg.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(sg.EXPORTS)
    # exported dynamic symbols of the .so (nm -D)
    out = subprocess.run(["nm", "-D", "--defined-only", sg.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_abi_version(sg):
    assert sg.sg_abi_version() == 3
    assert sg.sg_launch_count() == 0


def test_ctypes_layout_matches_header(sg, tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "sg.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(sg_prim),sizeof(sg_geometry),sizeof(sg_desc),sizeof(sg_slab),sizeof(sg_view_t),'
                   'sizeof(sg_info_t),offsetof(sg_info_t,own_hi),offsetof(sg_desc,init_scale),'
                   'sizeof(sg_plan_t),offsetof(sg_plan_t,recv_hi),sizeof(sg_build_opts),sizeof(sg_allocator),'
                   'offsetof(sg_info_t,nranks));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I" + os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    exp = [C.sizeof(sg.sg_prim), C.sizeof(sg.sg_geometry), C.sizeof(sg.sg_desc), C.sizeof(sg.sg_slab),
           C.sizeof(sg.sg_view_t), C.sizeof(sg.sg_info_t), sg.sg_info_t.own_hi.offset,
           sg.sg_desc.init_scale.offset, C.sizeof(sg.sg_plan_t), sg.sg_plan_t.recv_hi.offset,
           C.sizeof(sg.sg_build_opts), C.sizeof(sg.sg_allocator), sg.sg_info_t.nranks.offset]
    assert got == exp


def test_balanced_cuts_host_logic(sg):
    counts = np.array([0, 0, 5, 10, 10, 10, 5, 0, 0, 0])
    cuts = sg.sg_balanced_cuts(counts, 2)
    assert cuts[0] == 0 and cuts[-1] == 10
    pre = np.concatenate([[0], np.cumsum(counts)])
    # cut = smallest z with prefix(z) >= total/2
    assert cuts[1] == int(np.argmax(pre * 2 >= pre[-1]))
    for r in (1, 3, 4, 8, 10):
        c = sg.sg_balanced_cuts(counts, r)
        assert len(c) == r + 1 and all(b > a for a, b in zip(c, c[1:]))
    with pytest.raises(sg.SgError):
        sg.sg_balanced_cuts(counts, 11)
    with pytest.raises(sg.SgError):
        sg.sg_balanced_cuts(counts, 0)
    # balance quality on the C3 plane profile of the oracle
    from oracle.oracle import Oracle
    import workloads as W
    t = Oracle(W.config("C2")).build_tables()
    c = sg.sg_balanced_cuts(t.plane_count, 8)
    loads = [int(t.plane_count[a:b].sum()) for a, b in zip(c, c[1:])]
    # whole-plane granularity: no slab exceeds the mean by more than one plane
    assert max(loads) <= sum(loads) / 8 + int(t.plane_count.max())


def test_no_torch_types_in_header():
    txt = open(HEADER).read()
    assert "torch" not in re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    assert 'extern "C"' in txt


def test_neighbour_index_shift_lst2(sg):
    """Lst. 2 through the library's own host export (the kernels
    inline the same function): SPEC's printed 2-D examples (S:172-175,
    tests/golden/shift_examples.json, extended by a zero z shift -> offset 1,
    data 0) and, for every shift in [-4, 7]^3, the generalShift definition
    (S:177-180): target cell = floor(shift / 4) relative to the centre,
    data = shift mod 4, slot = (cx+1) + 3 (cy+1) + 9 (cz+1)."""
    from conftest import golden
    g = golden("shift_examples.json")
    assert g["pkg"] == 4
    for case in g["cases"]:
        slot, off, dat = sg.sg_neighbour_index_shift(case["shift"] + [0])
        assert list(off) == case["offset"] + [1] and list(dat) == case["data"] + [0]
        assert slot == off[0] + 3 * off[1] + 9 * off[2]
    for s in itertools.product(range(-4, 8), repeat=3):
        slot, off, dat = sg.sg_neighbour_index_shift(s)
        cell = [v // 4 for v in s]   # Python floor division
        assert list(off) == [c + 1 for c in cell], s
        assert list(dat) == [v % 4 for v in s], s
        assert slot == (cell[0] + 1) + 3 * (cell[1] + 1) + 9 * (cell[2] + 1)
    for bad in ([-5, 0, 0], [0, 8, 0], [0, 0, 100]):
        assert sg.sg_neighbour_index_shift(bad)[0] == -1


def test_slab_plan_host_logic(sg):
    """sg_slab_plan (host only): cuts as sg_balanced_cuts, stored planes one
    ghost plane per side, contiguous global id ranges that tile the domain,
    halo ranges = whole stored planes, the send range of rank r the size of
    the matching receive range of its neighbour."""
    from oracle.oracle import Oracle
    import workloads as W
    for name in ("C1", "C2"):
        t = Oracle(W.config(name)).build_tables()
        pc = t.plane_count
        nz = pc.size
        for world in (1, 2, 3, 5, 8):
            plans = [sg.sg_slab_plan(pc, world, r) for r in range(world)]
            assert all(c == sg.sg_balanced_cuts(pc, world) for _, c in plans)
            owned = []
            for r, (p, cuts) in enumerate(plans):
                assert (p["z_lo"], p["z_hi"]) == (cuts[r], cuts[r + 1])
                assert p["zs_lo"] == max(0, p["z_lo"] - 1) and p["zs_hi"] == min(nz, p["z_hi"] + 1)
                assert p["id_base"] == 2 + int(pc[:p["zs_lo"]].sum())
                assert p["n_pkg"] == 2 + int(pc[p["zs_lo"]:p["zs_hi"]].sum())
                g = lambda l: l - 2 + p["id_base"]  # noqa: E731
                owned.append((g(p["own_lo"]), g(p["own_hi"])))
                first = lambda z: 2 + int(pc[p["zs_lo"]:z].sum())  # noqa: E731
                if r > 0:
                    assert p["send_lo"] == (first(p["z_lo"]), first(p["z_lo"] + 1))
                    assert p["recv_lo"] == (2, first(p["z_lo"]))
                    q = plans[r - 1][0]
                    assert p["recv_lo"][1] - p["recv_lo"][0] == q["send_hi"][1] - q["send_hi"][0]
                    # the same global packages
                    assert g(p["recv_lo"][0]) == q["send_hi"][0] - 2 + q["id_base"]
                else:
                    assert p["send_lo"] == (0, 0) and p["recv_lo"] == (0, 0)
                if r == world - 1:
                    assert p["send_hi"] == (0, 0) and p["recv_hi"] == (0, 0)
                else:
                    assert p["recv_hi"] == (p["own_hi"], p["n_pkg"])
            assert owned[0][0] == 2 and owned[-1][1] == t.n_pkg
            assert all(a[1] == b[0] for a, b in zip(owned, owned[1:]))
    with pytest.raises(sg.SgError):
        sg.sg_slab_plan([1, 2, 3], 4, 0)
    with pytest.raises(sg.SgError):
        sg.sg_slab_plan([1, 2, 3], 2, 2)
