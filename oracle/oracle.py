"""ctypes front-end of the CPU oracle (oracle/sg_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may use it; the product package
(paper_2512_11473_b200/) never imports it.  Arrays are numpy; the oracle is
fp64 on a dense fine grid (M = 4N points per axis), tables follow SURVEY.md
8(c.1) O3-O5, fields O6-O10.  Every function cites the paper passage it
follows in sg_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sg_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

# -O3 -march=native (the oracle timed as a CPU
# program); -ffp-contract=off and no -ffast-math keep every double operation
# a separately rounded IEEE operation in the order written, so the results do
# not depend on the flags or the host.  The library is built per host CPU
# (native code of one box may not run on another).
CFLAGS = ["-O3", "-march=native", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
          "-shared", "-std=c11", "-Wall", "-Wno-unknown-pragmas"]


def _cpu_tag() -> str:
    import hashlib
    import platform
    sig = platform.machine()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith(("model name", "flags")):
                    sig += line
                if line.strip() == "":
                    break
    except OSError:
        pass
    return hashlib.sha1(sig.encode()).hexdigest()[:10]


LIB = os.path.join(HERE, f"liboracle.{_cpu_tag()}.so")


def build(force: bool = False) -> str:
    """Compile the oracle library for this host (gcc, no FMA contraction,
    IEEE double)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Prim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("p", C.c_double * 12)]


class _Grid(C.Structure):
    _fields_ = [("lower", C.c_double * 3), ("cell", C.c_double), ("n", C.c_int32 * 3),
                ("pad", C.c_int32), ("far", C.c_double), ("init_scale", C.c_double),
                ("win_lo", C.c_int32 * 3), ("win_n", C.c_int32 * 3)]


_lib = None
_active_mesh = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        L.or_sdf.restype = C.c_double
        L.or_sdf.argtypes = [P, C.c_int32, P]
        L.or_sdf_batch.argtypes = [P, C.c_int32, C.c_int64, P, P]
        L.or_far.restype = C.c_double
        L.or_far.argtypes = [P]
        L.or_tag.argtypes = [P, P, C.c_int32, P, P]
        L.or_compact.restype = C.c_int64
        L.or_compact.argtypes = [P, P, P, P, P, P]
        L.or_neighbours.argtypes = [P, P, C.c_int32, P, P, C.c_int64, P]
        L.or_phi_dense.argtypes = [P, P, C.c_int32, P, P]
        L.or_phi_point.restype = C.c_double
        L.or_phi_point.argtypes = [P, P, C.c_int32, P, C.c_int64, C.c_int64, C.c_int64]
        L.or_reinit_dense.argtypes = [P, P, C.c_int32, P, P, P, C.c_double]
        L.or_reinit_point_from_init.restype = C.c_double
        L.or_reinit_point_from_init.argtypes = [P, P, C.c_int32, P, C.c_int64, C.c_int64,
                                                C.c_int64, C.c_double]
        L.or_gradient_dense.argtypes = [P, P, C.c_int32, P, P, P, P]
        L.or_kernel_taps.restype = C.c_int32
        L.or_kernel_taps.argtypes = [C.c_double, C.c_double, P, P, P]
        L.or_heaviside.restype = C.c_double
        L.or_heaviside.argtypes = [C.c_double, C.c_double]
        L.or_kernel_dense.argtypes = [P, P, C.c_int32, P, P, C.c_double, P, P]
        L.or_probe.restype = C.c_int64
        L.or_probe.argtypes = [P, P, C.c_int32, P, P, P, C.c_int64, P, P, P]
        L.or_gather_packages.argtypes = [P, P, P, C.c_int64, C.c_double, C.c_double, P]
        L.or_table1_dense.argtypes = [P, P, C.c_int32, P, P, C.c_int32, C.c_double, P]
        L.or_relax.argtypes = [P, P, C.c_int32, P, P, P, P, C.c_int64, P, C.c_double,
                               C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32]
        L.or_sign_correct.argtypes = [P, P, C.c_int32, P, P, P, C.c_int64, P, P, P,
                                      C.c_double, C.c_int32, P]
        L.or_clean.restype = C.c_int32
        L.or_clean.argtypes = [P, P, C.c_int32, P, P, C.c_double, C.c_double, C.c_int32,
                               C.c_double, C.c_int32, P]
        L.or_mesh_set.argtypes = [P, P, C.c_int32, C.c_int32]
        L.or_mesh_sdf.restype = C.c_double
        L.or_mesh_sdf.argtypes = [P]
        L.or_set_threads.argtypes = [C.c_int32]
        L.or_get_threads.restype = C.c_int32
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def get_threads() -> int:
    return int(lib().or_get_threads())


@dataclass
class Tables:
    cat: np.ndarray        # u8[Nz,Ny,Nx] flattened: 0/1 inactive by sign, 2 inner, 3 core
    bg: np.ndarray         # u32[N^3]
    meta_cell: np.ndarray  # u32[n_pkg]
    meta_cat: np.ndarray   # u8[n_pkg]
    nb: np.ndarray         # u32[n_pkg, 27]
    plane_count: np.ndarray  # i64[Nz]
    n_pkg: int
    near_ties: int


class Oracle:
    """Dense fp64 oracle bound to one workload (geometry + grid).

    window: None (dense arrays over the whole domain) or a box of background
    cells ((x0, y0, z0), (x1, y1, z1)), half open: the dense arrays of O6-O10
    then cover only its fine points (shape (4(z1-z0), 4(y1-y0), 4(x1-x0)));
    values read outside the box but inside the domain are the initial phi
    (sg_oracle.c or_grid), exact at depth > (sweeps + stencil radius) from
    the box faces.  Tables (O3-O5) always cover the whole domain."""

    def __init__(self, w, window=None):
        self.w = w
        self._g = _Grid()
        self.window = None
        if window is not None:
            lo, hi = (tuple(int(v) for v in window[0]), tuple(int(v) for v in window[1]))
            assert all(0 <= lo[k] < hi[k] <= w.n[k] for k in range(3)), window
            self.window = (lo, hi)
            for k in range(3):
                self._g.win_lo[k] = 4 * lo[k]
                self._g.win_n[k] = 4 * (hi[k] - lo[k])
        for k in range(3):
            self._g.lower[k] = w.lower[k]
            self._g.n[k] = w.n[k]
        self._g.cell = w.cell
        self._g.far = w.far
        self._g.init_scale = w.init_scale
        self._prims = (_Prim * max(1, len(w.prims)))()
        for i, pr in enumerate(w.prims):
            self._prims[i].kind = pr.kind
            for j, v in enumerate(pr.p):
                self._prims[i].p[j] = v
        self.n_prims = len(w.prims)
        self.tables: Tables | None = None
        mesh = getattr(w, "mesh", None)
        self._mesh = None
        if mesh is not None:
            self._mesh = (np.ascontiguousarray(np.asarray(mesh.verts, np.float64)),
                          np.ascontiguousarray(np.asarray(mesh.tris, np.int32)))

    def _L(self):
        """The oracle library with this workload's mesh registered (one mesh
        at a time; a geometry without primitives evaluates the mesh)."""
        global _active_mesh
        L = lib()
        if self._mesh is not None and _active_mesh is not self._mesh:
            v, t = self._mesh
            L.or_mesh_set(_ptr(v), _ptr(t), v.size // 3, t.size // 3)
            _active_mesh = self._mesh
        return L

    # handles
    @property
    def g(self):
        return C.byref(self._g)

    @property
    def prims(self):
        return C.cast(self._prims, C.c_void_p)

    @property
    def far(self) -> float:
        return float(self._L().or_far(self.g))

    @property
    def dx(self) -> float:
        return self.w.cell / 4.0

    @property
    def m(self):
        """Dense array extents (Mx, My, Mz): the domain, or the window box."""
        if self.window is not None:
            lo, hi = self.window
            return tuple(4 * (hi[k] - lo[k]) for k in range(3))
        return tuple(4 * n for n in self.w.n)

    def _whole(self, what):
        assert self.window is None, f"{what}: whole-domain oracle only"

    # O1
    def sdf(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1, 3))
        out = np.empty(x.shape[0])
        self._L().or_sdf_batch(self.prims, self.n_prims, x.shape[0], _ptr(x), _ptr(out))
        return out

    # O3-O5
    def build_tables(self) -> Tables:
        nx, ny, nz = self.w.n
        ncell = nx * ny * nz
        cat = np.empty(ncell, np.uint8)
        ties = C.c_int64(0)
        self._L().or_tag(self.g, self.prims, self.n_prims, _ptr(cat), C.byref(ties))
        bg = np.empty(ncell, np.uint32)
        n_active = int(np.count_nonzero(cat >= 2))
        meta_cell = np.empty(n_active + 2, np.uint32)
        meta_cat = np.empty(n_active + 2, np.uint8)
        plane = np.zeros(nz, np.int64)
        n_pkg = int(self._L().or_compact(self.g, _ptr(cat), _ptr(bg), _ptr(meta_cell),
                                     _ptr(meta_cat), _ptr(plane)))
        assert n_pkg == n_active + 2
        nb = np.empty((n_pkg, 27), np.uint32)
        self._L().or_neighbours(self.g, self.prims, self.n_prims, _ptr(bg), _ptr(meta_cell),
                            n_pkg, _ptr(nb))
        self.tables = Tables(cat, bg, meta_cell, meta_cat, nb, plane, n_pkg, int(ties.value))
        return self.tables

    def _bg(self):
        if self.tables is None:
            self.build_tables()
        return self.tables.bg

    # O6
    def phi_dense(self) -> np.ndarray:
        """Dense initial phi, shape (Mz, My, Mx) (x fastest)."""
        mx, my, mz = self.m
        phi = np.empty((mz, my, mx))
        self._L().or_phi_dense(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(phi))
        return phi

    def phi_point(self, ix: int, iy: int, iz: int) -> float:
        return float(self._L().or_phi_point(self.g, self.prims, self.n_prims, _ptr(self._bg()),
                                        ix, iy, iz))

    # O7
    def reinit_step(self, phi: np.ndarray, cfl: float | None = None) -> np.ndarray:
        cfl = self.w.cfl if cfl is None else cfl
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        out = np.empty_like(phi)
        self._L().or_reinit_dense(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(phi),
                              _ptr(out), cfl)
        return out

    def reinit(self, phi: np.ndarray, iters: int, cfl: float | None = None) -> np.ndarray:
        for _ in range(iters):
            phi = self.reinit_step(phi, cfl)
        return phi

    def reinit_point_from_init(self, ix: int, iy: int, iz: int, cfl: float | None = None) -> float:
        cfl = self.w.cfl if cfl is None else cfl
        return float(self._L().or_reinit_point_from_init(self.g, self.prims, self.n_prims,
                                                     _ptr(self._bg()), ix, iy, iz, cfl))

    # O8
    def gradient(self, phi: np.ndarray):
        """Returns (grad, normal), each shape (3, Mz, My, Mx)."""
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        grad = np.empty((3,) + phi.shape)
        normal = np.empty((3,) + phi.shape)
        self._L().or_gradient_dense(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(phi),
                                _ptr(grad), _ptr(normal))
        return grad, normal

    # O9
    def taps(self, h_ratio: float | None = None):
        h_ratio = self.w.h_ratio if h_ratio is None else h_ratio
        return kernel_taps(h_ratio, self.dx)

    def kernel_integrals(self, phi: np.ndarray, h_ratio: float | None = None):
        """Returns (K shape (Mz,My,Mx), G shape (3,Mz,My,Mx))."""
        h_ratio = self.w.h_ratio if h_ratio is None else h_ratio
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        K = np.empty_like(phi)
        G = np.empty((3,) + phi.shape)
        self._L().or_kernel_dense(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(phi),
                              h_ratio, _ptr(K), _ptr(G))
        return K, G

    # O10
    def probe(self, phi: np.ndarray, grad: np.ndarray | None, pos: np.ndarray):
        """pos (n,3) any float dtype (promoted to double). Returns (phi, grad, oob)."""
        pos = np.ascontiguousarray(np.asarray(pos).astype(np.float64).reshape(-1, 3))
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        g3 = None if grad is None else np.ascontiguousarray(grad, dtype=np.float64)
        n = pos.shape[0]
        out_phi = np.empty(n)
        out_grad = np.empty((n, 3))
        oob = self._L().or_probe(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(phi),
                             _ptr(g3), n, _ptr(pos), _ptr(out_phi), _ptr(out_grad))
        return out_phi, out_grad, int(oob)

    # Table 1 workloads: op 0 sequential (phi + value), op 1 stencil
    def table1(self, phi: np.ndarray, op: int, value: float = 0.0) -> np.ndarray:
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        out = np.empty_like(phi)
        self._L().or_table1_dense(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(phi),
                              int(op), float(value), _ptr(out))
        return out

    # NEXT-2 particle relaxation (reading R-21); pos (n, 3) float64, updated copy
    def relax(self, phi, grad, G, pos, dp, h_ratio=1.3, step=0.1, max_disp=0.2,
              surface_offset=0.5, steps=1):
        self._whole("relax")
        pos = np.ascontiguousarray(np.asarray(pos, dtype=np.float64).reshape(-1, 3)).copy()
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        grad = np.ascontiguousarray(grad, dtype=np.float64)
        G = np.ascontiguousarray(G, dtype=np.float64)
        self._L().or_relax(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(phi), _ptr(grad),
                       _ptr(G), pos.shape[0], _ptr(pos), dp, h_ratio, step, max_disp,
                       surface_offset, int(steps))
        return pos

    # layout helper: dense plane -> package-major using the oracle's meta
    def sign_correct(self, phi: np.ndarray, tau: float | None = None, max_sweeps: int = 0):
        """NEXT-3 sign-consistency correction (R-22) on copies of this oracle's
        tables and of the dense phi.  Returns (bg, nb, cell_neg u8[ncell],
        phi, (coarse_sweeps, refined_sweeps)).  For an fp32 comparison pass
        phi and tau already rounded to float32 (the trust decision is then
        taken in the kernel's precision)."""
        self._whole("sign_correct")
        t = self.tables if self.tables is not None else self.build_tables()
        bg = t.bg.copy()
        nb = np.ascontiguousarray(t.nb.copy())
        cell_neg = np.empty(t.cat.size, np.uint8)
        out = np.ascontiguousarray(np.array(phi, dtype=np.float64, copy=True))
        tau = self.dx if tau is None else float(tau)
        sw = (C.c_int32 * 2)()
        self._L().or_sign_correct(self.g, self.prims, self.n_prims, _ptr(t.cat), _ptr(bg),
                              _ptr(t.meta_cell), t.n_pkg, _ptr(nb), _ptr(cell_neg), _ptr(out),
                              tau, int(max_sweeps), sw)
        return bg, nb, cell_neg, out, (int(sw[0]), int(sw[1]))

    def clean(self, phi: np.ndarray, threshold: float = 0.4, max_rounds: int = 5,
              h_ratio: float | None = None, reinit_iters: int | None = None,
              cfl: float | None = None):
        """NEXT-3 small-feature cleaning (R-23) of a copy of the dense phi.
        Returns (phi, rounds, modified per round)."""
        self._whole("clean")
        out = np.ascontiguousarray(np.array(phi, dtype=np.float64, copy=True))
        mods = np.zeros(max(1, max_rounds), np.int64)
        r = self._L().or_clean(self.g, self.prims, self.n_prims, _ptr(self._bg()), _ptr(out),
                           self.w.h_ratio if h_ratio is None else float(h_ratio), float(threshold),
                           self.w.iters if reinit_iters is None else int(reinit_iters),
                           self.w.cfl if cfl is None else float(cfl), int(max_rounds), _ptr(mods))
        return out, int(r), [int(v) for v in mods[:max_rounds]]

    def to_packages(self, dense: np.ndarray, far_neg: float, far_pos: float) -> np.ndarray:
        self._whole("to_packages")
        t = self.tables if self.tables is not None else self.build_tables()
        dense = np.ascontiguousarray(dense, dtype=np.float64)
        out = np.empty((t.n_pkg, 64))
        self._L().or_gather_packages(self.g, _ptr(dense), _ptr(t.meta_cell), t.n_pkg, far_neg,
                                 far_pos, _ptr(out))
        return out


def kernel_taps(h_ratio: float, dx: float):
    """(o int[n,3], w[n], gw[n,3]) of the O9 stencil."""
    o = np.empty((4096, 3), np.int32)
    w = np.empty(4096)
    gw = np.empty((4096, 3))
    n = int(lib().or_kernel_taps(h_ratio, dx, _ptr(o), _ptr(w), _ptr(gw)))
    return o[:n].copy(), w[:n].copy(), gw[:n].copy()


def heaviside(u: float, eps: float) -> float:
    return float(lib().or_heaviside(u, eps))


def box_to_packages(dense_box: np.ndarray) -> np.ndarray:
    """Layout helper (no arithmetic): a dense box of whole background cells,
    shape (4 bz, 4 by, 4 bx) x fastest, as per-cell packages
    [bz, by, bx, 64] in the canonical in-package order d = i + 4 j + 16 k
    (R-9).  Leading component axes are kept: (c, 4bz, 4by, 4bx) ->
    (c, bz, by, bx, 64)."""
    a = np.asarray(dense_box)
    lead = a.shape[:-3]
    mz, my, mx = a.shape[-3:]
    n = len(lead)
    # (..., bz, k, by, j, bx, i) -> (..., bz, by, bx, k, j, i)
    order = list(range(n)) + [n, n + 2, n + 4, n + 1, n + 3, n + 5]
    b = a.reshape(lead + (mz // 4, 4, my // 4, 4, mx // 4, 4)).transpose(order)
    return np.ascontiguousarray(b).reshape(lead + (mz // 4, my // 4, mx // 4, 64))
