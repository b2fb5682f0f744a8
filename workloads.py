"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no signed distance, tagging,
stencil or interpolation): only the workload definitions (grid sizes,
analytic geometry parameters, dtype, iteration counts) and the seeded particle
generator, which uses its own plain point-in-prism predicate and a
counter-based splitmix64 generator.  Both `oracle/` and
`paper_2512_11473_b200/` are driven from here; neither imports the other.

Workloads follow SURVEY.md 8(d) "Concrete synthetic inputs" (shapes of the
paper's workloads: the sphere of BASELINE.json configs[0], the extruded prism
of the teaser figure, the torus+box union, the shelled sphere of
Table 1, and the multi-shell scene).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Primitive kinds: numbers are part of the C-ABI (include/sg.h sg_prim_kind).
SPHERE, SHELL, BOX, TORUS_X, TORUS_Y, TORUS_Z, TRIPRISM_Z, LEAK = range(8)


@dataclass(frozen=True)
class Prim:
    kind: int
    p: tuple  # up to 12 doubles, meaning per kind documented in include/sg.h


@dataclass(frozen=True)
class Mesh:
    """Closed triangle mesh (NEXT-4 input): vertex coordinates flattened
    (x0, y0, z0, x1, ...) and triangles as vertex-index triples flattened,
    counter-clockwise seen from outside (outward normals)."""
    verts: tuple
    tris: tuple

    @property
    def n_verts(self) -> int:
        return len(self.verts) // 3

    @property
    def n_tris(self) -> int:
        return len(self.tris) // 3


@dataclass(frozen=True)
class Workload:
    name: str
    n: tuple  # background cells per axis
    cell: float  # l_c
    lower: tuple = (0.0, 0.0, 0.0)
    dtype: str = "f32"  # "f32" | "f64"
    prims: tuple = ()
    init_scale: float = 1.0
    far: float = 0.0  # 0 -> 4 l_c max(1, init_scale)  (reading R-4)
    iters: int = 20
    cfl: float = 0.3
    h_ratio: float = 1.3
    particles: str = ""  # "" | "prism_lattice" | "sphere_lattice"
    notes: str = ""
    mesh: Mesh | None = None  # NEXT-4: replaces the union of prims when set

    @property
    def dx(self) -> float:
        return self.cell / 4.0

    @property
    def far_value(self) -> float:
        if self.far > 0:
            return self.far
        return 4.0 * self.cell * max(1.0, self.init_scale)

    def with_(self, **kw) -> "Workload":
        d = dict(self.__dict__)
        d.update(kw)
        return Workload(**d)


def prism_teaser() -> Prim:
    """Extruded equilateral triangle (teaser): circumcentre (0.5, 0.5),
    circumradius 0.4, vertices at 90/210/330 degrees (ccw), z in [0.15, 0.85]."""
    v = []
    for deg in (90.0, 210.0, 330.0):
        a = math.radians(deg)
        v += [0.5 + 0.4 * math.cos(a), 0.5 + 0.4 * math.sin(a)]
    return Prim(TRIPRISM_Z, tuple(v) + (0.15, 0.85))


def _multi_shell() -> tuple:
    prims = [Prim(SHELL, (0.5, 0.5, 0.5, 0.3, 0.31))]
    for cz in (0.14, 0.86):
        for cy in (0.14, 0.86):
            for cx in (0.14, 0.86):
                prims.append(Prim(SHELL, (cx, cy, cz, 0.05, 0.055)))
    return tuple(prims)


CONFIGS = {
    # BASELINE.json configs[0]: sphere r=0.3, 16^3 cells x 4^3 packages, fp64
    "C1": Workload("C1", (16, 16, 16), 1.0 / 16, dtype="f64",
                   prims=(Prim(SPHERE, (0.5, 0.5, 0.5, 0.3)),), particles="sphere_lattice"),
    # configs[1]: extruded prism at 512^3 effective, reinit 20 + normals, fp32
    # configs[3] (C4) probes ~20M lattice particles against this grid.
    "C2": Workload("C2", (128, 128, 128), 1.0 / 128, dtype="f32",
                   prims=(prism_teaser(),), particles="prism_lattice"),
    # configs[2]: torus (axis y) U box at 2048^3 effective
    "C3": Workload("C3", (512, 512, 512), 1.0 / 512, dtype="f32",
                   prims=(Prim(TORUS_Y, (0.5, 0.5, 0.5, 0.3, 0.08)),
                          Prim(BOX, (0.5, 0.5, 0.5, 0.1, 0.1, 0.4)))),
    # configs[4]: thin-shell multi-body scene at 4096^3 effective
    # the particle set: lattice points at dp = dx inside the shell walls
    # (~8.99e8), shell_lattice_particles below
    "C5": Workload("C5", (1024, 1024, 1024), 1.0 / 1024, dtype="f32", prims=_multi_shell(),
                   particles="shell_lattice"),
    # Table 1 shell under reading R-19 (dx = 1/1024)
    "T1": Workload("T1", (256, 256, 256), 1.0 / 256, dtype="f32",
                   prims=(Prim(SHELL, (0.5, 0.5, 0.5, 0.3, 0.31)),)),
}


def config(name: str) -> Workload:
    return CONFIGS[name]


def fins(n: int = 32, dtype: str = "f64", thin: float = 0.5, thick: float = 4.0) -> Workload:
    """Small-feature scene (SPEC S:482-483 examples): a slab z in [0.2, 0.4]
    spanning the domain in x and y, with two walls on top (z up to 0.6, across
    the domain in x): one `thin` h thick at y = 0.3, one `thick` h thick at
    y = 0.7 (h = h_ratio dx, h_ratio 1.3)."""
    cell = 1.0 / n
    h = 1.3 * cell / 4.0
    return Workload(f"FIN{n}", (n, n, n), cell, dtype=dtype,
                    prims=(Prim(BOX, (0.5, 0.5, 0.3, 1.0, 1.0, 0.1)),
                           Prim(BOX, (0.5, 0.3, 0.5, 1.0, 0.5 * thin * h, 0.1)),
                           Prim(BOX, (0.5, 0.7, 0.5, 1.0, 0.5 * thick * h, 0.1))))


# ------------------------------------------------------------- meshes -------

def icosphere(level: int, c=(0.5, 0.5, 0.5), r: float = 0.3, rot: float = 0.0) -> Mesh:
    """Icosahedron subdivided `level` times, vertices projected onto the
    sphere (c, r) (20 * 4^level triangles, ccw from outside); `rot` rotates it
    about the axis (1, 2, 3) so no edge is grid-aligned."""
    t = (1.0 + 5 ** 0.5) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
         (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    v = [np.asarray(p, float) / np.linalg.norm(p) for p in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
         (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        mid = {}

        def m(a, b):
            k = (min(a, b), max(a, b))
            if k not in mid:
                p = v[a] + v[b]
                v.append(p / np.linalg.norm(p))
                mid[k] = len(v) - 1
            return mid[k]
        nf = []
        for a, b, cc in f:
            ab, bc, ca = m(a, b), m(b, cc), m(cc, a)
            nf += [(a, ab, ca), (b, bc, ab), (cc, ca, bc), (ab, bc, ca)]
        f = nf
    P = np.array(v)
    if rot:
        k = np.array([1.0, 2.0, 3.0]) / 14 ** 0.5
        K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
        R = np.eye(3) + math.sin(rot) * K + (1 - math.cos(rot)) * K @ K
        P = P @ R.T
    P = np.asarray(c) + r * P
    return Mesh(tuple(float(x) for x in P.ravel()), tuple(int(i) for tri in f for i in tri))


def box_mesh(c=(0.5, 0.5, 0.5), b=(0.2, 0.15, 0.25)) -> Mesh:
    """Axis-aligned box of half extents b as 12 triangles (ccw from outside)."""
    V = [(c[0] + sx * b[0], c[1] + sy * b[1], c[2] + sz * b[2])
         for sz in (-1, 1) for sy in (-1, 1) for sx in (-1, 1)]
    # vertex index = ix + 2 iy + 4 iz
    F = [(0, 2, 3), (0, 3, 1),  # z-
         (4, 5, 7), (4, 7, 6),  # z+
         (0, 1, 5), (0, 5, 4),  # y-
         (2, 6, 7), (2, 7, 3),  # y+
         (0, 4, 6), (0, 6, 2),  # x-
         (1, 3, 7), (1, 7, 5)]  # x+
    return Mesh(tuple(float(x) for p in V for x in p), tuple(i for t in F for i in t))


def read_stl(path: str, scale: float = 1.0, offset=(0.0, 0.0, 0.0)) -> Mesh:
    """Closed triangle mesh from an STL file (binary or ASCII), the paper's
    input format.  Vertices are merged by exact coordinate equality;
    facet normals in the file are ignored (orientation comes from the vertex
    order, counter-clockwise from outside); x -> scale * x + offset."""
    with open(path, "rb") as fh:
        data = fh.read()
    tris = None
    if len(data) >= 84:
        n = int(np.frombuffer(data[80:84], "<u4")[0])
        if 84 + 50 * n == len(data):  # binary
            rec = np.frombuffer(data[84:], dtype=np.dtype([("n", "<f4", 3), ("v", "<f4", (3, 3)),
                                                          ("a", "<u2")]), count=n)
            tris = rec["v"].astype(np.float64)
    if tris is None:  # ASCII
        vals = [list(map(float, ln.split()[1:4])) for ln in data.decode("ascii", "replace").splitlines()
                if ln.strip().startswith("vertex")]
        tris = np.asarray(vals, np.float64).reshape(-1, 3, 3)
    pts = tris.reshape(-1, 3) * scale + np.asarray(offset, np.float64)
    uniq, inv = np.unique(pts, axis=0, return_inverse=True)
    return Mesh(tuple(float(x) for x in uniq.ravel()), tuple(int(i) for i in inv.ravel()))


def write_stl(path: str, mesh: Mesh) -> None:
    """Binary STL of `mesh` (facet normals from the vertex order)."""
    V = np.asarray(mesh.verts, np.float64).reshape(-1, 3)
    T = np.asarray(mesh.tris, np.int64).reshape(-1, 3)
    rec = np.zeros(len(T), dtype=np.dtype([("n", "<f4", 3), ("v", "<f4", (3, 3)), ("a", "<u2")]))
    tri = V[T]
    nrm = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
    rec["n"] = nrm / np.maximum(np.linalg.norm(nrm, axis=1, keepdims=True), 1e-300)
    rec["v"] = tri
    with open(path, "wb") as fh:
        fh.write(b"sgrid-b200 binary STL".ljust(80, b" "))
        fh.write(np.uint32(len(T)).tobytes())
        fh.write(rec.tobytes())


def mesh_workload(name: str, mesh: Mesh, n: int, dtype: str = "f64") -> Workload:
    """A mesh geometry on an n^3 grid of the unit domain (NEXT-4)."""
    return Workload(name, (n, n, n), 1.0 / n, dtype=dtype, mesh=mesh)


# Leak balls (cx, cy, cz, r) in the unit domain of the configs: one inside
# the body, one straddling its surface, one in the far field (a stand-in for
# the sign errors of a mesh SDF on leaky input; SG_LEAK in sg.h).
LEAK_BALLS = ((0.5, 0.5, 0.5, 0.2), (0.78, 0.42, 0.55, 0.15), (0.12, 0.85, 0.2, 0.1))


def leaky(w: Workload, balls=LEAK_BALLS, margin_cells: float = 1.0) -> Workload:
    """`w` with SG_LEAK sign-error balls appended; the sign of f flips inside
    a ball where |f| >= margin_cells * l_c (core cells stay correct)."""
    leaks = tuple(Prim(LEAK, tuple(b) + (margin_cells * w.cell,)) for b in balls)
    return w.with_(name=w.name + "L", prims=tuple(w.prims) + leaks)


# ------------------------------------------------------------ random scenes --

def random_scene(seed: int, n: int, dtype: str = "f64") -> Workload:
    """Small seeded scene (union of 1-3 spheres/boxes/tori) on an n^3 grid,
    for table/field parity beyond the fixed configs.  Some scenes let the band
    touch the domain boundary on purpose (reading R-6)."""
    rng = np.random.default_rng(seed)
    cell = 1.0 / n
    prims = []
    for _ in range(int(rng.integers(1, 4))):
        kind = int(rng.choice([SPHERE, BOX, TORUS_X, TORUS_Y, TORUS_Z, SHELL]))
        c = tuple(float(v) for v in rng.uniform(0.25, 0.75, 3))
        if kind == SPHERE:
            prims.append(Prim(kind, c + (float(rng.uniform(0.1, 0.35)),)))
        elif kind == SHELL:
            r = float(rng.uniform(0.15, 0.3))
            prims.append(Prim(kind, c + (r, r + float(rng.uniform(0.01, 0.08)))))
        elif kind == BOX:
            prims.append(Prim(kind, c + tuple(float(v) for v in rng.uniform(0.05, 0.3, 3))))
        else:
            R = float(rng.uniform(0.12, 0.25))
            prims.append(Prim(kind, c + (R, float(rng.uniform(0.04, 0.1)))))
    return Workload(f"rand{seed}_{n}", (n, n, n), cell, dtype=dtype, prims=tuple(prims))


# ------------------------------------------------------- particle generator --

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based splitmix64 (Steele, Lea, Flood 2014) on uint64 arrays."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def _inside_prism(prim: Prim, x, y, z):
    """Closed point-in-prism predicate (edge-function signs; not an SDF)."""
    p = prim.p
    ok = (z >= p[6]) & (z <= p[7])
    for e in range(3):
        ax, ay = p[2 * e], p[2 * e + 1]
        bx, by = p[2 * ((e + 1) % 3)], p[2 * ((e + 1) % 3) + 1]
        ok &= (bx - ax) * (y - ay) - (by - ay) * (x - ax) >= 0.0
    return ok


def _inside_sphere(prim: Prim, x, y, z):
    c = prim.p
    return (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= c[3] ** 2


def lattice_particles(w: Workload, dp: float | None = None, seed: int = 0,
                      jitter: float = 0.25, order: str = "lattice",
                      dtype=np.float32) -> np.ndarray:
    """SPH-style particle set (C4): lattice points (i + 1/2) dp
    inside the body, each coordinate jittered by U(-jitter dp, +jitter dp)
    drawn from splitmix64(seed ^ (3 * index + axis)).  order "lattice" keeps
    z-slowest lattice order (sorted by cell), "shuffled" applies a seeded
    permutation.  Returns an (n, 3) array of `dtype`."""
    dp = w.dx if dp is None else dp
    prim = w.prims[0]
    inside = {TRIPRISM_Z: _inside_prism, SPHERE: _inside_sphere}[prim.kind]
    m = [int(round(w.n[k] * w.cell / dp)) for k in range(3)]
    xs = w.lower[0] + (np.arange(m[0]) + 0.5) * dp
    ys = w.lower[1] + (np.arange(m[1]) + 0.5) * dp
    X, Y = np.meshgrid(xs, ys, indexing="xy")  # X varies fastest along axis 1
    X = X.ravel()
    Y = Y.ravel()
    chunks = []
    for iz in range(m[2]):
        zc = w.lower[2] + (iz + 0.5) * dp
        sel = inside(prim, X, Y, zc)
        if sel.any():
            pts = np.empty((int(sel.sum()), 3), dtype=np.float64)
            pts[:, 0] = X[sel]
            pts[:, 1] = Y[sel]
            pts[:, 2] = zc
            chunks.append(pts)
    pos = np.concatenate(chunks) if chunks else np.zeros((0, 3))
    n = pos.shape[0]
    if jitter:
        ctr = (np.arange(n, dtype=np.uint64) * np.uint64(3))[:, None] + np.arange(3, dtype=np.uint64)[None, :]
        r = splitmix64(np.uint64(seed) ^ ctr)
        u = (r >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        pos = pos + (u - 0.5) * (2.0 * jitter * dp)
    if order == "shuffled":
        perm = np.random.default_rng(seed + 1).permutation(n)
        pos = pos[perm]
    return np.ascontiguousarray(pos.astype(dtype))


def random_positions(w: Workload, n: int, seed: int = 0, margin: float = 0.0,
                     dtype=np.float64) -> np.ndarray:
    """Uniform positions in the domain (optionally shrunk by `margin`)."""
    rng = np.random.default_rng(seed)
    lo = np.array(w.lower) + margin
    hi = np.array(w.lower) + np.array(w.n) * w.cell - margin
    return np.ascontiguousarray(rng.uniform(lo, hi, size=(n, 3)).astype(dtype))


# ------------------------------------------------ C5: shell-wall particles --
_SM_GAMMA = 0x9E3779B97F4A7C15
_SM_M1 = 0xBF58476D1CE4E5B9
_SM_M2 = 0x94D049BB133111EB


def _i64(c: int) -> int:
    """a uint64 constant as the int64 with the same bits"""
    return c - (1 << 64) if c >= (1 << 63) else c


def splitmix64_torch(x):
    """splitmix64 (same bits as splitmix64 above) on an int64 torch tensor
    holding uint64 bit patterns: wrapping multiplies, logical shifts."""
    import torch

    def srl(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)
    z = x + _i64(_SM_GAMMA)
    z = (z ^ srl(z, 30)) * _i64(_SM_M1)
    z = (z ^ srl(z, 27)) * _i64(_SM_M2)
    return z ^ srl(z, 31)


def shell_lattice_particles(w: Workload, seed: int = 0, jitter: float = 0.25, z_range=None,
                            box=None, device="cpu", dtype=None, chunk_planes: int = 256):
    """C5 particle set: lattice points p_i = (i + 1/2) dp, dp = dx,
    inside the walls of the scene's shells -- r_in^2 <= |p - c|^2 <= r_out^2
    for some shell, |p - c|^2 evaluated as ((ex ex + ey ey) + ez ez) in fp64 (a
    containment predicate, not an SDF) -- in lattice order (z slowest, then y,
    then x), each coordinate jittered by U(-jitter dp, +jitter dp) from
    splitmix64(seed ^ (3 L + axis)), L = ix + m (iy + m iz) the LATTICE index
    (so any sub-range of planes regenerates the same particles).
    z_range: lattice planes [z0, z1) (default all); box: optional lattice box
    ((x0, y0, z0), (x1, y1, z1)) restricting the output.  Built row by row:
    per (shell, lattice row) the wall segments in x are found from the row's
    distance to the centre, widened by one lattice point each side, and the
    candidates are tested with the predicate -- no scan of the 4096^3
    lattice.  Returns an (n, 3) torch tensor on `device`."""
    import torch
    dev = torch.device(device)
    dtype = dtype or (torch.float32 if w.dtype == "f32" else torch.float64)
    dp = w.dx
    m = int(round(w.n[0] * w.cell / dp))
    assert all(int(round(w.n[k] * w.cell / dp)) == m for k in range(3)) and w.lower == (0.0, 0.0, 0.0)
    shells = [pr.p[:5] for pr in w.prims if pr.kind == SHELL]
    z0, z1 = (0, m) if z_range is None else (max(0, z_range[0]), min(m, z_range[1]))
    if box is not None:
        z0, z1 = max(z0, box[0][2]), min(z1, box[1][2])
    f64, i64 = torch.float64, torch.int64
    out = []
    for za in range(z0, z1, chunk_planes):
        zb = min(z1, za + chunk_planes)
        segs = []  # (iz, iy, ia, ib, shell index) rows of int64
        for si, (cx, cy, cz, ri, ro) in enumerate(shells):
            iz = torch.arange(za, zb, device=dev, dtype=i64)
            ez = (iz.to(f64) + 0.5) * dp - cz
            keep = ez.abs() <= ro
            iz, ez = iz[keep], ez[keep]
            if iz.numel() == 0:
                continue
            hy = torch.sqrt(torch.clamp(ro * ro - ez * ez, min=0.0))
            ya = torch.clamp(torch.floor((cy - hy) / dp - 0.5).to(i64) - 1, 0, m - 1)
            yb = torch.clamp(torch.ceil((cy + hy) / dp - 0.5).to(i64) + 1, 0, m - 1)
            if box is not None:
                ya = torch.clamp(ya, min=box[0][1])
                yb = torch.clamp(yb, max=box[1][1] - 1)
            cnt = torch.clamp(yb - ya + 1, min=0)
            rz = torch.repeat_interleave(torch.arange(iz.numel(), device=dev), cnt)
            if rz.numel() == 0:
                continue
            start = torch.cumsum(cnt, 0) - cnt
            iy = ya[rz] + (torch.arange(rz.numel(), device=dev) - start[rz])
            ey = (iy.to(f64) + 0.5) * dp - cy
            d2 = ez[rz] * ez[rz] + ey * ey
            ho = torch.sqrt(torch.clamp(ro * ro - d2, min=0.0))
            hin = torch.sqrt(torch.clamp(ri * ri - d2, min=0.0))
            ok = d2 <= ro * ro
            izr, iy, ho, hin = iz[rz][ok], iy[ok], ho[ok], hin[ok]

            def lat(v, up):
                f = v / dp - 0.5
                return torch.clamp((torch.ceil(f) + 1 if up else torch.floor(f) - 1).to(i64), 0, m - 1)
            la, lb = lat(cx - ho, False), lat(cx - hin, True)
            ra, rb = lat(cx + hin, False), lat(cx + ho, True)
            merged = ra <= lb  # no hole in this row (or margins touch): one segment
            one = torch.stack([izr, iy, la, torch.where(merged, rb, lb),
                               torch.full_like(la, si)], 1)
            two = torch.stack([izr, iy, ra, rb, torch.full_like(la, si)], 1)[~merged]
            segs += [one, two]
        if not segs:
            continue
        S = torch.cat(segs)
        if box is not None:
            S[:, 2] = torch.clamp(S[:, 2], min=box[0][0])
            S[:, 3] = torch.clamp(S[:, 3], max=box[1][0] - 1)
            S = S[S[:, 3] >= S[:, 2]]
        key = (S[:, 0] * m + S[:, 1]) * m + S[:, 2]
        S = S[torch.argsort(key)]
        cnt = S[:, 3] - S[:, 2] + 1
        rs = torch.repeat_interleave(torch.arange(S.shape[0], device=dev), cnt)
        start = torch.cumsum(cnt, 0) - cnt
        ix = S[rs, 2] + (torch.arange(rs.numel(), device=dev) - start[rs])
        iy, iz, sh = S[rs, 1], S[rs, 0], S[rs, 4]
        del rs, start
        P = torch.tensor(shells, dtype=f64, device=dev)
        x = (ix.to(f64) + 0.5) * dp
        y = (iy.to(f64) + 0.5) * dp
        z = (iz.to(f64) + 0.5) * dp
        ex, ey, ez = x - P[sh, 0], y - P[sh, 1], z - P[sh, 2]
        d2 = (ex * ex + ey * ey) + ez * ez
        keep = (d2 >= P[sh, 3] * P[sh, 3]) & (d2 <= P[sh, 4] * P[sh, 4])
        del ex, ey, ez, d2, sh
        ix, iy, iz, x, y, z = ix[keep], iy[keep], iz[keep], x[keep], y[keep], z[keep]
        if jitter:
            L = ix + m * (iy + m * iz)
            pos = torch.stack([x, y, z], 1)
            for a in range(3):
                r = splitmix64_torch(seed ^ (3 * L + a))
                u = ((r >> 11) & ((1 << 53) - 1)).to(f64) * (1.0 / 9007199254740992.0)
                pos[:, a] += (u - 0.5) * (2.0 * jitter * dp)
        else:
            pos = torch.stack([x, y, z], 1)
        out.append(pos.to(dtype))
        del ix, iy, iz, x, y, z, pos
    if not out:
        return torch.zeros((0, 3), dtype=dtype, device=dev)
    return torch.cat(out).contiguous()


def particles(w: Workload, seed: int = 0, order: str = "lattice", device="cpu", dtype=None):
    """The workload's particle set as an (n, 3) torch tensor on `device`
    (C4: lattice_particles; C5: shell_lattice_particles, generated on the
    device); empty if the workload has none."""
    import torch
    npdt = np.float32 if w.dtype == "f32" else np.float64
    tdt = dtype or (torch.float32 if w.dtype == "f32" else torch.float64)
    if not w.particles:
        return torch.zeros((0, 3), dtype=tdt, device=device)
    if w.particles == "shell_lattice":
        p = shell_lattice_particles(w, seed=seed, device=device, dtype=tdt)
        if order == "shuffled":
            g = torch.Generator(device="cpu").manual_seed(seed + 1)
            p = p[torch.randperm(p.shape[0], generator=g).to(p.device)]
        return p
    return torch.from_numpy(lattice_particles(w, seed=seed, order=order, dtype=npdt)).to(device)
