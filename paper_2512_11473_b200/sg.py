"""Thin Python binding of libsg (include/sg.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libsg.so; this module
only converts Python/torch arguments into the C-ABI's plain pointers and
sizes.  There is no fallback: if libsg.so is missing, or no CUDA device is
present, the calls raise.

Low-level functions carry the C names (sg_build, sg_reinit, sg_gradient,
sg_probe, sg_table1, sg_info, sg_view, sg_destroy, ...).  `Grid` is a small
convenience wrapper over them that hands out zero-copy torch views.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsg.so")

SG_OK, SG_ERR_ARG, SG_ERR_OOM, SG_ERR_CUDA, SG_ERR_NCCL, SG_ERR_STATE, SG_ERR_DOMAIN = range(7)
SG_F32, SG_F64 = 0, 1
SG_GRAD, SG_NORMAL, SG_KINT = 1, 2, 4
VIEWS = {"bg": 0, "meta_cell": 1, "meta_cat": 2, "nb": 3, "phi": 4, "grad": 5, "normal": 6,
         "kint": 7, "gkint": 8, "plane_first": 9, "phi_next": 10, "cell_core": 11,
         "cell_neg": 12, "face": 13}
_STATUS = {0: "SG_OK", 1: "SG_ERR_ARG", 2: "SG_ERR_OOM", 3: "SG_ERR_CUDA", 4: "SG_ERR_NCCL",
           5: "SG_ERR_STATE", 6: "SG_ERR_DOMAIN"}

# exported symbols declared in include/sg.h (checked by the CPU test suite)
EXPORTS = ("sg_build", "sg_build_ex", "sg_build_refined", "sg_reinit", "sg_reinit_halo",
           "sg_gradient", "sg_probe", "sg_table1", "sg_relax",
           "sg_sign_correct", "sg_clean", "sg_info", "sg_view",
           "sg_destroy", "sg_destroy_async", "sg_balanced_cuts", "sg_plane_counts",
           "sg_slab_plan", "sg_comm_unique_id", "sg_comm_create", "sg_comm_create_local",
           "sg_comm_info", "sg_comm_check", "sg_comm_destroy", "sg_pool_trim",
           "sg_neighbour_index_shift", "sg_last_error", "sg_abi_version", "sg_launch_count")
SG_COMM_ID_BYTES = 128
SG_COMM_NCCL, SG_COMM_LOCAL = 0, 1


class SgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class sg_prim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad", C.c_int32), ("p", C.c_double * 12)]


class sg_geometry(C.Structure):
    _fields_ = [("prims", C.POINTER(sg_prim)), ("n_prims", C.c_int32), ("pad", C.c_int32),
                ("verts", C.POINTER(C.c_double)), ("tris", C.POINTER(C.c_int32)),
                ("n_verts", C.c_int32), ("n_tris", C.c_int32)]


class sg_desc(C.Structure):
    _fields_ = [("lower", C.c_double * 3), ("cell", C.c_double), ("n", C.c_int32 * 3),
                ("pkg", C.c_int32), ("dtype", C.c_int32), ("pad", C.c_int32),
                ("far", C.c_double), ("init_scale", C.c_double)]


class sg_slab(C.Structure):
    _fields_ = [("z_lo", C.c_int32), ("z_hi", C.c_int32), ("id_base", C.c_int64)]


class sg_relax_params(C.Structure):
    _fields_ = [("dp", C.c_double), ("h_ratio", C.c_double), ("step", C.c_double),
                ("max_disp", C.c_double), ("surface_offset", C.c_double), ("steps", C.c_int32),
                ("pad", C.c_int32)]


class sg_view_t(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("shape", C.c_int64 * 3), ("ndim", C.c_int32),
                ("elem_size", C.c_int32), ("dtype", C.c_int32), ("pad", C.c_int32)]


class sg_info_t(C.Structure):
    _fields_ = [("n_pkg", C.c_int64), ("n_core", C.c_int64), ("n_inner", C.c_int64),
                ("id_base", C.c_int64), ("dtype", C.c_int32), ("z_lo", C.c_int32),
                ("z_hi", C.c_int32), ("zs_lo", C.c_int32), ("zs_hi", C.c_int32),
                ("pad", C.c_int32), ("dx", C.c_double), ("far", C.c_double),
                ("kernel_sum", C.c_double), ("has_grad", C.c_int32), ("has_normal", C.c_int32),
                ("has_kint", C.c_int32), ("phi_cur", C.c_int32), ("device_bytes", C.c_int64),
                ("own_lo", C.c_int64), ("own_hi", C.c_int64), ("rank", C.c_int32),
                ("nranks", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class sg_plan_t(C.Structure):
    _fields_ = [("z_lo", C.c_int32), ("z_hi", C.c_int32), ("zs_lo", C.c_int32),
                ("zs_hi", C.c_int32), ("id_base", C.c_int64), ("n_pkg", C.c_int64),
                ("own_lo", C.c_int64), ("own_hi", C.c_int64), ("send_lo", C.c_int64 * 2),
                ("send_hi", C.c_int64 * 2), ("recv_lo", C.c_int64 * 2), ("recv_hi", C.c_int64 * 2)]

    def as_dict(self):
        return {k: (tuple(getattr(self, k)) if k.startswith(("send", "recv")) else getattr(self, k))
                for k, _ in self._fields_}


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class sg_allocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", C.c_void_p)]


class sg_build_opts(C.Structure):
    _fields_ = [("slab", C.POINTER(sg_slab)), ("comm", C.c_void_p),
                ("allocator", C.POINTER(sg_allocator))]


_lib = None


def lib():
    """Load libsg.so (built in-tree by paper_2512_11473_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libsg.so not built: run `python -m paper_2512_11473_b200.build` "
                              f"({LIB_PATH} missing); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.sg_build.argtypes = [C.POINTER(sg_desc), C.POINTER(sg_geometry), C.POINTER(sg_slab), P,
                               C.POINTER(P)]
        L.sg_build_refined.argtypes = [P, C.POINTER(sg_geometry), P, C.POINTER(P)]
        L.sg_reinit.argtypes = [P, I32, D, P]
        L.sg_reinit_halo.argtypes = [P, I32, D, P]
        L.sg_gradient.argtypes = [P, C.c_uint32, D, P]
        L.sg_probe.argtypes = [P, I64, P, P, P, P, P]
        L.sg_table1.argtypes = [P, I32, D, P]
        L.sg_relax.argtypes = [P, I64, P, C.POINTER(sg_relax_params), P]
        L.sg_sign_correct.argtypes = [P, D, I32, C.POINTER(I32), P]
        L.sg_clean.argtypes = [P, D, D, I32, D, I32, C.POINTER(I32), C.POINTER(I64), P]
        L.sg_info.argtypes = [P, C.POINTER(sg_info_t)]
        L.sg_view.argtypes = [P, I32, C.POINTER(sg_view_t)]
        L.sg_destroy.argtypes = [P]
        L.sg_destroy.restype = None
        L.sg_destroy_async.argtypes = [P, P]
        L.sg_balanced_cuts.argtypes = [P, I32, I32, P]
        L.sg_plane_counts.argtypes = [C.POINTER(sg_desc), C.POINTER(sg_geometry), I32, I32, P, P]
        L.sg_build_ex.argtypes = [C.POINTER(sg_desc), C.POINTER(sg_geometry),
                                  C.POINTER(sg_build_opts), P, C.POINTER(P)]
        L.sg_slab_plan.argtypes = [P, I32, I32, I32, C.POINTER(sg_plan_t), P]
        L.sg_comm_unique_id.argtypes = [P]
        L.sg_comm_create.argtypes = [P, I32, I32, C.POINTER(P)]
        L.sg_comm_create_local.argtypes = [I32, P]
        L.sg_comm_info.argtypes = [P, P, P, P]
        L.sg_comm_check.argtypes = [P]
        L.sg_comm_destroy.argtypes = [P]
        L.sg_comm_destroy.restype = None
        L.sg_pool_trim.argtypes = []
        L.sg_neighbour_index_shift.argtypes = [P, P, P]
        L.sg_neighbour_index_shift.restype = I32
        L.sg_last_error.restype = C.c_char_p
        L.sg_abi_version.restype = I32
        L.sg_launch_count.restype = C.c_uint64
        for name in ("sg_build", "sg_build_refined", "sg_reinit", "sg_reinit_halo", "sg_gradient", "sg_probe", "sg_table1", "sg_relax",
                     "sg_sign_correct", "sg_clean",
                     "sg_info",
                     "sg_view", "sg_destroy_async", "sg_balanced_cuts", "sg_plane_counts",
                     "sg_build_ex", "sg_slab_plan", "sg_comm_unique_id", "sg_comm_create",
                     "sg_comm_create_local", "sg_comm_info", "sg_comm_check", "sg_pool_trim"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != SG_OK:
        raise SgError(st, lib().sg_last_error().decode(errors="replace"))


def _stream(stream):
    """torch.cuda.Stream | int | None -> void*"""
    if stream is None:
        try:
            import torch
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            return C.c_void_p(0)
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def make_desc(w) -> tuple:
    """Workload-like object (n, cell, lower, dtype, prims, far, init_scale)
    -> (sg_desc, sg_geometry, keepalive)."""
    d = sg_desc()
    for k in range(3):
        d.lower[k] = float(w.lower[k])
        d.n[k] = int(w.n[k])
    d.cell = float(w.cell)
    d.pkg = 4
    d.dtype = SG_F64 if w.dtype in ("f64", "float64") else SG_F32
    d.far = float(getattr(w, "far", 0.0) or 0.0)
    d.init_scale = float(getattr(w, "init_scale", 1.0) or 1.0)
    prims = (sg_prim * max(1, len(w.prims)))()
    for i, pr in enumerate(w.prims):
        prims[i].kind = int(pr.kind)
        for j, v in enumerate(pr.p):
            prims[i].p[j] = float(v)
    geom = sg_geometry(C.cast(prims, C.POINTER(sg_prim)), len(w.prims), 0)
    keep = [prims]
    mesh = getattr(w, "mesh", None)
    if mesh is not None:
        verts = (C.c_double * len(mesh.verts))(*mesh.verts)
        tris = (C.c_int32 * len(mesh.tris))(*mesh.tris)
        geom.verts = C.cast(verts, C.POINTER(C.c_double))
        geom.tris = C.cast(tris, C.POINTER(C.c_int32))
        geom.n_verts = len(mesh.verts) // 3
        geom.n_tris = len(mesh.tris) // 3
        keep += [verts, tris]
    return d, geom, keep


# ------------------------------------------------------------ raw C calls --

def sg_build(desc: sg_desc, geom: sg_geometry, slab: sg_slab | None = None, stream=None) -> int:
    out = C.c_void_p()
    _check(lib().sg_build(C.byref(desc), C.byref(geom), C.byref(slab) if slab else None,
                          _stream(stream), C.byref(out)))
    return out.value


def sg_reinit(grid: int, iters: int, cfl: float = 0.3, stream=None) -> None:
    _check(lib().sg_reinit(C.c_void_p(grid), int(iters), float(cfl), _stream(stream)))


def sg_reinit_halo(grid: int, iters: int, cfl: float = 0.3, stream=None) -> None:
    _check(lib().sg_reinit_halo(C.c_void_p(grid), int(iters), float(cfl), _stream(stream)))


def sg_gradient(grid: int, fields: int = SG_GRAD | SG_NORMAL, h_ratio: float = 1.3,
                stream=None) -> None:
    _check(lib().sg_gradient(C.c_void_p(grid), int(fields), float(h_ratio), _stream(stream)))


def sg_probe(grid: int, n: int, pos_ptr: int, phi_ptr: int, grad_ptr: int | None = None,
             oob_ptr: int | None = None, stream=None) -> None:
    _check(lib().sg_probe(C.c_void_p(grid), int(n), C.c_void_p(pos_ptr), C.c_void_p(phi_ptr),
                          C.c_void_p(grad_ptr) if grad_ptr else None,
                          C.c_void_p(oob_ptr) if oob_ptr else None, _stream(stream)))


def sg_table1(grid: int, op: int, value: float = 1.0, stream=None) -> None:
    _check(lib().sg_table1(C.c_void_p(grid), int(op), float(value), _stream(stream)))


def sg_relax(grid: int, n: int, pos_ptr: int, dp: float, h_ratio: float = 1.3,
             step: float = 0.1, max_disp: float = 0.2, surface_offset: float = 0.5,
             steps: int = 1, stream=None) -> None:
    p = sg_relax_params(dp, h_ratio, step, max_disp, surface_offset, int(steps), 0)
    _check(lib().sg_relax(C.c_void_p(grid), int(n), C.c_void_p(pos_ptr), C.byref(p),
                          _stream(stream)))


def sg_sign_correct(grid: int, tau: float, max_sweeps: int = 0, stream=None) -> tuple:
    """Sign-consistency correction (NEXT-3); returns the (coarse, refined)
    numbers of sweeps that signed something."""
    sw = (C.c_int32 * 2)()
    _check(lib().sg_sign_correct(C.c_void_p(grid), float(tau), int(max_sweeps), sw,
                                 _stream(stream)))
    return int(sw[0]), int(sw[1])


def sg_clean(grid: int, h_ratio: float = 1.3, threshold: float = 0.4, reinit_iters: int = 20,
             cfl: float = 0.3, max_rounds: int = 5, stream=None) -> tuple:
    """Small-feature cleaning (NEXT-3); returns (rounds, [raised per round])."""
    r = C.c_int32(0)
    mods = (C.c_int64 * max(1, int(max_rounds)))()
    _check(lib().sg_clean(C.c_void_p(grid), float(h_ratio), float(threshold), int(reinit_iters),
                          float(cfl), int(max_rounds), C.byref(r), mods, _stream(stream)))
    return int(r.value), [int(mods[i]) for i in range(int(max_rounds))]


def sg_info(grid: int) -> dict:
    info = sg_info_t()
    _check(lib().sg_info(C.c_void_p(grid), C.byref(info)))
    return info.as_dict()


def sg_view(grid: int, what: int) -> sg_view_t:
    v = sg_view_t()
    _check(lib().sg_view(C.c_void_p(grid), int(what), C.byref(v)))
    return v


def sg_destroy(grid: int) -> None:
    lib().sg_destroy(C.c_void_p(grid))


def sg_destroy_async(grid: int, stream=None) -> None:
    _check(lib().sg_destroy_async(C.c_void_p(grid), _stream(stream)))


def sg_balanced_cuts(counts, nranks: int) -> list:
    import numpy as np
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
    cuts = np.zeros(nranks + 1, dtype=np.int32)
    _check(lib().sg_balanced_cuts(c.ctypes.data_as(C.c_void_p), int(c.size), int(nranks),
                                  cuts.ctypes.data_as(C.c_void_p)))
    return [int(v) for v in cuts]


def sg_plane_counts(desc: sg_desc, geom: sg_geometry, z_lo: int, z_hi: int, counts_ptr: int,
                    stream=None) -> None:
    _check(lib().sg_plane_counts(C.byref(desc), C.byref(geom), int(z_lo), int(z_hi),
                                 C.c_void_p(counts_ptr), _stream(stream)))


def sg_slab_plan(counts, nranks: int, rank: int) -> tuple:
    """Host-only z-slab plan (include/sg.h sg_slab_plan): (plan dict, cuts)."""
    import numpy as np
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
    cuts = np.zeros(nranks + 1, dtype=np.int32)
    p = sg_plan_t()
    _check(lib().sg_slab_plan(c.ctypes.data_as(C.c_void_p), int(c.size), int(nranks), int(rank),
                              C.byref(p), cuts.ctypes.data_as(C.c_void_p)))
    return p.as_dict(), [int(v) for v in cuts]


def sg_pool_trim() -> None:
    _check(lib().sg_pool_trim())


class Comm:
    """Communicator handle (include/sg.h sg_comm_*).

    Comm.nccl(group): one process per GPU, NCCL over NVLink; the unique id is
    broadcast with torch.distributed (rank 0 creates it).
    Comm.local(n): n in-process communicators on the current device (each to
    be driven by its own thread) -- the emulation used by the 1-GPU tests."""

    def __init__(self, handle: int):
        self.handle = handle
        r, n, k = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().sg_comm_info(C.c_void_p(handle), C.byref(r), C.byref(n), C.byref(k)))
        self.rank, self.nranks, self.kind = r.value, n.value, k.value

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * SG_COMM_ID_BYTES)()
        _check(lib().sg_comm_unique_id(buf))
        return bytes(buf.raw)

    @classmethod
    def nccl(cls, group=None) -> "Comm":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        uid = (C.c_char * SG_COMM_ID_BYTES).from_buffer_copy(obj[0])
        out = C.c_void_p()
        _check(lib().sg_comm_create(uid, rank, world, C.byref(out)))
        return cls(out.value)

    @classmethod
    def local(cls, n: int) -> list:
        arr = (C.c_void_p * n)()
        _check(lib().sg_comm_create_local(int(n), arr))
        return [cls(arr[i]) for i in range(n)]

    def check(self):
        """Raise SgError(SG_ERR_NCCL) on an asynchronous NCCL error."""
        _check(lib().sg_comm_check(C.c_void_p(self.handle)))

    def close(self):
        if getattr(self, "handle", None):
            lib().sg_comm_destroy(C.c_void_p(self.handle))
            self.handle = None


class TorchAllocator:
    """sg_allocator backed by PyTorch's caching allocator (grid memory then
    shows up in torch.cuda.memory_allocated and is shared with torch)."""

    def __init__(self):
        import torch

        def _alloc(nbytes, stream, ctx):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(),
                                                          int(stream or 0))
            except Exception:
                return None

        def _free(ptr, nbytes, stream, ctx):
            torch.cuda.caching_allocator_delete(int(ptr))

        self._a, self._f = _ALLOC_FN(_alloc), _FREE_FN(_free)  # keep the thunks alive
        self.struct = sg_allocator(self._a, self._f, None)


def sg_neighbour_index_shift(shift) -> tuple:
    """Lst. 2 (host-callable): shift (3 ints in [-4, 7]) -> (slot, offset
    triple, data triple); slot -1 if out of range."""
    sh = (C.c_int32 * 3)(*[int(v) for v in shift])
    off = (C.c_int32 * 3)()
    dat = (C.c_int32 * 3)()
    slot = int(lib().sg_neighbour_index_shift(sh, off, dat))
    return slot, tuple(off), tuple(dat)


def sg_launch_count() -> int:
    return int(lib().sg_launch_count())


def sg_abi_version() -> int:
    return int(lib().sg_abi_version())


# ---------------------------------------------------------------- torch ----

_TORCH_DT = {0: "float32", 1: "float64", 2: "uint32", 3: "uint8", 4: "int64"}
_TYPESTR = {0: "<f4", 1: "<f8", 2: "<u4", 3: "|u1", 4: "<i8"}


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def view_tensor(grid: int, name: str):
    """Zero-copy torch view of a device array of the grid (non-owning: valid
    until the grid is destroyed or, for phi, the next reinit swap)."""
    import torch
    v = sg_view(grid, VIEWS[name])
    if not v.ptr:
        raise SgError(SG_ERR_STATE, f"view '{name}' not computed yet")
    shape = [v.shape[i] for i in range(v.ndim)]
    if v.dtype == 2:  # torch lacks full uint32 support: expose as int32 bits
        t = torch.as_tensor(_CAI(v.ptr, shape, "<i4"), device="cuda")
        return t
    return torch.as_tensor(_CAI(v.ptr, shape, _TYPESTR[v.dtype]), device="cuda")


_DESC_CACHE: dict = {}


def _cached_desc(w):
    """make_desc memoised per (hashable) workload: rebuilding a grid every
    step does not re-marshal the descriptor."""
    try:
        hit = _DESC_CACHE.get(w)
    except TypeError:  # unhashable workload-like object
        return make_desc(w)
    if hit is None:
        hit = _DESC_CACHE[w] = make_desc(w)
    return hit


class Grid:
    """Owning handle around sg_build/sg_destroy with torch-friendly calls."""

    def __init__(self, w, slab: tuple | None = None, stream=None, parent=None, comm=None,
                 allocator=None):
        """slab: explicit (z_lo, z_hi, id_base); comm: a Comm (partitioned
        grid, collective calls); allocator: a TorchAllocator (grid memory
        from PyTorch's caching allocator) or None (the library's pool)."""
        self.w = w
        self.desc, self.geom, self._keep = _cached_desc(w)
        self.comm = comm
        self._allocator = allocator  # keep alive while the grid lives
        if parent is not None:  # NEXT-4: layer refined from `parent`
            out = C.c_void_p()
            _check(lib().sg_build_refined(C.c_void_p(parent.handle), C.byref(self.geom),
                                          _stream(stream), C.byref(out)))
            self.handle = out.value
            return
        sl = None
        if slab is not None:
            sl = sg_slab(int(slab[0]), int(slab[1]), int(slab[2]))
        if comm is None and allocator is None:
            self.handle = sg_build(self.desc, self.geom, sl, stream)
            return
        opts = sg_build_opts(C.pointer(sl) if sl is not None else None,
                             C.c_void_p(comm.handle) if comm is not None else None,
                             C.pointer(allocator.struct) if allocator is not None else None)
        out = C.c_void_p()
        _check(lib().sg_build_ex(C.byref(self.desc), C.byref(self.geom), C.byref(opts),
                                 _stream(stream), C.byref(out)))
        self.handle = out.value

    def refined(self, stream=None) -> "Grid":
        """The next finer layer (cell / 2, 2 n cells per axis) built from this
        grid (NEXT-4 multi-resolution, sg_build_refined)."""
        w = self.w
        wf = w.with_(name=w.name + "r", n=tuple(2 * k for k in w.n), cell=0.5 * w.cell)
        return Grid(wf, stream=stream, parent=self)

    @property
    def info(self) -> dict:
        return sg_info(self.handle)

    def reinit(self, iters: int, cfl: float = 0.3, stream=None):
        sg_reinit(self.handle, iters, cfl, stream)
        return self

    def gradient(self, fields: int = SG_GRAD | SG_NORMAL, h_ratio: float = 1.3, stream=None):
        sg_gradient(self.handle, fields, h_ratio, stream)
        return self

    def table1(self, op: int, value: float = 1.0, stream=None):
        sg_table1(self.handle, op, value, stream)
        return self

    def _check_pos(self, pos, what: str, device_only: bool = False):
        """The C-ABI reads n x 3 contiguous values of the grid dtype: reject
        anything else before it reaches the kernels."""
        import torch
        want = torch.float64 if self.desc.dtype == SG_F64 else torch.float32
        if pos.dtype != want:
            raise SgError(SG_ERR_ARG, f"{what}: positions are {pos.dtype}, the grid is {want}")
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise SgError(SG_ERR_ARG, f"{what}: positions must have shape (n, 3), got "
                                      f"{tuple(pos.shape)}")
        if not pos.is_contiguous():
            raise SgError(SG_ERR_ARG, f"{what}: positions must be contiguous (row-major n x 3)")
        if pos.device.type == "cuda":
            if pos.device.index is not None and pos.device.index != torch.cuda.current_device():
                raise SgError(SG_ERR_ARG, f"{what}: positions on {pos.device}, current device "
                                          f"is cuda:{torch.cuda.current_device()}")
        elif device_only or pos.device.type != "cpu":
            raise SgError(SG_ERR_ARG, f"{what}: positions must be a CUDA tensor")

    def probe(self, pos, want_grad: bool = True, oob=None, stream=None):
        """pos: torch tensor (n, 3) of the grid dtype on cuda (or pinned/
        pageable CPU tensor -> host path).  Returns (phi, grad|None)."""
        import torch
        self._check_pos(pos, "probe")
        if oob is not None and (oob.device.type != "cuda" or oob.element_size() != 8):
            raise SgError(SG_ERR_ARG, "probe: oob must be a CUDA tensor of one 8-byte counter")
        n = int(pos.shape[0])
        dt = pos.dtype
        phi = torch.empty(n, dtype=dt, device=pos.device, pin_memory=(pos.device.type == "cpu"
                                                                        and pos.is_pinned()))
        grad = None
        if want_grad:
            grad = torch.empty((n, 3), dtype=dt, device=pos.device,
                               pin_memory=(pos.device.type == "cpu" and pos.is_pinned()))
        sg_probe(self.handle, n, pos.data_ptr(), phi.data_ptr(),
                 grad.data_ptr() if grad is not None else None,
                 oob.data_ptr() if oob is not None else None, stream)
        return phi, grad

    def relax(self, pos, dp: float, steps: int = 1, h_ratio: float = 1.3, step: float = 0.1,
              max_disp: float = 0.2, surface_offset: float = 0.5, stream=None):
        """SPH relaxation steps (NEXT-2) of a device tensor (n, 3), in place."""
        self._check_pos(pos, "relax", device_only=True)
        sg_relax(self.handle, int(pos.shape[0]), pos.data_ptr(), dp, h_ratio, step, max_disp,
                 surface_offset, steps, stream)
        return pos

    def sign_correct(self, tau: float | None = None, max_sweeps: int = 0, stream=None) -> tuple:
        """Sign-consistency correction (NEXT-3); tau defaults to dx."""
        if tau is None:
            tau = self.info["dx"]
        return sg_sign_correct(self.handle, tau, max_sweeps, stream)

    def clean(self, threshold: float = 0.4, max_rounds: int = 5, h_ratio: float | None = None,
              reinit_iters: int | None = None, cfl: float | None = None, stream=None) -> tuple:
        """Small-feature cleaning (NEXT-3); returns (rounds, raised per round)."""
        w = self.w
        return sg_clean(self.handle, w.h_ratio if h_ratio is None else h_ratio, threshold,
                        w.iters if reinit_iters is None else reinit_iters,
                        w.cfl if cfl is None else cfl, max_rounds, stream)

    def view(self, name: str):
        return view_tensor(self.handle, name)

    def close(self):
        if getattr(self, "handle", None):
            sg_destroy(self.handle)
            self.handle = None

    def close_async(self, stream=None):
        if getattr(self, "handle", None):
            sg_destroy_async(self.handle, stream)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
