/*
 * sg.h -- C-ABI of the B200-native contiguous sparse-grid hot path.
 *
 * Method: F. Gu, X. Hu, "Contiguous Storage of Grid Data for Heterogeneous
 * Computing" (arXiv 2512.11473).  Citations "P:<line>" refer to the paper's
 * text (reference PAPER.md), "R-<n>" to the readings listed in DESIGN.md.
 *
 * Data structure:
 *   - a coarse background grid of N[0] x N[1] x N[2] cells of size l_c;
 *   - cells near the surface are activated (core: |f(centre)| < l_c, P:499-502;
 *     inner: not core but a 26-neighbour of a core cell) and own one
 *     data package of 4^3 data points at spacing dx = l_c / 4;
 *   - packages are stored contiguously, ids 2.. in ascending linear cell order
 *     (x fastest, z slowest; R-1); ids 0 and 1 are the singular negative and
 *     positive far-field packages;
 *   - per background cell a u32 table: package id, or 0/1 = inactive far field
 *     of that sign (R-5);
 *   - per package a meta record (linear cell, category) and a
 *     3x3x3 table of neighbour package ids, slot ox + 3 oy + 9 oz
 *     for cell offset (ox-1, oy-1, oz-1) (R-8); singular rows are self;
 *   - field values per package: 64 contiguous values, data index
 *     i + 4 j + 16 k (x fastest, R-9).  Vector fields are component-major
 *     inside a package: [package][component][64], except the gradient, which
 *     is stored interleaved with phi as [package][64][4] (see SG_VIEW_GRAD).
 *
 * Conventions for every call:
 *   - Every function returns sg_status; no C++ exception crosses the ABI.
 *     On failure sg_last_error() returns a thread-local message valid until
 *     the next sg_* call on this thread.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Calls are stream-ordered and asynchronous unless noted.
 *   - Device pointers are plain CUDA device addresses of the current device.
 *   - The grid handle owns all its device memory and frees it in
 *     sg_destroy: allocated through the caller's sg_allocator (sg_build_ex),
 *     else stream-ordered from the library's own memory pool on the device
 *     (a pool separate from the device's default pool; sg_pool_trim returns
 *     its free memory).  Call-scoped scratch always comes from that pool.
 *   - Argument errors are reported before any launch (SG_ERR_ARG); CUDA
 *     errors, including asynchronous ones from earlier launches, surface as
 *     SG_ERR_CUDA at the next call that checks.
 *   - There is no CPU fallback: without a CUDA device every compute call
 *     returns SG_ERR_CUDA.
 */
#ifndef SG_H_
#define SG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 3
#define SG_PKG 4        /* package subdivision, "default by 4"        */
#define SG_MAX_PRIMS 16 /* primitives per geometry                          */

typedef enum {
    SG_OK = 0,
    SG_ERR_ARG = 1,    /* invalid argument (null pointer, pkg != 4, n <= 0, ...) */
    SG_ERR_OOM = 2,    /* device allocation failed                             */
    SG_ERR_CUDA = 3,   /* CUDA runtime error (incl. no device)                 */
    SG_ERR_NCCL = 4,   /* multi-GPU communicator (NCCL missing or a call failed) */
    SG_ERR_STATE = 5,  /* wrong call order, e.g. probing grad before sg_gradient */
    SG_ERR_DOMAIN = 6  /* slab / domain inconsistency                           */
} sg_status;

typedef enum { SG_F32 = 0, SG_F64 = 1 } sg_dtype;

/* Analytic primitives (stand-in for the triangle-mesh SDF of P:516, which is
 * out of scope).  Parameters p[] per kind:
 *   SG_SPHERE      cx cy cz r
 *   SG_SHELL       cx cy cz r_in r_out
 *   SG_BOX         cx cy cz bx by bz        (half extents)
 *   SG_TORUS_X/Y/Z cx cy cz R r             (symmetry axis x / y / z)
 *   SG_TRIPRISM_Z  ax ay bx by cx cy z0 z1  (triangle ccw in xy, extruded in z)
 *   SG_LEAK        cx cy cz r margin        (sign-error region, see below)
 * The union of several primitives is their pointwise min, in order.
 * SG_LEAK entries are not part of the union: they model the sign errors of a
 * triangle-mesh SDF on leaky input as a post-operation on the
 * union value f: f <- -f wherever the point lies strictly inside one of the
 * leak balls ((x-c).(x-c) < r*r, evaluated as ((ex*ex + ey*ey) + ez*ez))
 * and |f| >= margin.  The magnitude is untouched; the build (tagging, table,
 * initial phi) sees the leaky f.  At least one non-leak primitive is needed.  The
 * fp64 evaluation order is fixed and compiled without FMA
 * contraction so that the tagging decision is reproducible bit for bit. */
typedef enum {
    SG_SPHERE = 0,
    SG_SHELL = 1,
    SG_BOX = 2,
    SG_TORUS_X = 3,
    SG_TORUS_Y = 4,
    SG_TORUS_Z = 5,
    SG_TRIPRISM_Z = 6,
    SG_LEAK = 7
} sg_prim_kind;

typedef struct {
    int32_t kind; /* sg_prim_kind */
    int32_t pad;
    double p[12];
} sg_prim;

typedef struct {
    const sg_prim* prims; /* host pointer, n_prims entries (0..SG_MAX_PRIMS)  */
    int32_t n_prims;
    int32_t pad;
    /* NEXT-4: closed triangle mesh (reading R-24).  When
     * n_tris > 0 the mesh's signed distance replaces the union of the
     * primitives (which must then be empty); otherwise these are ignored.
     * verts: host, n_verts x 3 fp64; tris: host, n_tris x 3 vertex indices,
     * counter-clockwise seen from outside.  Copied during sg_build.
     *   f(x) = s |x - q|: q the closest point of the nearest triangle
     *   (smallest squared distance, ties to the lowest index; closest point on
     *   a triangle by its Voronoi regions, Ericson RTCD 5.1.5, fp64 without
     *   FMA), s = sign((x - q) . N) with N the angle-weighted pseudonormal of
     *   the closest feature (Baerentzen & Aanaes): the unit face normal, the
     *   sum of the two adjacent face normals of an edge, or the sum over a
     *   vertex's corners (in triangle order) of corner angle * face normal.
     * The device evaluates it exactly up to 4 l_c from the surface (per-cell
     * triangle bins); the sign of cells farther away comes from the coarse
     * sign flood of sg_sign_correct, seeded by the cells within 4 l_c
     * -- the same sign for a closed mesh.  Out-of-domain
     * neighbour cells take the sign of the nearest in-domain cell.  Mesh
     * geometries: single-domain grids, no SG_LEAK entries, not accepted by
     * sg_plane_counts. */
    const double* verts;
    const int32_t* tris;
    int32_t n_verts;
    int32_t n_tris;
} sg_geometry;

typedef struct {
    double lower[3];   /* domain lower corner                                  */
    double cell;       /* background cell size l_c > 0                         */
    int32_t n[3];      /* background cells per axis, each >= 1; total < 2^32  */
    int32_t pkg;       /* must be SG_PKG (4)                                   */
    int32_t dtype;     /* sg_dtype of every field                              */
    int32_t pad;
    double far;        /* far-field magnitude; 0 -> 4 l_c max(1, init_scale) (R-4) */
    double init_scale; /* initial phi = init_scale * f; 0 -> 1                 */
} sg_desc;

/* z-slab of a multi-GPU partition (whole background planes, R-1).  The rank
 * owns planes [z_lo, z_hi) and additionally stores one ghost plane on each
 * side that lies inside the domain.  id_base is the global package id of the
 * first stored package (2 for the lowest slab); it is the number of active
 * cells in planes below the first stored plane, plus 2.  NULL slab = the
 * whole domain on one GPU. */
typedef struct {
    int32_t z_lo;
    int32_t z_hi;
    int64_t id_base;
} sg_slab;

typedef struct sg_grid sg_grid;

/* ------------------------------------------------- multi-GPU --
 * The paper runs on one device (SYCL); BASELINE north_star
 * partitions the packages over the GPUs of one node in z-slabs of the
 * background grid ("NCCL halo exchange of boundary packages over NVLink each
 * reinitialization iteration and particles binned to their owning rank").
 * A communicator joins one process (one GPU) per rank.  A grid built with a
 * communicator (sg_build_ex) is partitioned: the build all-gathers per-plane
 * package counts and cuts balanced slabs (sg_slab_plan); sg_reinit,
 * sg_gradient and sg_probe then exchange what the slab needs themselves.
 * Every call on such a grid is collective: all ranks call it, in the same
 * order, with the same scalar arguments.  Results equal the single-GPU grid's
 * bit for bit (Jacobi sweeps are order independent; ghosts hold the owner's
 * values). */
typedef struct sg_comm sg_comm;

#define SG_COMM_ID_BYTES 128 /* an NCCL unique id */
#define SG_MAX_RANKS 64

enum { SG_COMM_NCCL = 0, SG_COMM_LOCAL = 1 };

/* Allocator of the grid's device memory.  alloc returns `bytes` of device
 * memory of the current device usable on `stream` (NULL on failure ->
 * SG_ERR_OOM); free releases it (the library calls it once per allocation,
 * stream-ordered on the stream of sg_destroy_async, or after a device
 * synchronisation in sg_destroy).  ctx is passed through. */
typedef struct {
    void* (*alloc)(size_t bytes, void* stream, void* ctx);
    void (*free)(void* ptr, size_t bytes, void* stream, void* ctx);
    void* ctx;
} sg_allocator;

/* sg_gradient field selection */
enum {
    SG_GRAD = 1,   /* grad phi by central difference (Lst. 5)   */
    SG_NORMAL = 2, /* n = grad phi / |grad phi| (0 where |grad phi| = 0)   */
    SG_KINT = 4    /* kernel integrals K, G (reading R-14)      */
};

/* sg_view selectors */
enum {
    SG_VIEW_BG = 0,          /* u32 [stored cells]        background table          */
    SG_VIEW_META_CELL = 1,   /* u32 [n_pkg]               global linear cell index  */
    SG_VIEW_META_CAT = 2,    /* u8  [n_pkg]               0/1 singular, 2 inner, 3 core */
    SG_VIEW_NB = 3,          /* u32 [n_pkg][27]           neighbour package ids     */
    SG_VIEW_PHI = 4,         /* T   [n_pkg][64]           current phi               */
    SG_VIEW_GRAD = 5,        /* T   [n_pkg][64][4]        (phi, d/dx, d/dy, d/dz): the
                                phi of the sg_gradient call and grad phi, one
                                vector per data point (probe layout)            */
    SG_VIEW_NORMAL = 6,      /* T   [n_pkg][3][64]        normal                    */
    SG_VIEW_KINT = 7,        /* T   [n_pkg][64]           K                         */
    SG_VIEW_GKINT = 8,       /* T   [n_pkg][3][64]        G = grad K                */
    SG_VIEW_PLANE_FIRST = 9, /* i64 [stored planes + 1]   first package id per plane */
    SG_VIEW_PHI_NEXT = 10,   /* T   [n_pkg][64]           reinit scratch buffer     */
    /* per-cell bitmasks of the tagging pass, kept for the sign correction:
     * u32 [tag planes][n1][ceil(n0 / 32)], bit x % 32 of word x / 32 is cell
     * x of that row; tag planes = stored planes plus one on each side that
     * lies in the domain (sg_info zs_lo/zs_hi widened by one, clipped) */
    SG_VIEW_CELL_CORE = 11,  /* |f(centre)| < l_c                                 */
    SG_VIEW_CELL_NEG = 12,   /* f(centre) < 0 (after sg_sign_correct: corrected)  */
    SG_VIEW_FACE = 13        /* u32 [n_pkg][8]            face table: entries 0..5 are
                                neighbour slots 12, 14, 10, 16, 4, 22 (-x, +x, -y,
                                +y, -z, +z), 6..7 zero -- the 32 B row the 7-point
                                sweeps read instead of the 108 B neighbour row */
};

typedef struct {
    void* ptr;         /* device pointer, non-owning; NULL if not computed yet */
    int64_t shape[3];  /* unused trailing dims = 1                             */
    int32_t ndim;
    int32_t elem_size; /* bytes per element                                    */
    int32_t dtype;     /* 0 f32, 1 f64, 2 u32, 3 u8, 4 i64                     */
    int32_t pad;
} sg_view_t;

typedef struct {
    int64_t n_pkg;        /* packages stored, incl. the two singular ones      */
    int64_t n_core;       /* stored core packages                              */
    int64_t n_inner;      /* stored inner packages                             */
    int64_t id_base;      /* global id of local id 2 (sg_slab.id_base)         */
    int32_t dtype;
    int32_t z_lo, z_hi;   /* owned background planes                           */
    int32_t zs_lo, zs_hi; /* stored background planes (owned + ghosts)         */
    int32_t pad;
    double dx;            /* data spacing l_c / 4                              */
    double far;           /* far-field magnitude                               */
    double kernel_sum;    /* S = sum of kernel weights of the last SG_KINT     */
    int32_t has_grad, has_normal, has_kint, phi_cur;
    int64_t device_bytes; /* bytes held by the grid                            */
    int64_t own_lo;       /* owned local package ids [own_lo, own_hi); ghost   */
    int64_t own_hi;       /* packages are [2, own_lo) and [own_hi, n_pkg)      */
    int32_t rank;         /* communicator rank / size (0 / 1 without one)      */
    int32_t nranks;
} sg_info_t;

/* The z-slab plan of one rank (host only).  Local ids: 0, 1 singular, then
 * the stored packages in global id order (global id = local - 2 + id_base).
 * Halo ranges are local id ranges [a, b) of whole background planes:
 *   send_lo = first owned plane (-> rank - 1), send_hi = last owned plane
 *   (-> rank + 1), recv_lo = ghost plane below (<- rank - 1), recv_hi = ghost
 *   plane above (<- rank + 1); (0, 0) where there is no such neighbour. */
typedef struct {
    int32_t z_lo, z_hi;    /* owned planes                                   */
    int32_t zs_lo, zs_hi;  /* stored planes (owned + one ghost plane per side) */
    int64_t id_base;       /* global id of local id 2                         */
    int64_t n_pkg;         /* stored packages + 2                             */
    int64_t own_lo, own_hi;
    int64_t send_lo[2], send_hi[2], recv_lo[2], recv_hi[2];
} sg_plan_t;

/* ---------------------------------------------------------------- calls -- */

/* A fresh communicator id (SG_COMM_ID_BYTES bytes): rank 0 creates it and
 * sends it to every rank (e.g. torch.distributed.broadcast_object_list).
 * NCCL is loaded at run time (dlopen "libnccl.so.2"; a copy the process
 * already loaded -- PyTorch's -- is reused).  SG_ERR_NCCL if unavailable. */
sg_status sg_comm_unique_id(void* id);

/* Collective over `nranks` processes: rank `rank` joins the NCCL
 * communicator of `id` on the current device (NVLink / NVSwitch transport
 * within the node).  0 <= rank < nranks <= SG_MAX_RANKS. */
sg_status sg_comm_create(const void* id, int32_t rank, int32_t nranks, sg_comm** out);

/* An in-process group of nranks communicators on the current device,
 * written to comms[0 .. nranks).  Ranks exchange by device-to-device copies
 * with the NCCL communicator's semantics (stream-ordered grouped send/recv,
 * all-gather); each rank must be driven by its own host thread, since calls
 * on partitioned grids are collective and block until the peers arrive.
 * Emulates P slabs on one GPU (tests); every multi-GPU code path of the
 * library runs unchanged on it. */
sg_status sg_comm_create_local(int32_t nranks, sg_comm** comms);

/* rank, size and kind (SG_COMM_NCCL / SG_COMM_LOCAL); outputs may be NULL */
sg_status sg_comm_info(const sg_comm* comm, int32_t* rank, int32_t* nranks, int32_t* kind);

/* Asynchronous communicator errors (ncclCommGetAsyncError: a peer failed or
 * a transfer broke after its call returned): SG_OK, or SG_ERR_NCCL with the
 * NCCL message in sg_last_error().  The in-process communicator has none. */
sg_status sg_comm_check(const sg_comm* comm);

/* Destroy a communicator (after every grid built on it is destroyed). */
void sg_comm_destroy(sg_comm* comm);

/* Host-only (no device use): the plan of `rank` among `nranks` from the
 * per-plane package counts of the whole domain, counts[0 .. nz): cuts as
 * sg_balanced_cuts (written to cuts[0 .. nranks], may be NULL), stored planes,
 * global id base, local package count, owned range and halo ranges
 * (sg_plan_t).  The partitioned build uses exactly this function.
 * SG_ERR_ARG if nranks < 1, nz < nranks or rank outside [0, nranks). */
sg_status sg_slab_plan(const int64_t* counts, int32_t nz, int32_t nranks, int32_t rank,
                       sg_plan_t* plan, int32_t* cuts);

typedef struct {
    const sg_slab* slab;           /* explicit slab (no comm), NULL = whole domain   */
    const sg_comm* comm;           /* partition over the communicator's ranks
                                      (slab must be NULL); NULL = one GPU          */
    const sg_allocator* allocator; /* grid memory; NULL = the library's pool         */
} sg_build_opts;

/* sg_build with options (opts may be NULL = sg_build(desc, geom, NULL)).
 * With a communicator the call is collective: every rank counts the packages
 * of a uniform range of planes, the counts are all-gathered (one host
 * synchronisation: it also yields this rank's package count, so the build
 * itself does not read one back), and the rank builds the slab of
 * sg_slab_plan with one ghost plane per side.  Mesh geometries are
 * single-domain only.  Errors as sg_build, SG_ERR_NCCL. */
sg_status sg_build_ex(const sg_desc* desc, const sg_geometry* geom, const sg_build_opts* opts,
                      void* stream, sg_grid** out);

/* Return the free memory of the library's pool on the current device to the
 * system (grid memory in use is kept). */
sg_status sg_pool_trim(void);

/* Build the sparse grid for `geom` (P:499-526 steps 1-5, single layer):
 *   K1 core tagging at background-cell centres (fp64),
 *   K2 inner tagging + ordered compaction (ids in linear cell order),
 *   K3 27-neighbour table (out-of-domain neighbours: 0/1 by the sign of f at
 *      the virtual cell centre, R-6),
 *   K4 initial phi = init_scale * f at the 64 data points of each package,
 *      rounded to dtype; singular packages hold -far / +far.
 * One host synchronisation reads back the package count (replaces the
 * paper's USM shared scalar).  A repeated build of the same
 * (desc, geometry) in the process (no slab, mesh or communicator) sizes its
 * arrays from the previous build's counts and reads the count back only
 * after all its work is queued (checked; a mismatch rebuilds without the
 * hint; SG_BUILD_HINT=0 disables this).  slab may be NULL.  On success *out
 * owns the grid.  Errors: SG_ERR_ARG (null pointers, pkg != 4, n < 1,
 * cell <= 0, n_prims outside 1..SG_MAX_PRIMS, unknown kind or dtype, more than
 * 2^32 - 3 stored packages or 2^32 stored data points), SG_ERR_DOMAIN (slab
 * outside the domain), SG_ERR_OOM, SG_ERR_CUDA. */
sg_status sg_build(const sg_desc* desc, const sg_geometry* geom, const sg_slab* slab,
                   void* stream, sg_grid** out);

/* NEXT-4 multi-resolution ("several layers with successively
 * doubled resolutions are established ... subsequent layers that each with
 * doubled resolution are initialized based on the preceding coarser layer";
 * "For successive layers, only the cells covered by the coarse
 * core cells will be evaluated"): build the layer with cell size
 * parent.cell / 2 and 2 n cells per axis (same lower corner, dtype,
 * init_scale and far setting) of `geom` from `parent`.  Cells under a parent
 * core cell are evaluated; every other cell takes its parent cell's sign
 * (after sg_sign_correct on the parent: the corrected sign).  The result is
 * the grid a direct sg_build at the finer resolution gives: a fine core cell
 * (|f| < l_f) always has a core parent (|f(parent centre)| < l_f +
 * sqrt(3)/2 l_f < 2 l_f), and a non-core parent cell has one sign over its
 * whole cell.  For a mesh geometry no cell beyond the bin radius is ever
 * evaluated, so no sign flood runs on refined layers.  Single-domain parent
 * grids; the parent must stay alive during the call.  Errors as sg_build. */
sg_status sg_build_refined(const sg_grid* parent, const sg_geometry* geom, void* stream,
                           sg_grid** out);

/* `iters` Jacobi sweeps of upwind Godunov reinitialisation on every active
 * data point (reading R-12; phi' = phi - cfl dx s (|grad phi|_G - 1)),
 * double-buffered; inactive and singular data stay unchanged.  Neighbours
 * across package faces are reached through the neighbour table (Lst. 2).
 * iters >= 0, 0 < cfl <= 0.5.  Asynchronous.  On a slab grid built with an
 * explicit sg_slab only the owned packages are updated; the caller refreshes
 * the ghost packages of the current buffer (SG_VIEW_PHI, contiguous id
 * ranges, see sg_info) between sweeps, i.e. calls sg_reinit(grid, 1, ...)
 * once per exchange.  On a grid partitioned over a communicator the call is
 * collective and refreshes the ghosts itself, once per 4 sweeps (the ghost
 * reuse of sg_reinit_halo): in each group of up to 4 sweeps the first ones
 * run over owned + ghost packages, the last one updates the two boundary
 * planes first and sends them (grouped send/recv on an internal stream,
 * into the neighbours' ghost planes) while it updates the interior
 * packages. */
sg_status sg_reinit(sg_grid* grid, int32_t iters, double cfl, void* stream);

/* The same sweeps over every stored package, owned and ghost (a9 with ghost
 * reuse).  The ghost plane of a slab is 4 data points deep and a
 * sweep's dependence cone grows one point per sweep: the ghost packages go
 * wrong from their outer face inward (their out-of-slab neighbours are far
 * constants), one point per sweep, so after an exchange of the current
 * buffer up to 4 sweeps keep every owned package exact -- one exchange per 4
 * sweeps instead of one per sweep.  On a single-domain grid identical to
 * sg_reinit. */
sg_status sg_reinit_halo(sg_grid* grid, int32_t iters, double cfl, void* stream);

/* Derived fields from the current phi: any OR of SG_GRAD, SG_NORMAL, SG_KINT.
 * h_ratio = h / dx of the Wendland C2 kernel, in [0.5, 2] (stencil radius
 * <= 3 < 4, so every tap stays in the 27-neighbourhood).  Asynchronous.
 * Partitioned grid: collective; the (phi, grad) ghost planes are exchanged
 * afterwards (probe corners may lie in a ghost plane). */
sg_status sg_gradient(sg_grid* grid, uint32_t fields, double h_ratio, void* stream);

/* Grid-particle coupling (reading R-15): for each of n positions
 * (row-major n x 3, grid dtype) look up the containing background cell; an
 * inactive cell yields its far constant, an active one the trilinear
 * interpolation of phi (and of grad phi if `grad` != NULL) over the 8
 * surrounding data points, fetched through the package's neighbour row with
 * NeighbourIndexShift (Lst. 2).  Positions outside the stored domain or NaN
 * return (+far, 0) and increment *oob_count (device u64, may be NULL).
 * pos / phi (n) / grad (n x 3) may be device pointers (asynchronous) or host
 * pointers, pinned or pageable (then the call stages them through device
 * buffers in pipelined chunks and returns after the results are in host
 * memory).  grad != NULL requires a prior sg_gradient with SG_GRAD
 * (SG_ERR_STATE otherwise).  n == 0 is a no-op.
 * Partitioned grid (collective, any n >= 0 per rank): each rank passes its
 * own particles; K9 bins them to the rank owning their background plane
 * (stable order; out-of-domain / NaN positions stay and count as OOB), the
 * per-rank counts are all-gathered (one host synchronisation), positions go
 * to their owners and results come back with grouped send/recv, and the
 * results are returned in the caller's order -- bit-identical to a
 * single-GPU probe. */
sg_status sg_probe(const sg_grid* grid, int64_t n, const void* pos, void* phi, void* grad,
                   unsigned long long* oob_count, void* stream);

/* Table-1 workloads of the paper, on the current phi:
 *   op 0 "sequential": phi += value at every active data point (in place;
 *        on a slab grid the ghost packages too, so they stay equal to their
 *        owner's values); grad / normal / K / G become stale (has_* cleared);
 *   op 1 "stencil": out = 7-point Laplacian of phi at every active data point
 *        ((sum of 6 neighbours - 6 phi) / dx^2), written to the active
 *        packages of the SG_VIEW_PHI_NEXT buffer (phi is unchanged; the
 *        singular packages of that buffer keep the far constants). */
sg_status sg_table1(sg_grid* grid, int32_t op, double value, void* stream);

/* SPH particle relaxation against the level set (NEXT-2; "the
 * integral field is interpolated by bi- or tri-linear interpolation to the
 * particle's position and used in the form of surface force to drive the
 * particle"; force law and bounding are reading R-21):
 *   a_i  = -2 ( sum_{j != i} V grad W(x_i - x_j) - G(x_i) ),  V = dp^3,
 *          Wendland C2 with h = h_ratio dp (pairs from a cell-linked list),
 *          G = the kernel-gradient integral field interpolated trilinearly;
 *   dx_i = step dp^2 a_i, its length clamped to max_disp dp;
 *   bounding: with phi, grad phi probed at the moved position, a particle with
 *          phi > -surface_offset dp moves by -(phi + surface_offset dp) n,
 *          n = grad phi / |grad phi|.
 * One call performs `steps` Jacobi steps (positions double-buffered).  pos is
 * a device array n x 3 of the grid dtype, updated in place; particles outside
 * the stored domain are left unchanged.  Requires sg_gradient with SG_GRAD and
 * SG_KINT (SG_ERR_STATE otherwise).  Pair sums within a cell follow an atomic
 * binning order: results are reproducible to rounding, not bit for bit. */
typedef struct {
    double dp;             /* particle spacing (> 0)                         */
    double h_ratio;        /* h / dp of the pair kernel, in [0.5, 2]          */
    double step;           /* dimensionless step (displacement = step dp^2 a) */
    double max_disp;       /* clamp of the displacement, in units of dp       */
    double surface_offset; /* bounding offset, in units of dp                 */
    int32_t steps;         /* >= 0                                            */
    int32_t pad;
} sg_relax_params;

sg_status sg_relax(sg_grid* grid, int64_t n, void* pos, const sg_relax_params* params,
                   void* stream);

/* Sign-consistency correction (NEXT-3; "only the sign of level
 * set for those data points very close to the surface is directly used,
 * those at other locations are obtained by a two-step diffusion process from
 * the near interface to the entire domain.  The first coarse step is on the
 * mesh cells and the second refined one is on the data packages"; reading
 * R-22).  Both steps are synchronous (Jacobi) sweeps of one majority rule:
 * an unsigned site with at least one signed face neighbour takes the sign
 * held by more of its signed face neighbours (a tie leaves it unsigned for
 * that sweep); a step ends at the first sweep that signs nothing.
 *   coarse: sites = background cells of the domain (6 face neighbours inside
 *     the domain).  Core cells keep the sign of f at their centre; all other
 *     cells start unsigned.  Afterwards the table entry of every inactive
 *     cell (0/1) and every singular entry of the neighbour table that refers
 *     to an in-domain cell are rewritten from the corrected cell signs
 *     (entries for out-of-domain neighbours, R-6, are kept); cells never
 *     reached keep their sign.
 *   refined: sites = data points of the active packages (6 face neighbours,
 *     across package faces through the neighbour table; a neighbour point in
 *     a singular package is signed: package 0 negative, 1 positive).  Points
 *     with |phi| < tau (compared in the grid dtype) keep their sign; all
 *     other active points start unsigned.  Finally phi <- -|phi| / +|phi| at
 *     every signed point; points never reached keep phi.
 * On a layer built by sg_build_refined the coarse step revisits only the
 * cells evaluated on that layer (under a parent core cell): every other cell
 * carries its parent's sign and starts signed ("only on the coarsest
 * layer all cells are evaluated.  For refined layers, the operation is
 * limited to inner cells or data packages").
 * tau > 0 (typically dx).  max_sweeps > 0 caps each step, <= 0 means no cap.
 * sweeps (host int32[2], may be NULL) receives the number of sweeps of the
 * coarse and the refined step that signed at least one site.  Operates on
 * the current phi buffer in place and clears has_grad/has_normal/has_kint.
 * Single-domain grids only (SG_ERR_ARG for a slab grid).  The host
 * synchronises with `stream` once per batch of sweeps (convergence test). */
sg_status sg_sign_correct(sg_grid* grid, double tau, int32_t max_sweeps, int32_t* sweeps,
                          void* stream);

/* Small-feature cleaning (NEXT-3; "we reimplemented the
 * level-set cleaning algorithms (only on the finest layer) in Ref.
 * [yu2023level] so that it can be run on GPU"; the criterion is not restated
 * in the paper, reading R-23 takes the stand-in of SPEC S:476-484).  Rounds
 * of:
 *   1. K = kernel integral of the current phi (as sg_gradient SG_KINT with
 *      h_ratio; S = sum of the kernel weights, so K / S is the fraction of
 *      the kernel support inside the body);
 *   2. every active data point inside the body within dx of the surface
 *      (-dx < phi < 0) with K < threshold * S (compared in the grid dtype)
 *      is raised to phi = +dx (the thin feature is carved away); if no point
 *      was raised the call ends;
 *   3. reinit_iters reinitialisation sweeps (sg_reinit with cfl).
 * At most max_rounds rounds.  modified (host int64[max_rounds], may be NULL)
 * receives the number of raised points per round (0 for rounds not run);
 * rounds (may be NULL) the number of rounds that raised something.  The host
 * synchronises with `stream` once per round.  Afterwards K / G
 * (SG_VIEW_KINT) describe the final phi only if the last round raised
 * nothing; grad / normal are stale.  Single-domain grids only (SG_ERR_ARG
 * for a slab grid); h_ratio in [0.5, 2], threshold in [0, 1], cfl in
 * (0, 0.5]. */
sg_status sg_clean(sg_grid* grid, double h_ratio, double threshold, int32_t reinit_iters,
                   double cfl, int32_t max_rounds, int32_t* rounds, int64_t* modified,
                   void* stream);

sg_status sg_info(const sg_grid* grid, sg_info_t* info);
sg_status sg_view(const sg_grid* grid, int32_t what, sg_view_t* view);

/* Release the grid.  sg_destroy synchronises the device first (safe from any
 * stream); sg_destroy_async frees stream-ordered on `stream` (the caller
 * guarantees no other stream still uses the grid). */
void sg_destroy(sg_grid* grid);
sg_status sg_destroy_async(sg_grid* grid, void* stream);

/* Host-only helper for the z-slab partition (no device use): given per-plane
 * package counts counts[0..nz) choose nranks contiguous slabs with cut planes
 * cuts[0..nranks] (cuts[0] = 0, cuts[nranks] = nz) so that each rank's count
 * is as close as possible to total/nranks: cut r is the smallest plane z with
 * prefix(z) >= r*total/nranks (ties go to the lowest plane), clamped so every
 * slab has at least one plane when nz >= nranks.  Returns SG_ERR_ARG if
 * nranks < 1 or nz < nranks. */
sg_status sg_balanced_cuts(const int64_t* counts, int32_t nz, int32_t nranks, int32_t* cuts);

/* Per-plane package counts of background planes [z_lo, z_hi) of the whole
 * domain (tagging only, no package storage): counts is a device i64 array of
 * z_hi - z_lo entries.  Used to balance the slabs before sg_build. */
sg_status sg_plane_counts(const sg_desc* desc, const sg_geometry* geom, int32_t z_lo,
                          int32_t z_hi, int64_t* counts, void* stream);

/* NeighbourIndexShift of Lst. 2 for PKG_SIZE = 4, host-callable
 * (no device use; the kernels inline the same function): for a
 * package-relative data shift per axis, shift[k] in [-4, 7] (SPEC S:167-171,
 * "nearest-neighbour access"), writes offset[k] = (shift[k] + 4) / 4 in
 * {0, 1, 2} and data[k] = shift[k] + 4 - 4 offset[k] in [0, 4) (either output
 * may be NULL) and returns the neighbour-table slot ox + 3 oy + 9 oz (R-8);
 * returns -1 (outputs unspecified) if shift is NULL or a component is out
 * of range. */
int32_t sg_neighbour_index_shift(const int32_t* shift, int32_t* offset, int32_t* data);

const char* sg_last_error(void);
int32_t sg_abi_version(void);
/* Number of device kernels this library has launched in this process. */
uint64_t sg_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SG_H_ */
