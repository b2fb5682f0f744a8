// sg_internal.cuh -- private definitions of libsg (grid handle, launch and
// error plumbing).  Not part of the ABI; see include/sg.h.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sg.h"

namespace sg {

// Analytic geometry, passed by value to the kernels that evaluate f
// (parameter space, ~1.6 KB).
struct Geom {
    int32_t n;       // union primitives (kinds other than SG_LEAK), in order
    int32_t n_leak;  // SG_LEAK post-operations (sign-error balls)
    int32_t kind[SG_MAX_PRIMS];
    double p[SG_MAX_PRIMS][12];
    double leak[SG_MAX_PRIMS][5];  // cx cy cz r margin
    // NEXT-4 closed triangle mesh (device arrays, valid during sg_build);
    // mesh_nt == 0: the union of the primitives is the geometry
    int32_t mesh_nt = 0, mesh_nv = 0;
    const double* mv = nullptr;         // [nv][3] vertices
    const int32_t* mt = nullptr;        // [nt][3] ccw from outside
    const double* mfn = nullptr;        // [nt][3] unit face normals
    const double* men = nullptr;        // [nt][3 edges][3] edge pseudonormals
    const double* mvn = nullptr;        // [nv][3] vertex pseudonormals
    const double* msph = nullptr;       // [nt][4] bounding sphere (centroid, radius)
    const uint32_t* bin_off = nullptr;  // [cells + 1] CSR of triangles per cell
    const uint32_t* bin_tri = nullptr;
    double mesh_rb = 0.0;               // bin radius: exact below it
};

// Grid constants passed by value to every kernel.
// Unsigned division by a grid extent fixed for a launch (Hacker's Delight
// 10-8, "unsigned division by invariant integers"): q = n / d exactly for all
// 32-bit n, as one multiply-high, two adds and two shifts instead of the
// ~20-instruction runtime division (the cell -> (x, y, z) decompositions of
// the build kernels).
struct FastDiv {
    uint32_t d = 1, m = 0, s = 0;
    FastDiv() = default;
    explicit FastDiv(uint32_t dd) : d(dd) {
        if (d > 1) {
            uint32_t l = 0;
            while ((uint64_t(1) << l) < d) ++l;  // ceil(log2 d)
            m = (uint32_t)(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
            s = l - 1;
        }
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (d == 1) return n;
        const uint32_t t = __umulhi(m, n);
        return (t + ((n - t) >> 1)) >> s;
    }
};

struct GridC {
    double lower[3];
    double upper[3];  // lower + n * cell
    double cell;      // l_c
    double dx;        // l_c / 4
    double far;
    double init_scale;
    int32_t n[3];
    int32_t zs_lo, zs_hi;  // stored planes
    int32_t z_lo, z_hi;    // owned planes
    int64_t plane;         // n[0] * n[1]
    double inv_cell, inv_dx;
    int32_t dyadic;        // l_c is a power of two: x / l_c == x * (1 / l_c) exactly
    // fp32 index arithmetic is bit-identical to the fp64 definition when l_c
    // is a power of two, lower = 0 and upper is a float (see sg_probe.cu)
    int32_t idx32;
    FastDiv fdx, fdy;  // division by n[0], n[1] (cell index -> x, y, z)
    float upperf[3];
    float inv_cellf, inv_dxf;
};

struct Error : std::runtime_error {
    sg_status st;
    Error(sg_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

extern std::atomic<uint64_t> g_launches;

void set_last_error(const std::string& m);
void clear_last_error();

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define SG_CUDA(x)                                                  \
    do {                                                            \
        cudaError_t e_ = (x);                                       \
        if (e_ != cudaSuccess) ::sg::throw_cuda(e_, #x, __FILE__, __LINE__); \
    } while (0)

// After every kernel launch: surface launch errors, count the launch.
#define SG_LAUNCHED()                                               \
    do {                                                            \
        SG_CUDA(cudaGetLastError());                                \
        ::sg::g_launches.fetch_add(1, std::memory_order_relaxed);   \
    } while (0)

#define SG_ARG(cond, msg)                                           \
    do {                                                            \
        if (!(cond)) throw ::sg::Error(SG_ERR_ARG, msg);            \
    } while (0)

// NVTX range over one C-ABI call (header-only NVTX v3: free unless a tool
// such as nsys / ncu attaches)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
sg_status guard(F&& f) {
    clear_last_error();
    try {
        f();
        return SG_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.st;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return SG_ERR_OOM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SG_ERR_CUDA;
    }
}

// Stream-ordered device allocation from the library's own pool on the
// current device (memory kept in the pool across grids: its release
// threshold is raised; the device's default pool is left alone).  Free with
// cudaFreeAsync.
void* dalloc(size_t bytes, cudaStream_t s);

// ---- communicator backends (sg_comm.cu) ----
// all-gather: dst = [nranks][bytes], rank r's `src` at offset r * bytes;
// stream-ordered on s (device buffers)
void comm_allgather(const sg_comm* c, const void* src, void* dst, size_t bytes, cudaStream_t s);
// one group of point-to-point transfers, stream-ordered on s; zero-byte ops
// must be left out by both sides
struct P2P {
    int peer;
    bool send;
    void* buf;
    size_t bytes;
};
void comm_group(const sg_comm* c, const P2P* ops, int n, cudaStream_t s);
int comm_rank(const sg_comm* c);
int comm_size(const sg_comm* c);
int comm_kind(const sg_comm* c);  // SG_COMM_NCCL / SG_COMM_LOCAL
// the z-slab plan (sg_slab_plan)
void slab_plan(const int64_t* counts, int32_t nz, int32_t nranks, int32_t rank, sg_plan_t* p,
               int32_t* cuts);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Resident blocks of `kernel` on the current device (SMs x blocks per SM at
// `threads` threads and `smem` dynamic shared bytes): the grid of a
// persistent launch.  Cached per (kernel, device, threads, smem); thread safe.
int resident_blocks(const void* kernel, int threads, size_t smem = 0);
// streaming multiprocessors of the current device (cached per device)
int sm_count();

// NeighbourIndexShift (Lst. 2) for PKG_SIZE = 4, one axis: a
// package-relative data shift s in [-4, 7] maps to the
// neighbour offset o = (s + 4) / 4 in {0, 1, 2} (slot ox + 3 oy + 9 oz of the
// 27-entry row, R-8) and the data index s + 4 - 4 o in that package.  Every
// kernel that crosses a package face goes through this function; the host
// export sg_neighbour_index_shift() runs the same code.
struct Shift {
    int off, data;
};
__host__ __device__ __forceinline__ Shift nb_shift(int s) {
    const int o = (s + 4) >> 2;  // s + 4 >= 0: shift == floor division
    return {o, s + 4 - 4 * o};
}

}  // namespace sg

namespace sg {
struct TPlan;
}

struct sg_grid {
    sg_desc desc;  // as built (the refined layer derives its own from it)
    sg::GridC gc;
    sg::Geom geom;
    int32_t dtype = SG_F32;
    int32_t esz = 4;
    int64_t id_base = 2;
    int64_t n_pkg = 2, n_core = 0, n_inner = 0;
    int64_t ncell_stored = 0;
    // topology: background table, meta, neighbour table
    uint32_t* bg = nullptr;
    uint32_t* meta_cell = nullptr;
    uint8_t* meta_cat = nullptr;
    uint32_t* nb = nullptr;
    // [n_pkg][8]: the six face-neighbour ids of nb (-x, +x, -y, +y, -z, +z;
    // slots 12, 14, 10, 16, 4, 22) + 2 zero pads, one 32 B sector per package:
    // the 7-point sweeps read this instead of their 108 B nb row
    uint32_t* face = nullptr;
    int64_t* plane_first = nullptr;  // [stored planes + 1]
    // tagging bitmasks kept for the sign correction: [tag planes][n1][W]
    uint32_t* cell_core = nullptr;
    uint32_t* cell_neg = nullptr;
    uint32_t* cell_eval = nullptr;  // refined layer: cells under a parent core cell
    int32_t tag_W = 0, zt_lo = 0, zt_hi = 0;
    // fields
    void* phi[2] = {nullptr, nullptr};
    int cur = 0;
    void* grad = nullptr;
    void* normal = nullptr;
    void* kint = nullptr;
    void* gkint = nullptr;
    bool has_grad = false, has_normal = false, has_kint = false;
    double kernel_sum = 0.0;
    int device = 0;
    std::vector<std::pair<void*, size_t>> allocs;
    // owned package range [own_lo, own_hi) in local ids
    int64_t own_lo = 2, own_hi = 2;
    // caller's allocator (sg_build_ex), else the library pool
    bool has_allocator = false;
    sg_allocator allocator{};
    // partition over a communicator (sg_build_ex with comm)
    sg::TPlan* tplan = nullptr;  // two-sweep reinit tiles (sg_tsweep.cu), lazily built

    const sg_comm* comm = nullptr;
    int32_t rank = 0, nranks = 1;
    std::vector<int32_t> cuts;  // [nranks + 1] plane cuts of every rank
    sg_plan_t plan{};           // this rank's plan (halo ranges)
    cudaStream_t comm_stream = nullptr;  // exchanges overlapping interior sweeps
    cudaEvent_t ev_b = nullptr, ev_x = nullptr;
    bool partitioned() const { return comm != nullptr && nranks > 1; }

    void* alloc(size_t bytes, cudaStream_t s) {
        void* p = nullptr;
        if (has_allocator) {
            p = allocator.alloc(bytes ? bytes : 256, (void*)s, allocator.ctx);
            if (!p) throw sg::Error(SG_ERR_OOM, "sg_allocator.alloc returned NULL");
        } else {
            p = sg::dalloc(bytes, s);
        }
        allocs.emplace_back(p, bytes ? bytes : 256);
        return p;
    }
    // return one allocation of alloc() before the grid is destroyed
    void release(void* p, cudaStream_t s) {
        for (size_t i = 0; i < allocs.size(); ++i)
            if (allocs[i].first == p) {
                if (has_allocator)
                    allocator.free(p, allocs[i].second, (void*)s, allocator.ctx);
                else
                    cudaFreeAsync(p, s);
                allocs.erase(allocs.begin() + i);
                return;
            }
    }
    int64_t bytes() const {
        int64_t b = 0;
        for (auto& a : allocs) b += (int64_t)a.second;
        return b;
    }
};

// kernels / launchers implemented per translation unit
namespace sg {
// Two-sweep tile plan of a grid (sg_tsweep.cu): the active packages in Morton
// order of their background cells, cut into tiles of at most kTI packages; a
// tile lists its packages, the packages of its face / edge neighbourhood
// ("halo") with the x-rows of them the two sweeps need, and every slot's six
// face neighbours as tile-local slots.  Device arrays come from the grid's
// allocator; the plan is rebuilt after anything rewrites the face table.
struct TPlan {
    int state = 0;  // 0: not built, 1: ready, -1: not applicable (single sweeps)
    int64_t t_cap = 0;
    uint32_t n_tiles = 0;
    void* arena = nullptr;
    int4* cnt = nullptr;        // [t_cap]: (packages, halo packages, first-sweep halo rows, -)
    uint32_t* ids = nullptr;    // [t_cap][kTCap] global id of each slot
    uint4* lf = nullptr;        // [t_cap][kTCap] face neighbours as slots (8 x u16)
    uint16_t* m2 = nullptr;     // [t_cap][kTCap] halo slot: x-rows to load (bit r)
    uint16_t* comp = nullptr;   // [t_cap][kTComp] first-sweep halo rows (slot << 4 | row)
    uint32_t* ctr = nullptr;    // [2]: tiles emitted, capacity overflow
};
void tplan_invalidate(sg_grid* g, cudaStream_t s);
void tplan_release(sg_grid* g, cudaStream_t s);
bool tsweep_ready(sg_grid* g, cudaStream_t s);  // builds the plan on first use
const void* tsweep_key(const sg_grid* g);
void tsweep_launch(sg_grid* g, int cur, float inv_dx, float dx2, float cdx, float ncfl,
                   cudaStream_t s);

void launch_reinit(sg_grid* g, int32_t iters, double cfl, cudaStream_t s, bool halo = false);
void launch_gradient(sg_grid* g, uint32_t fields, double h_ratio, cudaStream_t s);
void launch_probe(const sg_grid* g, int64_t n, const void* pos, void* phi, void* grad,
                  unsigned long long* oob, cudaStream_t s);
void launch_table1(sg_grid* g, int32_t op, double value, cudaStream_t s);
// refresh the ghost packages of `field` (per_pkg_bytes per package) from the
// neighbour ranks of a partitioned grid (grouped send/recv on s)
void halo_exchange(const sg_grid* g, void* field, size_t per_pkg_bytes, cudaStream_t s);

// NEXT-4 triangle mesh (sg_mesh.cu): device copies, pseudonormals, per-cell
// triangle bins; fills the mesh fields of `g`
struct MeshDev {
    std::vector<void*> allocs;
    uint32_t bin_entries = 0;
};
MeshDev mesh_prepare(const GridC& gc, const sg_geometry* geom, Geom& g, cudaStream_t s);
void mesh_release(MeshDev& m, cudaStream_t s);
void launch_tag_mesh(const GridC& gc, const Geom& g, int32_t W, uint32_t* core_w, uint32_t* neg_w,
                     uint32_t* known_w, cudaStream_t s);
// NEXT-4 multi-resolution: tagging of a layer refined from `parent` (cells
// under a parent core cell evaluated, the others inherit the parent's sign)
struct ParentBits {
    const uint32_t* core;
    const uint32_t* neg;
    int32_t W;  // words per parent row
};
void launch_tag_refine_mesh(const GridC& gc, const Geom& g, int32_t W, ParentBits pb,
                            uint32_t* core_w, uint32_t* neg_w, uint32_t* eval_w, cudaStream_t s);
void launch_phi_init_mesh(const GridC& gc, const Geom& g, const uint32_t* meta_cell,
                          int64_t n_pkg, int32_t dtype, void* phi0, void* phi1, cudaStream_t s);
// coarse sign flood of the sign correction (sg_sign.cu) on tagging bitmasks
// [nz][ny][W]: cells with a known bit keep their neg bit, the others take it
// from the flood; returns the number of sweeps that signed something
int cell_flood(int32_t nx, int32_t W, int32_t ny, int32_t nz, const uint32_t* known, uint32_t* neg,
               cudaStream_t s);
}  // namespace sg
