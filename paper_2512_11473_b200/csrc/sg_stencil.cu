// sg_stencil.cu -- package sweeps: reinitialisation (K5), gradient/normal
// (K6), kernel integrals (K7) and the Table-1 workloads.
//
// Execution pattern = the paper's MeshPackageDynamics / package_for (Lst. 4,
// P:380-395): every kernel runs over the contiguous id range of active
// packages; neighbour data across package faces is reached through the
// 27-entry neighbour table with NeighbourIndexShift (Lst. 2):
//   nb_off = (shift + 4) / 4,  data = shift + 4 - 4 nb_off.
//
// Thread mapping of K5/K6/Table-1: 16 threads per package, thread r owns the
// x-row (j, k) = (r & 3, r >> 2), i.e. 4 consecutive values = one 16 B (fp32)
// vector load/store.  Rows of the +-y / +-z neighbours are whole vectors
// (inside the package, or row j=3/0, k=3/0 of the face neighbour); the +-x
// neighbours of the row ends are single values of the x-face neighbours.
// The six face-neighbour ids are loaded once per package by lanes 0..5 of the
// 16-lane group and broadcast with warp shuffles.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "sg_internal.cuh"
#include "sg_godunov.cuh"

namespace sg {

// ------------------------------------------------------------ row access --

__device__ __forceinline__ void ld_row(const float* __restrict__ p, float (&r)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    r[0] = v.x;
    r[1] = v.y;
    r[2] = v.z;
    r[3] = v.w;
}
__device__ __forceinline__ void ld_row(const double* __restrict__ p, double (&r)[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    r[0] = a.x;
    r[1] = a.y;
    r[2] = b.x;
    r[3] = b.y;
}
__device__ __forceinline__ void ld_row_s(const float* p, float (&r)[4]) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
}
__device__ __forceinline__ void ld_row_s(const double* p, double (&r)[4]) {
    const double2 a = reinterpret_cast<const double2*>(p)[0];
    const double2 b = reinterpret_cast<const double2*>(p)[1];
    r[0] = a.x; r[1] = a.y; r[2] = b.x; r[3] = b.y;
}
__device__ __forceinline__ void st_row(float* p, const float (&r)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
}
__device__ __forceinline__ void st_row(double* p, const double (&r)[4]) {
    reinterpret_cast<double2*>(p)[0] = make_double2(r[0], r[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(r[2], r[3]);
}

// The six face neighbours r = 0..5 (-x, +x, -y, +y, -z, +z) are neighbour-
// table slots ox + 3 oy + 9 oz = {12, 14, 10, 16, 4, 22} (Lst. 2 offsets,
// R-8); the sweeps read them from the compact face table (sg_grid::face),
// entry r of a package's 32 B row.

// The 7-point cross of one x-row: own row c, rows ym/yp/zm/zp and the two
// x-end values xm/xp.  Lst. 2 with shifts -1 and 4 (the only ones a
// radius-1 stencil produces): shift -1 -> (offset 0, data 3), 4 -> (2, 0).
template <class T>
struct Cross {
    T c[4], ym[4], yp[4], zm[4], zp[4];
    T xm, xp;
};

// `face`: the grid's compact face table ([pkg][8], sg_grid::face)
template <class T>
__device__ __forceinline__ bool load_cross(const T* __restrict__ in,
                                           const uint32_t* __restrict__ face, int64_t pkg,
                                           bool valid, Cross<T>& x) {
    const int r = threadIdx.x & 15;
    const int j = r & 3, k = r >> 2;
    uint32_t f = 0;
    if (valid && r < 6) f = __ldg(face + pkg * 8 + r);
    const int base = threadIdx.x & 16;
    const uint32_t nxm = __shfl_sync(0xffffffffu, f, base + 0);
    const uint32_t nxp = __shfl_sync(0xffffffffu, f, base + 1);
    // a lane reads the -y face only for j = 0, the +y face only for j = 3 (z:
    // k = 0 / 3): one shuffle each for its y and z neighbour
    const uint32_t ny = __shfl_sync(0xffffffffu, f, base + (j == 0 ? 2 : 3));
    const uint32_t nz = __shfl_sync(0xffffffffu, f, base + (k == 0 ? 4 : 5));
    if (!valid) return false;
    // 32-bit element offsets (sg_build rejects grids of >= 2^32 data points)
    const uint32_t b0 = (uint32_t)pkg * 64u, by = ny * 64u, bz = nz * 64u;
    ld_row(in + (b0 + 4 * r), x.c);
    ld_row(in + (j > 0 ? b0 + 4 * (r - 1) : by + 4 * (3 + 4 * k)), x.ym);
    ld_row(in + (j < 3 ? b0 + 4 * (r + 1) : by + 4 * (0 + 4 * k)), x.yp);
    ld_row(in + (k > 0 ? b0 + 4 * (r - 4) : bz + 4 * (j + 12)), x.zm);
    ld_row(in + (k < 3 ? b0 + 4 * (r + 4) : bz + 4 * j), x.zp);
    x.xm = __ldg(in + (nxm * 64u + 4 * r + 3));
    x.xp = __ldg(in + (nxp * 64u + 4 * r));
    return true;
}

// K5 -- reinitialisation sweep over packages [lo, hi).  Eight threads per
// package; thread (j, k), k in {0, 1}, owns the two x-rows (j, k) and
// (j, k + 2), which share their middle z-row (j, k + 1): 9 row loads + 4
// x-end values for 8 points.  The six face-neighbour ids are loaded by six
// lanes of the 8-lane group and broadcast with shuffles (Lst. 2 with shifts
// -1 -> (offset 0, data 3) and 4 -> (offset 2, data 0)).
// The 7-point cross of the two x-rows (j, k) and (j, k + 2) of one package
template <class T>
struct Cross2 {
    T c0[4], c1[4], zlo[4], zmid[4], zhi[4], ym0[4], yp0[4], ym1[4], yp1[4];
    T xm0, xp0, xm1, xp1;
};

// The four 8-lane groups of a warp hold consecutive packages pkg0 .. pkg0+3
// (k_sweep), and lane (j, k) of every group owns the same rows (j, k), (j, k+2).
// When the x-face neighbour of a package is the next (previous) id -- an
// x-run of active cells, the common case -- its x = 0 (x = 3) values are
// already in the registers of the same lane of the next (previous) group:
// they come by a shuffle of 8 lanes instead of four scalar loads, which cut
// 16-of-256-byte sector fetches from the L2.  `next_ok`: package pkg + 1 is
// processed by the next group in this iteration (pkg + 1 < hi).
// O32: element offsets fit in 32 bits (n_pkg * 64 < 2^32, every grid up to
// ~4.5x C5): one 32-bit select + one wide multiply-add per load address
// instead of a 64-bit pointer select
template <class T, bool O32 = true>
__device__ __forceinline__ void load_cross2(const T* __restrict__ in, uint32_t pkg, bool valid,
                                            bool next_ok, uint32_t f, int j, int k,
                                            Cross2<T>& x) {
    using Off = typename std::conditional<O32, uint32_t, size_t>::type;
    const int base = threadIdx.x & 24;
    const int grp = (threadIdx.x >> 3) & 3;
    const uint32_t nxm = __shfl_sync(0xffffffffu, f, base + 0);
    const uint32_t nxp = __shfl_sync(0xffffffffu, f, base + 1);
    // a lane reads the -y face only for j = 0, the +y face only for j = 3,
    // the -z face only for k = 0 and the +z face only for k = 1: one shuffle
    // each for "its" y and z neighbour (lanes j = 1, 2 take an unused id)
    const uint32_t ny = __shfl_sync(0xffffffffu, f, base + (j == 0 ? 2 : 3));
    const uint32_t nz = __shfl_sync(0xffffffffu, f, base + (k == 0 ? 4 : 5));
    const bool sh_m = grp > 0 && nxm == pkg - 1;
    const bool sh_p = grp < 3 && next_ok && nxp == pkg + 1;
    if (valid) {
        const Off b0 = (Off)pkg * 64, by = (Off)ny * 64, bz = (Off)nz * 64;
        const int r0 = j + 4 * k, r1 = r0 + 8;
        ld_row(in + (b0 + 4 * r0), x.c0);
        ld_row(in + (b0 + 4 * r1), x.c1);
        ld_row(in + (b0 + 4 * (r0 + 4)), x.zmid);
        ld_row(in + (k == 0 ? bz + 4 * (j + 12) : b0 + 4 * j), x.zlo);
        ld_row(in + (k == 0 ? b0 + 4 * (j + 12) : bz + 4 * j), x.zhi);
        ld_row(in + (j > 0 ? b0 + 4 * (r0 - 1) : by + 4 * (3 + 4 * k)), x.ym0);
        ld_row(in + (j < 3 ? b0 + 4 * (r0 + 1) : by + 4 * (4 * k)), x.yp0);
        ld_row(in + (j > 0 ? b0 + 4 * (r1 - 1) : by + 4 * (3 + 4 * (k + 2))), x.ym1);
        ld_row(in + (j < 3 ? b0 + 4 * (r1 + 1) : by + 4 * (4 * (k + 2))), x.yp1);
        if (!sh_m) {
            x.xm0 = __ldg(in + ((Off)nxm * 64 + 4 * r0 + 3));
            x.xm1 = __ldg(in + ((Off)nxm * 64 + 4 * r1 + 3));
        }
        if (!sh_p) {
            x.xp0 = __ldg(in + ((Off)nxp * 64 + 4 * r0));
            x.xp1 = __ldg(in + ((Off)nxp * 64 + 4 * r1));
        }
    }
    // every lane takes part (the caller's trip count is warp-uniform)
    const T m0 = __shfl_up_sync(0xffffffffu, x.c0[3], 8);
    const T m1 = __shfl_up_sync(0xffffffffu, x.c1[3], 8);
    const T p0 = __shfl_down_sync(0xffffffffu, x.c0[0], 8);
    const T p1 = __shfl_down_sync(0xffffffffu, x.c1[0], 8);
    if (sh_m) {
        x.xm0 = m0;
        x.xm1 = m1;
    }
    if (sh_p) {
        x.xp0 = p0;
        x.xp1 = p1;
    }
}

// Persistent package sweep: an 8-lane group takes packages pkg, pkg + G, ...;
// the face ids of the next package are loaded while the current one is
// processed, so the face-row gathers do not wait on the face table.
// Op(x, pkg, r0, r1) consumes the cross of rows r0 = j + 4k and r1 = r0 + 8.
template <class T, class Op, bool O32 = true>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 4 : 2) k_sweep(const T* __restrict__ in,
                                               const uint32_t* __restrict__ face, uint32_t lo,
                                               uint32_t hi, Op op) {
    const uint32_t G = gridDim.x * 32u;  // package groups in flight
    uint32_t pkg = lo + ((blockIdx.x * 256u + threadIdx.x) >> 3);
    const int g8 = threadIdx.x & 7;
    const int j = g8 & 3, k = g8 >> 2;
    // warp-uniform trip count: the warp's 4 groups have consecutive ids
    const uint32_t wfirst = lo + ((blockIdx.x * 256u + (threadIdx.x & ~31u)) >> 3);
    uint32_t f = 0;
    if (pkg < hi && g8 < 6) f = __ldg(face + (size_t)pkg * 8 + g8);
    for (uint32_t w0 = wfirst; w0 < hi; w0 += G) {
        const uint32_t nxt = pkg + G;
        uint32_t fn = 0;
        if (nxt < hi && g8 < 6) fn = __ldg(face + (size_t)nxt * 8 + g8);
        Cross2<T> x;
        const bool valid = pkg < hi;
        load_cross2<T, O32>(in, pkg, valid, pkg + 1 < hi, f, j, k, x);
        if (valid) op(x, pkg, j + 4 * k, j + 4 * k + 8);
        pkg = nxt;
        f = fn;
    }
}

// K5 -- one Jacobi Godunov sweep (O7, reading R-12)
template <class T>
struct ReinitOp {
    T* out;
    StC<T> c;
    __device__ __forceinline__ void operator()(const Cross2<T>& x, uint32_t pkg, int r0,
                                               int r1) const {
        T o0[4], o1[4];
        if constexpr (std::is_same<T, float>::value) {
            godunov_row(x.c0, x.xm0, x.xp0, x.ym0, x.yp0, x.zlo, x.zmid, c, o0);
            godunov_row(x.c1, x.xm1, x.xp1, x.ym1, x.yp1, x.zmid, x.zhi, c, o1);
        } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            o0[i] = godunov(x.c0[i], i > 0 ? x.c0[i - 1] : x.xm0, i < 3 ? x.c0[i + 1] : x.xp0,
                            x.ym0[i], x.yp0[i], x.zlo[i], x.zmid[i], c);
            o1[i] = godunov(x.c1[i], i > 0 ? x.c1[i - 1] : x.xm1, i < 3 ? x.c1[i + 1] : x.xp1,
                            x.ym1[i], x.yp1[i], x.zmid[i], x.zhi[i], c);
        }
        }
        T* O = out + (size_t)pkg * 64;
        st_row(O + 4 * r0, o0);
        st_row(O + 4 * r1, o1);
    }
};

// grid size of a persistent sweep: resident blocks, at most the work
template <class K>
static unsigned persistent_blocks(K kernel, int64_t packages) {
    return (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(packages * 8, 256), resident_blocks((const void*)kernel, 256)));
}

// K6 -- gradient by Lst. 5 with the arithmetic-mean regulariser, divided by
// dx (R-13): (phi_{+1} - phi_{-1}) / (2 dx); optional unit normal.
// Gradient layout: [pkg][64][4] = (phi, d/dx, d/dy, d/dz) per data point --
// the probe reads one 16 B vector per trilinear corner.  Normal layout:
// [pkg][component][64].
__device__ __forceinline__ void st_vec4(float* p, float a, float b, float c, float d) {
    *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st_vec4(double* p, double a, double b, double c, double d) {
    reinterpret_cast<double2*>(p)[0] = make_double2(a, b);
    reinterpret_cast<double2*>(p)[1] = make_double2(c, d);
}

// 1 / |g| from |g|^2, 0 for g = 0: fp32 via MUFU rsqrt (~2 ulp, inside the
// 1e-5 normal tolerance), fp64 exactly rounded sqrt and division
__device__ __forceinline__ float inv_norm(float m2) { return m2 > 0.f ? rsqrtf(m2) : 0.f; }
__device__ __forceinline__ double inv_norm(double m2) { return m2 > 0.0 ? 1.0 / sqrt(m2) : 0.0; }

// store tile of one package's (phi, grad) rows: point d at 4 d + 4 (d / 8)
// -- a 16 B pad every 8 points keeps both the row-wise writes (lane r,
// points 4 r .. 4 r + 3) and the point-wise reads (lane r, point r + 16 i)
// free of shared-memory bank conflicts
constexpr int kTileStride = 64 * 4 + 8 * 4;
__device__ __forceinline__ int tile_ofs(int d) { return 4 * d + 4 * (d >> 3); }

template <class T>
__device__ __forceinline__ void grad_package(const T* __restrict__ in, T* __restrict__ grad,
                                             T* __restrict__ normal,
                                             const uint32_t* __restrict__ face, int64_t pkg,
                                             bool valid, const StC<T>& c, T* tile);

template <class T>
__global__ void __launch_bounds__(256) k_gradient(const T* __restrict__ in, T* __restrict__ grad,
                                                  T* __restrict__ normal,
                                                  const uint32_t* __restrict__ face, int64_t lo,
                                                  int64_t hi, StC<T> c) {
    __shared__ __align__(16) T s_tile[16][kTileStride];
    const int64_t pkg = lo + (((int64_t)blockIdx.x * 256 + threadIdx.x) >> 4);
    grad_package(in, grad, normal, face, pkg, pkg < hi, c, s_tile[threadIdx.x >> 4]);
}

// K6 for one x-row (lane r = threadIdx.x & 15 of a 16-lane group) of `pkg`
template <class T>
__device__ __forceinline__ void grad_package(const T* __restrict__ in, T* __restrict__ grad,
                                             T* __restrict__ normal,
                                             const uint32_t* __restrict__ face, int64_t pkg,
                                             bool valid, const StC<T>& c, T* tile) {
    Cross<T> x;
    if (!load_cross(in, face, pkg, valid, x)) return;
    T gx[4], gy[4], gz[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const T l = i > 0 ? x.c[i - 1] : x.xm;
        const T r = i < 3 ? x.c[i + 1] : x.xp;
        gx[i] = (r - l) * c.inv_2dx;
        gy[i] = (x.yp[i] - x.ym[i]) * c.inv_2dx;
        gz[i] = (x.zp[i] - x.zm[i]) * c.inv_2dx;
    }
    const int r = threadIdx.x & 15;
    if (grad) {
        // (phi, grad) of the row's 4 points are 64 contiguous bytes per lane;
        // stored directly, each store instruction would hit a 16 B piece of
        // 16 lines (ncu: k_gradient L1-bound on store wavefronts).  Through
        // the package's shared tile the 16 lanes store 256 contiguous bytes
        // per instruction.
#pragma unroll
        for (int i = 0; i < 4; ++i) st_vec4(tile + tile_ofs(4 * r + i), x.c[i], gx[i], gy[i], gz[i]);
        __syncwarp(0xFFFFu << (threadIdx.x & 16));
        T* G = grad + pkg * 256;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int d = r + 16 * i;
            T v[4];
            ld_row_s(tile + tile_ofs(d), v);
            st_vec4(G + 4 * d, v[0], v[1], v[2], v[3]);
        }
    }
    if (normal) {
        T nx[4], ny[4], nz[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const T inv = inv_norm(gx[i] * gx[i] + gy[i] * gy[i] + gz[i] * gz[i]);
            nx[i] = gx[i] * inv;
            ny[i] = gy[i] * inv;
            nz[i] = gz[i] * inv;
        }
        T* N = normal + pkg * 192 + 4 * r;
        st_row(N, nx);
        st_row(N + 64, ny);
        st_row(N + 128, nz);
    }
}

// K6 for two x-rows of `pkg` by an 8-lane group (lane (j, k), k in {0, 1}:
// rows j + 4k and j + 4k + 8), the cross of load_cross2 (warp layout of
// k_sweep: the four groups of a warp hold consecutive packages).  Same
// formula per point as grad_package (bit-identical); the (phi, grad) rows go
// through the package's shared tile so every store instruction writes 128
// contiguous bytes per group.  Used by the fused K6 + K7 kernel: two K6
// warps per 8 packages instead of four leave room for more K7 warps.
template <class T>
__device__ __forceinline__ void grad_package8(const T* __restrict__ in, T* __restrict__ grad,
                                              T* __restrict__ normal,
                                              const uint32_t* __restrict__ face, uint32_t pkg,
                                              bool valid, bool next_ok, const StC<T>& c, T* tile) {
    const int g8 = threadIdx.x & 7, j = g8 & 3, k = g8 >> 2;
    uint32_t f = 0;
    if (valid && g8 < 6) f = __ldg(face + (size_t)pkg * 8 + g8);
    Cross2<T> x;
    load_cross2<T, true>(in, pkg, valid, next_ok, f, j, k, x);
    if (!valid) return;
    const int r0 = j + 4 * k, r1 = r0 + 8;
    T g[2][3][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const T l0 = i > 0 ? x.c0[i - 1] : x.xm0, q0 = i < 3 ? x.c0[i + 1] : x.xp0;
        const T l1 = i > 0 ? x.c1[i - 1] : x.xm1, q1 = i < 3 ? x.c1[i + 1] : x.xp1;
        g[0][0][i] = (q0 - l0) * c.inv_2dx;
        g[0][1][i] = (x.yp0[i] - x.ym0[i]) * c.inv_2dx;
        g[0][2][i] = (x.zmid[i] - x.zlo[i]) * c.inv_2dx;
        g[1][0][i] = (q1 - l1) * c.inv_2dx;
        g[1][1][i] = (x.yp1[i] - x.ym1[i]) * c.inv_2dx;
        g[1][2][i] = (x.zhi[i] - x.zmid[i]) * c.inv_2dx;
    }
    if (grad) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            st_vec4(tile + tile_ofs(4 * r0 + i), x.c0[i], g[0][0][i], g[0][1][i], g[0][2][i]);
            st_vec4(tile + tile_ofs(4 * r1 + i), x.c1[i], g[1][0][i], g[1][1][i], g[1][2][i]);
        }
        __syncwarp(0xFFu << (threadIdx.x & 24));
        T* G = grad + (size_t)pkg * 256;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int d = g8 + 8 * i;
            T v[4];
            ld_row_s(tile + tile_ofs(d), v);
            st_vec4(G + 4 * d, v[0], v[1], v[2], v[3]);
        }
    }
    if (normal) {
        T* N = normal + (size_t)pkg * 192;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = h ? r1 : r0;
            T nx[4], ny[4], nz[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const T inv = inv_norm(g[h][0][i] * g[h][0][i] + g[h][1][i] * g[h][1][i] +
                                       g[h][2][i] * g[h][2][i]);
                nx[i] = g[h][0][i] * inv;
                ny[i] = g[h][1][i] * inv;
                nz[i] = g[h][2][i] * inv;
            }
            st_row(N + 4 * r, nx);
            st_row(N + 64 + 4 * r, ny);
            st_row(N + 128 + 4 * r, nz);
        }
    }
}

// Table 1 "stencil": 7-point Laplacian
template <class T>
__global__ void __launch_bounds__(256) k_laplace(const T* __restrict__ in, T* __restrict__ out,
                                                 const uint32_t* __restrict__ face, int64_t lo,
                                                 int64_t hi, T inv_dx2) {
    const int64_t pkg = lo + (((int64_t)blockIdx.x * 256 + threadIdx.x) >> 4);
    Cross<T> x;
    if (!load_cross(in, face, pkg, pkg < hi, x)) return;
    T o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const T l = i > 0 ? x.c[i - 1] : x.xm;
        const T r = i < 3 ? x.c[i + 1] : x.xp;
        o[i] = (((l + r) + (x.ym[i] + x.yp[i])) + (x.zm[i] + x.zp[i]) - T(6) * x.c[i]) * inv_dx2;
    }
    st_row(out + pkg * 64 + 4 * (threadIdx.x & 15), o);
}

// Table 1 "sequential": a minor change to every active value
template <class T>
__global__ void k_add(T* __restrict__ phi, int64_t n4, int64_t off4, T v) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n4) return;
    T* p = phi + 4 * (off4 + t);
    T r[4];
    ld_row(p, r);
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] += v;
    st_row(p, r);
}

// ------------------------------------------------------ kernel integral --
// K7 (reading R-14): K = sum_o w[o] H(-phi_{I+o}),
// G = sum_o gw[o] H(-phi_{I+o}) over the taps |o| dx < 2h of a Wendland C2
// kernel.  The weights depend on o only through s = |o|^2:
// w[o] = Wt[s], gw[o] = Gt[s] * o (Gt[s] = W'(|o| dx) (-1/|o|) dx^3).
//
// Mapping: 16 threads per package, 8 packages per 128-thread block.  Each
// package stages its (4 + 2R)^3 neighbourhood of H(-phi) in shared memory
// (values fetched through the package's neighbour row with Lst. 2; shifts in
// [-R, 3 + R] stay inside [-4, 7]), then every thread produces one x-row of 4
// outputs: for every (oy, oz) of the stencil it reads one staged row of
// 4 + 2R values (vector shared loads) and applies all its x-taps to the 4
// outputs with register-resident weights (taps unrolled at compile time,
// R = ceil(2 h_ratio) - 1, all |o|^2 <= (R+1)^2 - 1 enumerated; taps outside
// the support carry weight 0).  Packages whose whole staged neighbourhood is
// uniformly H = 0 or H = 1 take the closed form K = S H, G = 0 (exact in exact
// arithmetic since sum gw = 0).

__device__ __forceinline__ float heav(float u, float eps, float inv_eps) {
    if (u < -eps) return 0.f;
    if (u > eps) return 1.f;
    const float q = u * inv_eps;
    // MUFU sine: absolute error <= 2^-21.4 on [-pi, pi] -> |dH| < 1.2e-7,
    // |dK| < 1.2e-7 S, well inside the fp32 tolerance (1e-5)
    return 0.5f * (1.f + q + __sinf(3.14159265358979f * q) * 0.318309886183790672f);
}
__device__ __forceinline__ double heav(double u, double eps, double inv_eps) {
    if (u < -eps) return 0.0;
    if (u > eps) return 1.0;
    const double q = u * inv_eps;
    return 0.5 * (1.0 + q + sinpi(q) * 0.318309886183790672);
}

// fp32 band rows: the smooth form saturated to [0, 1] in the same FMA.  The
// form is nondecreasing (derivative (1 + cos pi q) / 2 >= 0) with value 1 at
// q = 1 and 0 at q = -1, so saturation reproduces the outer branches: exactly
// for abs(q) >= 1.5 (margin 0.09 over the MUFU sine error), and within the
// sine error (~1e-7) just outside the band
__device__ __forceinline__ float heav_sat(float u, float eps, float inv_eps) {
    const float lin = fmaf(u, 0.5f * inv_eps, 0.5f);
    return __saturatef(fmaf(__sinf(u * (3.14159265358979f * inv_eps)), 0.159154943091895336f, lin));
}
__device__ __forceinline__ double heav_sat(double u, double eps, double inv_eps) {
    return heav(u, eps, inv_eps);
}

template <class T>
struct KintC {
    T wt[16];     // Wt[s], s = |o|^2
    T gt[4][16];  // m * Gt[s] for |o_k| = m (pre-multiplied: no per-tap multiply)
    T S;          // sum of all weights (host, double rounded to T)
    T eps, inv_eps;
};

template <int R>
struct KGeo {
    static constexpr int RS = 4 + 2 * R;                 // staged width
    static constexpr int RSX = (RS + 3) & ~3;            // padded row (16 B multiple)
    static constexpr int SLICE = RS * RSX + 4;           // padded z-slice (bank shift)
    static constexpr int VOL = RS * SLICE;               // floats per package
    static constexpr int S2MAX = (R + 1) * (R + 1) - 1;  // largest |o|^2 enumerated
};

// S2M: the largest |o|^2 enumerated -- (R+1)^2 - 1 in general; 6 for R = 2
// when the taps at |o|^2 = 8 lie outside the support (h_ratio <= sqrt 2, e.g.
// the default 1.3: 81 taps), which drops their zero-weight FMAs and the whole
// (|oy|, |oz|) = (2, 2) row group (same bits: fma(0, h, acc) = acc)
// GR: K6 fused in horizontally -- warps 4..5 of a 192-thread block compute the
// gradient / normal of the block's 8 packages (8 lanes per package,
// grad_package8) while warps 0..3 compute their kernel integrals: the
// HBM-write-bound K6 warps and the issue-bound K7 warps share every SM.
// fp32 tap loop of k_kint on paired-FP32 instructions: the (up to) four
// rows of a (abs oy, abs oz) group are combined by the sign butterfly with
// FADD2 / FFMA2 (value pairs (q, q + 1) are aligned register pairs of the
// staged float4 rows), and every tap whose window offset R + ox is even
// updates output points (0, 1) and (2, 3) with one FFMA2 each; odd offsets
// stay scalar.  Per output the operations and their order are those of the
// generic loop -- bit-identical results.
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
    return __ffma2_rn(b, make_float2(-1.f, -1.f), a);  // a - b, exact as FADD
}
template <int R, int S2M, class Load>
__device__ __forceinline__ void kint_taps_f2(const KintC<float>& c, Load&& load, float (&acc)[4],
                                             float (&gx)[4], float (&gy)[4], float (&gz)[4]) {
    float2 A[2], X[2], Y[2], Z[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) A[u] = X[u] = Y[u] = Z[u] = make_float2(0.f, 0.f);
    auto pairs = [](const float (&h)[8], float2 (&o)[4]) {
#pragma unroll
        for (int u = 0; u < 4; ++u) o[u] = make_float2(h[2 * u], h[2 * u + 1]);
    };
    auto el = [](const float2 (&v)[4], int q) { return (q & 1) ? v[q >> 1].y : v[q >> 1].x; };
#pragma unroll
    for (int ga = 0; ga <= R; ++ga) {
#pragma unroll
        for (int gb = 0; gb <= R; ++gb) {
            if (ga * ga + gb * gb > S2M) continue;
            float2 S[4], Dy[4], Dz[4];
            if (ga == 0 && gb == 0) {
                float h[8];
                load(0, 0, h);
                pairs(h, S);
            } else if (gb == 0 || ga == 0) {
                float hp[8], hm[8];
                load(gb == 0 ? ga : 0, gb == 0 ? 0 : gb, hp);
                load(gb == 0 ? -ga : 0, gb == 0 ? 0 : -gb, hm);
                float2 p2[4], m2[4];
                pairs(hp, p2);
                pairs(hm, m2);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    S[u] = __fadd2_rn(p2[u], m2[u]);
                    (gb == 0 ? Dy : Dz)[u] = f2sub(p2[u], m2[u]);
                }
            } else {
                float hpp[8], hpm[8], hmp[8], hmm[8];
                load(ga, gb, hpp);
                load(ga, -gb, hpm);
                load(-ga, gb, hmp);
                load(-ga, -gb, hmm);
                float2 pp[4], pm[4], mp[4], mm[4];
                pairs(hpp, pp);
                pairs(hpm, pm);
                pairs(hmp, mp);
                pairs(hmm, mm);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 a1 = __fadd2_rn(pp[u], pm[u]), b1 = __fadd2_rn(mp[u], mm[u]);
                    const float2 c1 = f2sub(pp[u], pm[u]), d1 = f2sub(mp[u], mm[u]);
                    S[u] = __fadd2_rn(a1, b1);
                    Dy[u] = f2sub(a1, b1);
                    Dz[u] = __fadd2_rn(c1, d1);
                }
            }
#pragma unroll
            for (int ox = -R; ox <= R; ++ox) {
                const int s2 = ox * ox + ga * ga + gb * gb;
                if (s2 > S2M) continue;
                const float w = c.wt[s2];
                const float wx = ox > 0 ? c.gt[ox][s2] : -c.gt[-ox][s2];
                const float wy = c.gt[ga][s2];
                const float wz = c.gt[gb][s2];
                const int q0 = R + ox;
                if ((q0 & 1) == 0) {
                    const float2 w2 = make_float2(w, w), wx2 = make_float2(wx, wx);
                    const float2 wy2 = make_float2(wy, wy), wz2 = make_float2(wz, wz);
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int p = (q0 >> 1) + u;
                        A[u] = __ffma2_rn(w2, S[p], A[u]);
                        if (ox) X[u] = __ffma2_rn(wx2, S[p], X[u]);
                        if (ga) Y[u] = __ffma2_rn(wy2, Dy[p], Y[u]);
                        if (gb) Z[u] = __ffma2_rn(wz2, Dz[p], Z[u]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float& a = (i & 1) ? A[i >> 1].y : A[i >> 1].x;
                        float& x = (i & 1) ? X[i >> 1].y : X[i >> 1].x;
                        float& y = (i & 1) ? Y[i >> 1].y : Y[i >> 1].x;
                        float& z = (i & 1) ? Z[i >> 1].y : Z[i >> 1].x;
                        const float hv = el(S, q0 + i);
                        a = fmaf(w, hv, a);
                        if (ox) x = fmaf(wx, hv, x);
                        if (ga) y = fmaf(wy, el(Dy, q0 + i), y);
                        if (gb) z = fmaf(wz, el(Dz, q0 + i), z);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        acc[2 * u] = A[u].x;
        acc[2 * u + 1] = A[u].y;
        gx[2 * u] = X[u].x;
        gx[2 * u + 1] = X[u].y;
        gy[2 * u] = Y[u].x;
        gy[2 * u + 1] = Y[u].y;
        gz[2 * u] = Z[u].x;
        gz[2 * u + 1] = Z[u].y;
    }
}

template <class T, int R, int S2M, bool GR = false>
__global__ void __launch_bounds__(GR ? 192 : 128, (R == 2 && S2M == 6 && sizeof(T) == 4) ? (GR ? 6 : 10) : 1) k_kint(const T* __restrict__ in,
                                              const uint32_t* __restrict__ nb, int64_t lo,
                                              int64_t hi, KintC<T> c, T* __restrict__ K,
                                              T* __restrict__ G, T* __restrict__ grad = nullptr,
                                              T* __restrict__ normal = nullptr,
                                              const uint32_t* __restrict__ face = nullptr,
                                              StC<T> cs = StC<T>{}) {
    if constexpr (GR) {
        if (threadIdx.x >= 128) {  // K6: warps 4-5, 8 lanes per package
            __shared__ __align__(16) T s_gtile[8][kTileStride];
            const int q = (threadIdx.x - 128) >> 3;
            const int64_t pkg = lo + (int64_t)blockIdx.x * 8 + q;
            grad_package8(in, grad, normal, face, (uint32_t)pkg, pkg < hi, pkg + 1 < hi, cs,
                          s_gtile[q]);
            return;
        }
    }
    using Geo = KGeo<R>;
    constexpr int RS = Geo::RS, RSX = Geo::RSX, SLICE = Geo::SLICE, VOL = Geo::VOL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* s_h = reinterpret_cast<T*>(smem_raw);
    __shared__ uint32_t s_nb[8][28];

    const int lp = threadIdx.x >> 4;  // package slot in block (0..7)
    const int r = threadIdx.x & 15;   // x-row (j, k) of this thread
    const int64_t pkg = lo + (int64_t)blockIdx.x * 8 + lp;
    const bool valid = pkg < hi;
    if (valid) {
        s_nb[lp][r] = __ldg(nb + pkg * 27 + r);
        if (r < 11) s_nb[lp][16 + r] = __ldg(nb + pkg * 27 + 16 + r);
    }
    __syncwarp();
    T* H = s_h + lp * VOL;
    bool all1 = true, all0 = true;
    if (valid) {
        // staged x-rows (ly, lz) of the region, thread r takes rows r, r+16, ...
        // A row spans x-shifts [-R, 3+R]: data 4-R..3 of the -x neighbour,
        // the whole row of the centre column package, data 0..R-1 of the +x
        // neighbour (Lst. 2) -- three loads per row (vector loads for R = 2).
        constexpr int NR = RS * RS, RPT = (NR + 15) / 16;
#pragma unroll
        for (int m = 0; m < RPT; ++m) {
            const int rowi = r + 16 * m;
            if (rowi < NR) {
                // R = 2: the 8 lanes of a 16 B store phase write rows
                // ly = 0..3 of two consecutive slices (banks 8 ly and
                // 8 ly + 4): with 8 consecutive ly of one slice, rows ly and
                // ly + 4 shared banks (ncu: 2-way conflicts on half the
                // staging stores)
                const int ly = RS == 8 ? (rowi & 3) + 4 * ((rowi >> 3) & 1) : rowi % RS;
                const int lz = RS == 8 ? 2 * (rowi >> 4) + ((rowi >> 2) & 1) : rowi / RS;
                const int sy = ly - R, sz = lz - R;
                const Shift hy = nb_shift(sy), hz = nb_shift(sz);
                const int dyz = 4 * hy.data + 16 * hz.data;
                const uint32_t* slot = &s_nb[lp][3 * hy.off + 9 * hz.off];
                const T* p0 = in + (size_t)slot[0] * 64 + dyz;
                const T* p1 = in + (size_t)slot[1] * 64 + dyz;
                const T* p2 = in + (size_t)slot[2] * 64 + dyz;
                T v[RSX];
                if constexpr (R == 2 && sizeof(T) == 4) {
                    const float2 a2 = __ldg(reinterpret_cast<const float2*>(p0 + 2));
                    const float4 b4 = __ldg(reinterpret_cast<const float4*>(p1));
                    const float2 c2 = __ldg(reinterpret_cast<const float2*>(p2));
                    v[0] = a2.x; v[1] = a2.y;
                    v[2] = b4.x; v[3] = b4.y; v[4] = b4.z; v[5] = b4.w;
                    v[6] = c2.x; v[7] = c2.y;
                } else {
#pragma unroll
                    for (int q = 0; q < R; ++q) v[q] = __ldg(p0 + 4 - R + q);
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[R + q] = __ldg(p1 + q);
#pragma unroll
                    for (int q = 0; q < R; ++q) v[R + 4 + q] = __ldg(p2 + q);
#pragma unroll
                    for (int q = RS; q < RSX; ++q) v[q] = T(0);
                }
                // H(-phi): rows with no value inside the smoothing band
                // |phi| <= eps take the exact 0 / 1 select only (no sine);
                // the others the branch-free smooth form
                // One min / max pass classifies the row: it meets the band
                // when min |v| <= eps; otherwise H is exactly 1 (0) on all of
                // it iff max v < 0 (min v > 0).  (A band row is never taken
                // as uniform, even where its smooth values round to 1 / 0:
                // the taps then give the same values to rounding.)
                T h[RSX];
                T vmin = v[0], vmax = v[0], amin = fabs(v[0]);
#pragma unroll
                for (int q = 1; q < RS; ++q) {
                    vmin = fmin(vmin, v[q]);
                    vmax = fmax(vmax, v[q]);
                    amin = fmin(amin, fabs(v[q]));
                }
                const bool smooth = !(amin > c.eps);
                if (smooth) {
#pragma unroll
                    for (int q = 0; q < RSX; ++q) h[q] = heav_sat(-v[q], c.eps, c.inv_eps);
                } else {
#pragma unroll
                    for (int q = 0; q < RSX; ++q) h[q] = v[q] < T(0) ? T(1) : T(0);
                }
                all1 = all1 && !smooth && vmax < T(0);
                all0 = all0 && !smooth && vmin > T(0);
                T* dst = H + lz * SLICE + ly * RSX;
#pragma unroll
                for (int q = 0; q < RSX; q += 4) {
                    if constexpr (sizeof(T) == 4) {
                        *reinterpret_cast<float4*>(dst + q) =
                            make_float4(h[q], h[q + 1], h[q + 2], h[q + 3]);
                    } else {
                        reinterpret_cast<double2*>(dst + q)[0] = make_double2(h[q], h[q + 1]);
                        reinterpret_cast<double2*>(dst + q)[1] = make_double2(h[q + 2], h[q + 3]);
                    }
                }
            }
        }
    }
    // package-uniform neighbourhood? (16 lanes of a package share a half-warp)
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
        all1 = __shfl_xor_sync(0xffffffffu, (int)all1, o) && all1;
        all0 = __shfl_xor_sync(0xffffffffu, (int)all0, o) && all0;
    }
    __syncwarp();
    if (!valid) return;
    const int j = r & 3, k = r >> 2;
    T acc[4], gx[4], gy[4], gz[4];
    if (all1 || all0) {
        const T v = all1 ? c.S : T(0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc[i] = v;
            gx[i] = gy[i] = gz[i] = T(0);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = gx[i] = gy[i] = gz[i] = T(0);
        // rows (oy, oz) grouped by (|oy|, |oz|) = (a, b): with the sign
        // butterfly of the (up to) four rows (+-a, +-b)
        //   S  = sum of the rows            -> K and G_x
        //   Dy = rows(+a) - rows(-a)        -> G_y  (weight a Gt)
        //   Dz = rows(+b) - rows(-b)        -> G_z  (weight b Gt)
        // every tap weight is applied once per group instead of once per row
        auto load = [&](int oy, int oz, T (&h)[RSX]) {
            const T* row = H + (k + R + oz) * SLICE + (j + R + oy) * RSX;
#pragma unroll
            for (int q = 0; q < RSX; q += 4) {
                if constexpr (sizeof(T) == 4) {
                    const float4 v = *reinterpret_cast<const float4*>(row + q);
                    h[q] = v.x; h[q + 1] = v.y; h[q + 2] = v.z; h[q + 3] = v.w;
                } else {
                    const double2 a2 = *reinterpret_cast<const double2*>(row + q);
                    const double2 b2 = *reinterpret_cast<const double2*>(row + q + 2);
                    h[q] = a2.x; h[q + 1] = a2.y; h[q + 2] = b2.x; h[q + 3] = b2.y;
                }
            }
        };
        if constexpr (sizeof(T) == 4 && RSX == 8) {
            kint_taps_f2<R, S2M>(c, [&](int oy, int oz, float (&h)[8]) { load(oy, oz, h); }, acc,
                                 gx, gy, gz);
        } else {
#pragma unroll
            for (int ga = 0; ga <= R; ++ga) {
#pragma unroll
                for (int gb = 0; gb <= R; ++gb) {
                    if (ga * ga + gb * gb > S2M) continue;
                    T S[RSX], Dy[RSX], Dz[RSX];
                    if (ga == 0 && gb == 0) {
                        load(0, 0, S);
                    } else if (gb == 0) {
                        T p_[RSX], m_[RSX];
                        load(ga, 0, p_);
                        load(-ga, 0, m_);
#pragma unroll
                        for (int q = 0; q < RSX; ++q) { S[q] = p_[q] + m_[q]; Dy[q] = p_[q] - m_[q]; }
                    } else if (ga == 0) {
                        T p_[RSX], m_[RSX];
                        load(0, gb, p_);
                        load(0, -gb, m_);
#pragma unroll
                        for (int q = 0; q < RSX; ++q) { S[q] = p_[q] + m_[q]; Dz[q] = p_[q] - m_[q]; }
                    } else {
                        T pp[RSX], pm[RSX], mp[RSX], mm[RSX];
                        load(ga, gb, pp);
                        load(ga, -gb, pm);
                        load(-ga, gb, mp);
                        load(-ga, -gb, mm);
#pragma unroll
                        for (int q = 0; q < RSX; ++q) {
                            const T a1 = pp[q] + pm[q], b1 = mp[q] + mm[q];
                            const T c1 = pp[q] - pm[q], d1 = mp[q] - mm[q];
                            S[q] = a1 + b1;
                            Dy[q] = a1 - b1;
                            Dz[q] = c1 + d1;
                        }
                    }
#pragma unroll
                    for (int ox = -R; ox <= R; ++ox) {
                        const int s2 = ox * ox + ga * ga + gb * gb;
                        if (s2 > S2M) continue;
                        const T w = c.wt[s2];
                        const T wx = ox > 0 ? c.gt[ox][s2] : -c.gt[-ox][s2];
                        const T wy = c.gt[ga][s2];
                        const T wz = c.gt[gb][s2];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const T hv = S[i + R + ox];
                            acc[i] = fma(w, hv, acc[i]);
                            if (ox) gx[i] = fma(wx, hv, gx[i]);
                            if (ga) gy[i] = fma(wy, Dy[i + R + ox], gy[i]);
                            if (gb) gz[i] = fma(wz, Dz[i + R + ox], gz[i]);
                        }
                    }
                }
            }
        }
    }
    st_row(K + pkg * 64 + 4 * r, acc);
    T* Gp = G + pkg * 192 + 4 * r;
    st_row(Gp, gx);
    st_row(Gp + 64, gy);
    st_row(Gp + 128, gz);
}

// singular packages (R-16): K = S / 0, G = 0; grad = normal = 0 (the phi
// slot of the gradient layout holds the far constants)
template <class T>
__global__ void k_singular(T* K, T* G, T* grad, T* normal, T S, T far) {
    const int t = threadIdx.x;  // 128 threads: two packages x 64
    if (K) K[t] = t < 64 ? S : T(0);
    if (grad) {
        grad[4 * t] = t < 64 ? -far : far;
        grad[4 * t + 1] = grad[4 * t + 2] = grad[4 * t + 3] = T(0);
    }
    for (int c = 0; c < 3; ++c) {
        const int idx = (t >> 6) * 192 + c * 64 + (t & 63);
        if (G) G[idx] = T(0);
        if (normal) normal[idx] = T(0);
    }
}

// ---------------------------------------------------------- launchers ----

template <class T>
static StC<T> stencil_consts(const sg_grid* g, double cfl) {
    StC<T> c;
    c.inv_dx = (T)(1.0 / g->gc.dx);
    c.dx2 = (T)(g->gc.dx * g->gc.dx);
    c.cdx = (T)(cfl * g->gc.dx);
    c.inv_2dx = (T)(0.5 / g->gc.dx);
    c.ncfl = (T)(-cfl);
    return c;
}

template <class T>
static bool reinit_launch(sg_grid* g, int cur, const StC<T>& c, int64_t lo, int64_t hi,
                          cudaStream_t s) {
    if (hi <= lo) return false;
    const ReinitOp<T> op{(T*)g->phi[1 - cur], c};
    // 32-bit element offsets below 2^32 data points (the stored packages)
    auto kern = g->n_pkg * 64 < ((int64_t)1 << 32) ? k_sweep<T, ReinitOp<T>, true>
                                                   : k_sweep<T, ReinitOp<T>, false>;
    const unsigned blocks = persistent_blocks(kern, hi - lo);
    kern<<<blocks, 256, 0, s>>>((const T*)g->phi[cur], g->face, (uint32_t)lo, (uint32_t)hi, op);
    return true;
}

// Partitioned grid (a9): groups of up to 4 sweeps per ghost
// exchange (the ghost plane is 4 data points deep; see sg_reinit_halo).  The
// first sweeps of a group run over owned + ghost packages; the last one
// updates the two boundary planes first (the packages the neighbours need),
// hands them to the internal high-priority comm stream for the grouped
// send/recv into the neighbours' ghost planes, and updates the interior
// packages while the transfer runs.  Jacobi sweeps: bit-identical to one GPU.
// enqueue the schedule on s starting from buffer `cur`; returns the final one
template <class T>
static int reinit_partitioned_enqueue(sg_grid* g, int cur, int32_t iters, double cfl,
                                      cudaStream_t s) {
    const StC<T> c = stencil_consts<T>(g, cfl);
    const sg_plan_t& p = g->plan;
    const bool lower = g->rank > 0, upper = g->rank < g->nranks - 1;
    // [b0lo, b0hi): first owned plane (if rank - 1 exists); [b1lo, b1hi):
    // last owned plane (if rank + 1 exists); interior between them
    const int64_t b0lo = p.own_lo, b0hi = lower ? p.send_lo[1] : p.own_lo;
    const int64_t b1hi = p.own_hi, b1lo = std::max(b0hi, upper ? p.send_hi[0] : p.own_hi);
    const size_t per = (size_t)64 * g->esz;
    for (int done = 0; done < iters;) {
        const int m = std::min(4, iters - done);
        for (int i = 0; i + 1 < m; ++i) {
            if (reinit_launch<T>(g, cur, c, 2, g->n_pkg, s)) SG_LAUNCHED();
            cur = 1 - cur;
        }
        if (reinit_launch<T>(g, cur, c, b0lo, b0hi, s)) SG_LAUNCHED();
        if (reinit_launch<T>(g, cur, c, b1lo, b1hi, s)) SG_LAUNCHED();
        SG_CUDA(cudaEventRecord(g->ev_b, s));
        SG_CUDA(cudaStreamWaitEvent(g->comm_stream, g->ev_b, 0));
        halo_exchange(g, g->phi[1 - cur], per, g->comm_stream);
        SG_CUDA(cudaEventRecord(g->ev_x, g->comm_stream));
        if (reinit_launch<T>(g, cur, c, b0hi, b1lo, s)) SG_LAUNCHED();
        SG_CUDA(cudaStreamWaitEvent(s, g->ev_x, 0));
        cur = 1 - cur;
        done += m;
    }
    return cur;
}

// Partitioned reinit over NCCL as one CUDA graph (sweeps, the fork to the
// comm stream, the captured NCCL send/recv groups, the joins): the sweeps of
// a slab are a few microseconds each at 8 ranks, so host launch latency
// would dominate.  Cached like the single-GPU graphs (plus the communicator
// and the halo ranges in the key).  A capture that fails (e.g. an NCCL
// without graph support) falls back to eager launches for the process;
// SG_COMM_GRAPHS=0 disables it.  The in-process communicator rendezvous on
// the host at every exchange, so it always runs eagerly.
struct PGraphKey {
    const void* p0;
    const void* p1;
    const void* face;
    const void* comm;
    int64_t n_pkg, own_lo, own_hi, r[8];
    int32_t iters, dt, device, cur;
    double cfl, dx;
    bool operator==(const PGraphKey& o) const {
        if (p0 != o.p0 || p1 != o.p1 || face != o.face || comm != o.comm || n_pkg != o.n_pkg ||
            own_lo != o.own_lo || own_hi != o.own_hi || iters != o.iters || dt != o.dt ||
            device != o.device || cur != o.cur || cfl != o.cfl || dx != o.dx)
            return false;
        for (int i = 0; i < 8; ++i)
            if (r[i] != o.r[i]) return false;
        return true;
    }
};
static std::mutex g_pgraph_mu;
struct PGraph {
    cudaGraphExec_t exec;
    uint64_t launches;  // kernel nodes per replay (sg_launch_count)
};
static std::vector<std::pair<PGraphKey, PGraph>> g_pgraphs;
static bool g_pgraph_off = false;

template <class T>
static void reinit_partitioned(sg_grid* g, int32_t iters, double cfl, cudaStream_t s) {
    static const bool env_on = [] {
        const char* e = std::getenv("SG_COMM_GRAPHS");
        return !(e && e[0] == '0');
    }();
    if (!env_on || iters < 2 || comm_kind(g->comm) != SG_COMM_NCCL || g_pgraph_off) {
        g->cur = reinit_partitioned_enqueue<T>(g, g->cur, iters, cfl, s);
        return;
    }
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    const sg_plan_t& p = g->plan;
    const PGraphKey key{g->phi[0], g->phi[1], g->face, g->comm, g->n_pkg, g->own_lo, g->own_hi,
                        {p.send_lo[0], p.send_lo[1], p.send_hi[0], p.send_hi[1], p.recv_lo[0],
                         p.recv_lo[1], p.recv_hi[0], p.recv_hi[1]},
                        iters, (int32_t)sizeof(T), dev, g->cur, cfl, g->gc.dx};
    std::lock_guard<std::mutex> lk(g_pgraph_mu);
    cudaGraphExec_t exec = nullptr;
    uint64_t nl = 0;
    for (auto& e : g_pgraphs)
        if (e.first == key) {
            exec = e.second.exec;
            nl = e.second.launches;
        }
    if (!exec) {
        cudaStream_t cap = nullptr;
        SG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaGraph_t graph = nullptr;
        bool ok = true;
        int cur_end = g->cur;
        const uint64_t l0 = g_launches.load();
        try {
            SG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            cur_end = reinit_partitioned_enqueue<T>(g, g->cur, iters, cfl, cap);
            SG_CUDA(cudaStreamEndCapture(cap, &graph));
            SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        } catch (const Error&) {
            ok = false;
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(cap, &junk);  // leave capture mode if still in it
            if (junk) cudaGraphDestroy(junk);
            cudaGetLastError();
        }
        if (graph) cudaGraphDestroy(graph);
        cudaStreamDestroy(cap);
        (void)cur_end;
        nl = g_launches.load() - l0;  // captured, not yet run
        g_launches.fetch_sub(nl);
        if (!ok || !exec) {
            g_pgraph_off = true;  // eager from now on
            g->cur = reinit_partitioned_enqueue<T>(g, g->cur, iters, cfl, s);
            return;
        }
        if (g_pgraphs.size() >= 16) {
            cudaGraphExecDestroy(g_pgraphs.front().second.exec);
            g_pgraphs.erase(g_pgraphs.begin());
        }
        g_pgraphs.push_back({key, PGraph{exec, nl}});
    }
    SG_CUDA(cudaGraphLaunch(exec, s));
    g_launches.fetch_add(nl);
    if (iters & 1) g->cur = 1 - g->cur;
}

// Multi-sweep reinit runs as one CUDA graph of `iters` kernel nodes.  The
// sweeps of an L2-resident band take ~10 us each, so launch gaps matter.
// Graphs are cached process-wide keyed by every kernel parameter (buffer
// pointers, id range, iters, start buffer, cfl): a rebuilt grid of the same
// shape gets the same pool addresses and reuses the instantiated graph.
struct GraphKey {
    const void* p0;
    const void* p1;
    const void* nb;
    const void* plan;  // two-sweep tile plan (nullptr: single sweeps)
    int64_t lo, hi;
    int32_t iters, dt, device;
    double cfl, dx;  // the captured StC (inv_dx, dx^2, cfl dx) derives from both
    bool operator==(const GraphKey& o) const {
        return p0 == o.p0 && p1 == o.p1 && nb == o.nb && plan == o.plan && lo == o.lo &&
               hi == o.hi && iters == o.iters && dt == o.dt && device == o.device &&
               cfl == o.cfl && dx == o.dx;
    }
};

static std::mutex g_graph_mu;
static std::vector<std::pair<GraphKey, cudaGraphExec_t>> g_graphs;  // small LRU
// capture streams, one per device (a stream belongs to the device current at
// its creation)
static std::vector<cudaStream_t> g_capture;

template <class T>
static void reinit_t(sg_grid* g, int32_t iters, double cfl, bool halo, cudaStream_t s) {
    if (g->partitioned()) {
        reinit_partitioned<T>(g, iters, cfl, s);
        return;
    }
    const StC<T> c = stencil_consts<T>(g, cfl);
    // owned packages, or (halo) every stored package: owned and ghost
    const int64_t lo = halo ? 2 : g->own_lo, hi = halo ? g->n_pkg : g->own_hi;
    if (iters == 1 || hi <= lo) {
        for (int it = 0; it < iters; ++it) {
            if (hi > lo) {
                reinit_launch<T>(g, g->cur, c, lo, hi, s);
                SG_LAUNCHED();
            }
            g->cur = 1 - g->cur;
        }
        return;
    }
    // two sweeps per launch (sg_tsweep.cu) where the grid allows it; the
    // tile plan is built here, outside any capture
    bool ts = false;
    if constexpr (std::is_same<T, float>::value) ts = !halo && tsweep_ready(g, s);
    const int64_t launches = ts ? iters / 2 + (iters & 1) : iters;
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    const GraphKey key{g->phi[g->cur], g->phi[1 - g->cur], g->face, ts ? tsweep_key(g) : nullptr,
                       lo, hi, iters, (int32_t)sizeof(T), dev, cfl, g->gc.dx};
    std::lock_guard<std::mutex> lk(g_graph_mu);
    cudaGraphExec_t exec = nullptr;
    for (size_t i = 0; i < g_graphs.size(); ++i)
        if (g_graphs[i].first == key) {
            exec = g_graphs[i].second;
            std::swap(g_graphs[i], g_graphs.back());  // most recent last
            break;
        }
    if (!exec) {
        if ((int)g_capture.size() <= dev) g_capture.resize(dev + 1, nullptr);
        cudaStream_t& cap = g_capture[dev];
        if (!cap) SG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaGraph_t graph;
        SG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        int cur = g->cur;
        if (ts) {
            for (int it = 0; it + 1 < iters; it += 2) {
                tsweep_launch(g, cur, (float)c.inv_dx, (float)c.dx2, (float)c.cdx, (float)c.ncfl, cap);
                cur = 1 - cur;
            }
            if (iters & 1) reinit_launch<T>(g, cur, c, lo, hi, cap);
        } else {
            for (int it = 0; it < iters; ++it) {
                reinit_launch<T>(g, cur, c, lo, hi, cap);
                cur = 1 - cur;
            }
        }
        SG_CUDA(cudaStreamEndCapture(cap, &graph));
        SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        SG_CUDA(cudaGraphDestroy(graph));
        if (g_graphs.size() >= 32) {
            cudaGraphExecDestroy(g_graphs.front().second);
            g_graphs.erase(g_graphs.begin());
        }
        g_graphs.push_back({key, exec});
    }
    SG_CUDA(cudaGraphLaunch(exec, s));
    g_launches.fetch_add((uint64_t)launches, std::memory_order_relaxed);
    if (launches & 1) g->cur = 1 - g->cur;
}

void launch_reinit(sg_grid* g, int32_t iters, double cfl, cudaStream_t s, bool halo) {
    if (g->dtype == SG_F64)
        reinit_t<double>(g, iters, cfl, halo, s);
    else
        reinit_t<float>(g, iters, cfl, halo, s);
}

// Wendland C2 weights (reading R-14), evaluated on the host in double:
// sigma = 21 / (16 pi h^3), q = r / h, W = sigma (1 - q/2)^4 (2q + 1),
// W' = -5 sigma q (1 - q/2)^3 / h; per |o|^2 = s2 (r = sqrt(s2) dx):
// Wt[s2] = W(r) dx^3, Gt[s2] = W'(r) (-1/|o|) dx^3 (so gw[o] = Gt[s2] o),
// both 0 outside the support |o| dx < 2h.  S = sum of w over the taps.
template <class T>
static KintC<T> make_kint(double h_ratio, double dx, int R, double* S_out) {
    const double pi = 3.14159265358979323846;
    const double h = h_ratio * dx;
    const double sigma = 21.0 / (16.0 * pi * h * h * h);
    KintC<T> c{};
    double wt[16] = {0}, S = 0.0;
    for (int s2 = 0; s2 < 16; ++s2) {
        const double len = std::sqrt((double)s2);
        if (!(len * dx < 2.0 * h)) continue;
        const double q = len * dx / h;
        const double a = 1.0 - 0.5 * q;
        wt[s2] = sigma * a * a * a * a * (2.0 * q + 1.0) * dx * dx * dx;
        const double dW = -5.0 * sigma * q * a * a * a / h * dx * dx * dx;
        c.wt[s2] = (T)wt[s2];
        for (int m = 0; m < 4; ++m) c.gt[m][s2] = (T)(len > 0 ? m * (-dW / len) : 0.0);
    }
    // S: the weights summed over every tap o in [-R, R]^3 (multiplicity of
    // each |o|^2), in double
    for (int oz = -R; oz <= R; ++oz)
        for (int oy = -R; oy <= R; ++oy)
            for (int ox = -R; ox <= R; ++ox) {
                const int s2 = ox * ox + oy * oy + oz * oz;
                if (s2 < 16) S += wt[s2];
            }
    c.S = (T)S;
    *S_out = S;
    c.eps = (T)dx;
    c.inv_eps = (T)(1.0 / dx);
    return c;
}

// gp / np non-null: K6 fused in (k_kint<..., true>)
template <class T, int R>
static void launch_kint_r(sg_grid* g, const T* phi, const KintC<T>& c, cudaStream_t s,
                          T* gp = nullptr, T* np = nullptr, StC<T> cs = StC<T>{}) {
    const int64_t lo = g->own_lo, hi = g->own_hi;
    if (hi <= lo) return;
    const size_t smem = sizeof(T) * 8 * KGeo<R>::VOL;
    const bool gr = gp || np;
    auto kern = gr ? k_kint<T, R, KGeo<R>::S2MAX, true> : k_kint<T, R, KGeo<R>::S2MAX, false>;
    if constexpr (R == 2) {
        if (c.wt[7] == T(0) && c.wt[8] == T(0))  // |o|^2 = 8 outside the support
            kern = gr ? k_kint<T, 2, 6, true> : k_kint<T, 2, 6, false>;
    }
    // dynamic + static (the fused K6 warps' store tiles) above the 48 KB
    // default needs the opt-in (fp64 at R >= 2)
    if (smem + (gr ? 8 * kTileStride * sizeof(T) : 0) + 8 * 28 * 4 > 48 * 1024)
        SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)ceil_div(hi - lo, 8), gr ? 192 : 128, smem, s>>>(
        phi, g->nb, lo, hi, c, (T*)g->kint, (T*)g->gkint, gp, np, g->face, cs);
    SG_LAUNCHED();
}

template <class T>
static void gradient_t(sg_grid* g, uint32_t fields, double h_ratio, cudaStream_t s) {
    const int64_t lo = g->own_lo, hi = g->own_hi;
    const T* phi = (const T*)g->phi[g->cur];
    const StC<T> c = stencil_consts<T>(g, 0.0);
    const size_t vec_bytes = (size_t)g->n_pkg * 192 * sizeof(T);
    const bool want_g = fields & (SG_GRAD | SG_NORMAL), want_k = fields & SG_KINT;
    if ((fields & SG_GRAD) && !g->grad) g->grad = g->alloc((size_t)g->n_pkg * 256 * sizeof(T), s);
    if ((fields & SG_NORMAL) && !g->normal) g->normal = g->alloc(vec_bytes, s);
    if (want_k && !g->kint) g->kint = g->alloc((size_t)g->n_pkg * 64 * sizeof(T), s);
    if (want_k && !g->gkint) g->gkint = g->alloc(vec_bytes, s);
    T* gp = (fields & SG_GRAD) ? (T*)g->grad : nullptr;
    T* np = (fields & SG_NORMAL) ? (T*)g->normal : nullptr;
    // K6 (HBM-write bound) and K7 (issue bound) both requested: one kernel,
    // K6 warps beside K7 warps in every block (k_kint<..., true>), so the two
    // share the SMs instead of queueing one behind the other
    // (SG_FUSE_K6K7=0: separate kernels, A/B)
    static const bool fuse_env = [] {
        const char* e = std::getenv("SG_FUSE_K6K7");
        return !(e && e[0] == '0');
    }();
    const bool fuse = want_g && want_k && fuse_env;
    if (want_k) {
        // largest |o_k| of a tap: o_k < 2 h_ratio  ->  R = ceil(2 h_ratio) - 1
        const int R = (int)std::ceil(2.0 * h_ratio) - 1;
        double S = 0.0;
        const KintC<T> kc = make_kint<T>(h_ratio, g->gc.dx, R, &S);
        T* fg = fuse ? gp : nullptr;
        T* fn = fuse ? np : nullptr;
        switch (R) {
        case 0: launch_kint_r<T, 0>(g, phi, kc, s, fg, fn, c); break;
        case 1: launch_kint_r<T, 1>(g, phi, kc, s, fg, fn, c); break;
        case 2: launch_kint_r<T, 2>(g, phi, kc, s, fg, fn, c); break;
        default: launch_kint_r<T, 3>(g, phi, kc, s, fg, fn, c); break;
        }
        // singular packages (R-16) of every field written here
        k_singular<T><<<1, 128, 0, s>>>((T*)g->kint, (T*)g->gkint, fg, fn, kc.S, (T)g->gc.far);
        SG_LAUNCHED();
        g->has_kint = true;
        g->kernel_sum = S;
    }
    if (want_g && !fuse) {
        if (hi > lo) {
            // (a persistent 8-lane variant like the reinit sweep measured
            // slower here: the kernel is bound by its 1.8 KB/package of writes)
            const unsigned blocks = (unsigned)ceil_div((hi - lo) * 16, 256);
            k_gradient<T><<<blocks, 256, 0, s>>>(phi, gp, np, g->face, lo, hi, c);
            SG_LAUNCHED();
        }
        k_singular<T><<<1, 128, 0, s>>>(nullptr, nullptr, gp, np, T(0), (T)g->gc.far);
        SG_LAUNCHED();
    }
    // partitioned grid: the (phi, grad) ghost planes for probes whose
    // trilinear corners lie in a ghost plane
    if (gp) halo_exchange(g, gp, (size_t)256 * sizeof(T), s);
    if (gp) g->has_grad = true;
    if (np) g->has_normal = true;
}

void launch_gradient(sg_grid* g, uint32_t fields, double h_ratio, cudaStream_t s) {
    if (g->dtype == SG_F64)
        gradient_t<double>(g, fields, h_ratio, s);
    else
        gradient_t<float>(g, fields, h_ratio, s);
}

template <class T>
static void table1_t(sg_grid* g, int32_t op, double value, cudaStream_t s) {
    const int64_t lo = g->own_lo, hi = g->own_hi;
    if (op == 0) {
        // the add is pointwise: on a slab grid it covers the ghost packages
        // too, which then hold exactly what their owner computes
        const int64_t lo = 2, hi = g->n_pkg;
        if (hi <= lo) return;
        const int64_t n4 = (hi - lo) * 16;
        k_add<T><<<(unsigned)ceil_div(n4, 256), 256, 0, s>>>((T*)g->phi[g->cur], n4, lo * 16,
                                                            (T)value);
    } else {
        if (hi <= lo) return;
        const unsigned blocks = (unsigned)ceil_div((hi - lo) * 16, 256);
        k_laplace<T><<<blocks, 256, 0, s>>>((const T*)g->phi[g->cur], (T*)g->phi[1 - g->cur],
                                            g->face, lo, hi, (T)(1.0 / (g->gc.dx * g->gc.dx)));
    }
    SG_LAUNCHED();
}

void launch_table1(sg_grid* g, int32_t op, double value, cudaStream_t s) {
    if (g->dtype == SG_F64)
        table1_t<double>(g, op, value, s);
    else
        table1_t<float>(g, op, value, s);
}

}  // namespace sg

using namespace sg;

extern "C" sg_status sg_reinit(sg_grid* g, int32_t iters, double cfl, void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_reinit");
        SG_ARG(g != nullptr, "sg_reinit: null grid");
        SG_ARG(iters >= 0, "sg_reinit: iters must be >= 0");
        SG_ARG(cfl > 0.0 && cfl <= 0.5, "sg_reinit: cfl must be in (0, 0.5]");
        SG_CUDA(cudaGetLastError());
        launch_reinit(g, iters, cfl, (cudaStream_t)stream);
        g->has_grad = g->has_normal = g->has_kint = false;  // derived fields are stale
    });
}

extern "C" sg_status sg_reinit_halo(sg_grid* g, int32_t iters, double cfl, void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_reinit_halo");
        SG_ARG(g != nullptr, "sg_reinit_halo: null grid");
        SG_ARG(iters >= 0, "sg_reinit_halo: iters must be >= 0");
        SG_ARG(cfl > 0.0 && cfl <= 0.5, "sg_reinit_halo: cfl must be in (0, 0.5]");
        SG_CUDA(cudaGetLastError());
        launch_reinit(g, iters, cfl, (cudaStream_t)stream, true);
        g->has_grad = g->has_normal = g->has_kint = false;
    });
}

extern "C" sg_status sg_gradient(sg_grid* g, uint32_t fields, double h_ratio, void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_gradient");
        SG_ARG(g != nullptr, "sg_gradient: null grid");
        SG_ARG(fields != 0 && (fields & ~7u) == 0, "sg_gradient: fields must be a non-empty OR of SG_GRAD/SG_NORMAL/SG_KINT");
        if (fields & SG_KINT)
            SG_ARG(h_ratio >= 0.5 && h_ratio <= 2.0, "sg_gradient: h_ratio must be in [0.5, 2]");
        SG_CUDA(cudaGetLastError());
        launch_gradient(g, fields, h_ratio, (cudaStream_t)stream);
    });
}

extern "C" sg_status sg_table1(sg_grid* g, int32_t op, double value, void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_table1");
        SG_ARG(g != nullptr, "sg_table1: null grid");
        SG_ARG(op == 0 || op == 1, "sg_table1: op must be 0 (sequential) or 1 (stencil)");
        SG_CUDA(cudaGetLastError());
        launch_table1(g, op, value, (cudaStream_t)stream);
        // op 0 changes phi: grad / normal / K / G describe the old field
        if (op == 0) g->has_grad = g->has_normal = g->has_kint = false;
    });
}
