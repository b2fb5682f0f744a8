// sg_mesh.cu -- signed distance to a closed triangle mesh (NEXT-4).
//
// "the initialization of the level-set is mainly carried out on
// CPUs ... because the sign distance function from triangle mesh
// [baerentzen2005robust] is not implemented on GPU"; P:791-794 names the GPU
// version as future work.  Reading R-24 (include/sg.h sg_geometry):
//   f(x) = s |x - q|, q the closest point of the mesh (nearest triangle by
//   squared distance, ties to the lowest triangle index; closest point on a
//   triangle by the Voronoi-region test of Ericson, RTCD 5.1.5), s the sign
//   of (x - q) . N with N the angle-weighted pseudonormal of the closest
//   feature (face normal / sum of the two face normals of an edge / sum of
//   the incident face normals weighted by their corner angles at a vertex).
// Compiled with -fmad=false: every fp64 operation rounds separately in the
// order written, so |f| -- and with it the core test |f(centre)| < l_c -- is
// bit-identical to any IEEE evaluation in the same order.
//
// Device work: triangles are binned per background cell (CSR over cells,
// triangle AABB dilated by the bin radius rb = 4 l_c); a query point inside
// cell c scans c's bin, so the result is exact whenever |f| <= rb (every
// triangle nearer than rb is in the bin).  Cells with |f(centre)| > rb are
// "unknown": only their sign is needed, and the build takes it from the
// coarse sign flood of the sign correction, seeded by the known
// cells.  Host work, O(n_tris) once per build: pseudonormals (edge
// adjacency by hashing) -- the mesh's preprocessing, not the per-point path.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <unordered_map>
#include <vector>

#include "sg_internal.cuh"

namespace sg {

// ------------------------------------------------------------ host prep ---

static inline double dot3(const double* a, const double* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

struct MeshHost {
    std::vector<double> fn, en, vn, sph;
};

// pseudonormals (R-24): unit face normals n = (b - a) x (c - a) / |.|; an
// edge's normal is n_t + n_t' of its two faces (n_t alone on a border edge);
// a vertex's is the sum over its corners, in triangle order, of angle * n_t
static MeshHost mesh_normals(const double* V, const int32_t* T, int nv, int nt) {
    MeshHost h;
    h.fn.assign((size_t)nt * 3, 0.0);
    h.en.assign((size_t)nt * 9, 0.0);
    h.vn.assign((size_t)nv * 3, 0.0);
    h.sph.assign((size_t)nt * 4, 0.0);
    for (int t = 0; t < nt; ++t) {  // bounding spheres (pruning only, never a result)
        double c[3] = {0.0, 0.0, 0.0}, r2 = 0.0;
        for (int v = 0; v < 3; ++v)
            for (int k = 0; k < 3; ++k) c[k] += V[3 * T[3 * t + v] + k] / 3.0;
        for (int v = 0; v < 3; ++v) {
            const double e[3] = {V[3 * T[3 * t + v]] - c[0], V[3 * T[3 * t + v] + 1] - c[1],
                                 V[3 * T[3 * t + v] + 2] - c[2]};
            r2 = std::max(r2, dot3(e, e));
        }
        for (int k = 0; k < 3; ++k) h.sph[4 * t + k] = c[k];
        h.sph[4 * t + 3] = std::sqrt(r2) * (1.0 + 1e-12) + 1e-300;
    }
    for (int t = 0; t < nt; ++t) {
        const double* a = V + 3 * T[3 * t];
        const double* b = V + 3 * T[3 * t + 1];
        const double* c = V + 3 * T[3 * t + 2];
        const double ab[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        const double ac[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        const double n[3] = {ab[1] * ac[2] - ab[2] * ac[1], ab[2] * ac[0] - ab[0] * ac[2],
                             ab[0] * ac[1] - ab[1] * ac[0]};
        const double l = std::sqrt(dot3(n, n));
        for (int k = 0; k < 3; ++k) h.fn[3 * t + k] = l > 0.0 ? n[k] / l : 0.0;
    }
    for (int t = 0; t < nt; ++t) {
        for (int k = 0; k < 3; ++k) {
            const int i = T[3 * t + k], j = T[3 * t + (k + 1) % 3], m = T[3 * t + (k + 2) % 3];
            const double* p = V + 3 * i;
            const double u[3] = {V[3 * j] - p[0], V[3 * j + 1] - p[1], V[3 * j + 2] - p[2]};
            const double w[3] = {V[3 * m] - p[0], V[3 * m + 1] - p[1], V[3 * m + 2] - p[2]};
            const double lu = std::sqrt(dot3(u, u)), lw = std::sqrt(dot3(w, w));
            double cs = (lu > 0.0 && lw > 0.0) ? dot3(u, w) / (lu * lw) : 1.0;
            cs = std::min(1.0, std::max(-1.0, cs));
            const double ang = std::acos(cs);
            for (int q = 0; q < 3; ++q) h.vn[3 * i + q] += ang * h.fn[3 * t + q];
        }
    }
    std::unordered_map<uint64_t, int> half;  // directed edge (i -> j) -> 3 t + e
    half.reserve((size_t)nt * 3);
    for (int t = 0; t < nt; ++t)
        for (int e = 0; e < 3; ++e) {
            const uint32_t i = (uint32_t)T[3 * t + e], j = (uint32_t)T[3 * t + (e + 1) % 3];
            half[((uint64_t)i << 32) | j] = 3 * t + e;
        }
    for (int t = 0; t < nt; ++t)
        for (int e = 0; e < 3; ++e) {
            const uint32_t i = (uint32_t)T[3 * t + e], j = (uint32_t)T[3 * t + (e + 1) % 3];
            auto it = half.find(((uint64_t)j << 32) | i);
            for (int q = 0; q < 3; ++q) {
                const double o = it == half.end() ? 0.0 : h.fn[3 * (it->second / 3) + q];
                h.en[9 * t + 3 * e + q] = it == half.end() ? h.fn[3 * t + q] : h.fn[3 * t + q] + o;
            }
        }
    return h;
}

// ---------------------------------------------------------------- bins ----

struct BinC {
    double lower[3], cell, rb;
    int32_t n[3];
};

__device__ __forceinline__ void tri_cells(const BinC& b, const double* __restrict__ V,
                                          const int32_t* __restrict__ T, int t, int (&lo)[3],
                                          int (&hi)[3]) {
    const double* p0 = V + 3 * T[3 * t];
    const double* p1 = V + 3 * T[3 * t + 1];
    const double* p2 = V + 3 * T[3 * t + 2];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double mn = fmin(p0[k], fmin(p1[k], p2[k])) - b.rb;
        const double mx = fmax(p0[k], fmax(p1[k], p2[k])) + b.rb;
        lo[k] = max(0, (int)floor((mn - b.lower[k]) / b.cell));
        hi[k] = min(b.n[k] - 1, (int)floor((mx - b.lower[k]) / b.cell));
    }
}

// cell (x, y, z) within rb of the triangle's AABB (box-box distance); the
// cell range of tri_cells is the AABB dilated by rb, this drops its corners
__device__ __forceinline__ bool cell_near(const BinC& b, const double* __restrict__ V,
                                          const int32_t* __restrict__ T, int t, int x, int y,
                                          int z) {
    const int c[3] = {x, y, z};
    double d2 = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double mn = fmin(V[3 * T[3 * t] + k], fmin(V[3 * T[3 * t + 1] + k], V[3 * T[3 * t + 2] + k]));
        const double mx = fmax(V[3 * T[3 * t] + k], fmax(V[3 * T[3 * t + 1] + k], V[3 * T[3 * t + 2] + k]));
        const double lo = b.lower[k] + (double)c[k] * b.cell, hi = lo + b.cell;
        const double gap = fmax(0.0, fmax(lo - mx, mn - hi));
        d2 += gap * gap;
    }
    return d2 <= b.rb * b.rb * 1.0000001;  // conservative
}

__global__ void k_bin_count(BinC b, const double* __restrict__ V, const int32_t* __restrict__ T,
                            int nt, uint32_t* __restrict__ cnt) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    int lo[3], hi[3];
    tri_cells(b, V, T, t, lo, hi);
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x)
                if (cell_near(b, V, T, t, x, y, z))
                    atomicAdd(cnt + ((int64_t)z * b.n[1] + y) * b.n[0] + x, 1u);
}

__global__ void k_bin_fill(BinC b, const double* __restrict__ V, const int32_t* __restrict__ T,
                           int nt, const uint32_t* __restrict__ off, uint32_t* __restrict__ cur,
                           uint32_t* __restrict__ tri) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    int lo[3], hi[3];
    tri_cells(b, V, T, t, lo, hi);
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x) {
                if (!cell_near(b, V, T, t, x, y, z)) continue;
                const int64_t c = ((int64_t)z * b.n[1] + y) * b.n[0] + x;
                tri[off[c] + atomicAdd(cur + c, 1u)] = (uint32_t)t;
            }
}

// ------------------------------------------------------------- distance ---

// closest point q of p on triangle (a, b, c) (Ericson, RTCD 5.1.5); returns
// the Voronoi region: 0 face, 1/2/3 vertex a/b/c, 4/5/6 edge ab/bc/ca
__device__ __forceinline__ int tri_closest(const double* a, const double* b, const double* c,
                                           const double* p, double* q) {
    const double ab[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    const double ac[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    const double ap[3] = {p[0] - a[0], p[1] - a[1], p[2] - a[2]};
    const double d1 = (ab[0] * ap[0] + ab[1] * ap[1]) + ab[2] * ap[2];
    const double d2 = (ac[0] * ap[0] + ac[1] * ap[1]) + ac[2] * ap[2];
    if (d1 <= 0.0 && d2 <= 0.0) {
        q[0] = a[0]; q[1] = a[1]; q[2] = a[2];
        return 1;
    }
    const double bp[3] = {p[0] - b[0], p[1] - b[1], p[2] - b[2]};
    const double d3 = (ab[0] * bp[0] + ab[1] * bp[1]) + ab[2] * bp[2];
    const double d4 = (ac[0] * bp[0] + ac[1] * bp[1]) + ac[2] * bp[2];
    if (d3 >= 0.0 && d4 <= d3) {
        q[0] = b[0]; q[1] = b[1]; q[2] = b[2];
        return 2;
    }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double v = d1 / (d1 - d3);
        q[0] = a[0] + v * ab[0]; q[1] = a[1] + v * ab[1]; q[2] = a[2] + v * ab[2];
        return 4;
    }
    const double cp[3] = {p[0] - c[0], p[1] - c[1], p[2] - c[2]};
    const double d5 = (ab[0] * cp[0] + ab[1] * cp[1]) + ab[2] * cp[2];
    const double d6 = (ac[0] * cp[0] + ac[1] * cp[1]) + ac[2] * cp[2];
    if (d6 >= 0.0 && d5 <= d6) {
        q[0] = c[0]; q[1] = c[1]; q[2] = c[2];
        return 3;
    }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double w = d2 / (d2 - d6);
        q[0] = a[0] + w * ac[0]; q[1] = a[1] + w * ac[1]; q[2] = a[2] + w * ac[2];
        return 6;
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        q[0] = b[0] + w * (c[0] - b[0]); q[1] = b[1] + w * (c[1] - b[1]);
        q[2] = b[2] + w * (c[2] - b[2]);
        return 5;
    }
    const double den = 1.0 / ((va + vb) + vc);
    const double v = vb * den, w = vc * den;
    q[0] = (a[0] + ab[0] * v) + ac[0] * w;
    q[1] = (a[1] + ab[1] * v) + ac[1] * w;
    q[2] = (a[2] + ab[2] * v) + ac[2] * w;
    return 0;
}

// lower bound test: the triangle (bounding sphere c, r) is farther from p
// than sqrt(best) (sb): |p - c| > sb + r.  With the relative margin a skipped
// triangle is strictly farther than the best one, so skipping never changes
// the nearest triangle (ties included).
__device__ __forceinline__ bool farther(const double* sph, const double* p, double sb) {
    const double e0 = p[0] - sph[0], e1 = p[1] - sph[1], e2 = p[2] - sph[2];
    const double lim = sb + sph[3];
    return (e0 * e0 + e1 * e1) + e2 * e2 > lim * lim * 1.000000001;
}

// signed distance of p (inside background cell `cell`) from the triangles of
// the cell's bin; known = false when no triangle lies within rb (the sign is
// then left to the flood and |f| is only known to exceed rb)
__device__ double mesh_sdf(const Geom& g, int64_t cell, const double* p, bool& known) {
    const uint32_t b0 = g.bin_off[cell], b1 = g.bin_off[cell + 1];
    double best = 0.0;
    int bt = -1, breg = 0;
    double bq[3] = {0.0, 0.0, 0.0};
    double sb = INFINITY;
    for (uint32_t k = b0; k < b1; ++k) {
        const int t = (int)g.bin_tri[k];
        if (bt >= 0 && farther(g.msph + 4 * t, p, sb)) continue;
        const int32_t* tv = g.mt + 3 * t;
        double q[3];
        const int reg = tri_closest(g.mv + 3 * tv[0], g.mv + 3 * tv[1], g.mv + 3 * tv[2], p, q);
        const double e0 = p[0] - q[0], e1 = p[1] - q[1], e2 = p[2] - q[2];
        const double d2 = (e0 * e0 + e1 * e1) + e2 * e2;
        if (bt < 0 || d2 < best || (d2 == best && t < bt)) {
            best = d2;
            bt = t;
            breg = reg;
            bq[0] = q[0]; bq[1] = q[1]; bq[2] = q[2];
            sb = sqrt(best);
        }
    }
    const double d = bt < 0 ? INFINITY : sqrt(best);
    known = bt >= 0 && d <= g.mesh_rb;
    if (!known) return d;
    const double* N;
    if (breg == 0) N = g.mfn + 3 * bt;
    else if (breg <= 3) N = g.mvn + 3 * g.mt[3 * bt + breg - 1];
    else N = g.men + 9 * bt + 3 * (breg - 4);
    const double s = ((p[0] - bq[0]) * N[0] + (p[1] - bq[1]) * N[1]) + (p[2] - bq[2]) * N[2];
    return s < 0.0 ? -d : d;
}

// K1 for a mesh: per 32-cell word, core = |f(centre)| < l_c, neg = f < 0,
// known = |f| <= rb (sign trustworthy; the rest is flooded)
__global__ void __launch_bounds__(256) k_tag_mesh(GridC gc, Geom g, int32_t W,
                                                  uint32_t* __restrict__ core_w,
                                                  uint32_t* __restrict__ neg_w,
                                                  uint32_t* __restrict__ known_w) {
    const int cx = blockIdx.x * blockDim.x + threadIdx.x;
    const int cy = blockIdx.y, cz = blockIdx.z;
    const bool in = cx < gc.n[0];
    double f = INFINITY;
    bool known = false;
    if (in) {
        const double p[3] = {gc.lower[0] + ((double)cx + 0.5) * gc.cell,
                             gc.lower[1] + ((double)cy + 0.5) * gc.cell,
                             gc.lower[2] + ((double)cz + 0.5) * gc.cell};
        f = mesh_sdf(g, ((int64_t)cz * gc.n[1] + cy) * gc.n[0] + cx, p, known);
    }
    const uint32_t cw = __ballot_sync(0xffffffffu, in && fabs(f) < gc.cell);
    const uint32_t nw = __ballot_sync(0xffffffffu, in && known && f < 0.0);
    const uint32_t kw = __ballot_sync(0xffffffffu, in && known);
    if ((threadIdx.x & 31) == 0 && cx < gc.n[0]) {
        const int64_t i = ((int64_t)cz * gc.n[1] + cy) * W + (cx >> 5);
        core_w[i] = cw;
        neg_w[i] = nw;
        known_w[i] = kw;
    }
}

// K1 of a refined layer for a mesh (NEXT-4 multi-resolution):
// only cells under a parent core cell are evaluated (all within 2.9 l_c < rb
// of the surface: exact); the others take the sign of their parent cell
__global__ void __launch_bounds__(256) k_tag_refine_mesh(GridC gc, Geom g, int32_t W, ParentBits pb,
                                                         uint32_t* __restrict__ core_w,
                                                         uint32_t* __restrict__ neg_w,
                                                         uint32_t* __restrict__ eval_w) {
    const int cx = blockIdx.x * blockDim.x + threadIdx.x;
    const int cy = blockIdx.y, cz = blockIdx.z;
    const bool in = cx < gc.n[0];
    bool core = false, neg = false, pc = false;
    if (in) {
        const int px = cx >> 1;
        const int64_t pw = ((int64_t)(cz >> 1) * (gc.n[1] >> 1) + (cy >> 1)) * pb.W + (px >> 5);
        pc = (__ldg(pb.core + pw) >> (px & 31)) & 1u;
        neg = (__ldg(pb.neg + pw) >> (px & 31)) & 1u;
        if (pc) {
            const double p[3] = {gc.lower[0] + ((double)cx + 0.5) * gc.cell,
                                 gc.lower[1] + ((double)cy + 0.5) * gc.cell,
                                 gc.lower[2] + ((double)cz + 0.5) * gc.cell};
            bool known;
            const double f = mesh_sdf(g, ((int64_t)cz * gc.n[1] + cy) * gc.n[0] + cx, p, known);
            core = fabs(f) < gc.cell;
            neg = f < 0.0;
        }
    }
    const uint32_t cw = __ballot_sync(0xffffffffu, in && core);
    const uint32_t nw = __ballot_sync(0xffffffffu, in && neg);
    const uint32_t ew = __ballot_sync(0xffffffffu, in && pc);
    if ((threadIdx.x & 31) == 0 && cx < gc.n[0]) {
        const int64_t i = ((int64_t)cz * gc.n[1] + cy) * W + (cx >> 5);
        core_w[i] = cw;
        neg_w[i] = nw;
        eval_w[i] = ew;
    }
}

void launch_tag_refine_mesh(const GridC& gc, const Geom& g, int32_t W, ParentBits pb,
                            uint32_t* core_w, uint32_t* neg_w, uint32_t* eval_w, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(gc.n[0], 256), (unsigned)gc.n[1], (unsigned)gc.n[2]);
    k_tag_refine_mesh<<<grid, 256, 0, s>>>(gc, g, W, pb, core_w, neg_w, eval_w);
    SG_LAUNCHED();
}

// K4 for a mesh: phi = init_scale * f at the 64 data points of each active
// package (every such point is within 3.4 l_c < rb of the surface: exact).
// One 64-thread block per package, a thread per data point; the package's
// bin is staged through shared memory in chunks of 64 triangles, so the 64
// points read each triangle's vertices once from global memory (broadcast
// shared loads afterwards).  Same nearest-triangle rule as mesh_sdf.
constexpr int kMeshChunk = 64;

template <class T>
__global__ void __launch_bounds__(64) k_phi_init_mesh(GridC gc, Geom g,
                                                      const uint32_t* __restrict__ meta_cell,
                                                      int64_t n_pkg, T* __restrict__ phi0,
                                                      T* __restrict__ phi1) {
    __shared__ double sv[kMeshChunk][9];
    __shared__ double ss[kMeshChunk][4];
    __shared__ int st[kMeshChunk];
    const int64_t id = blockIdx.x;
    const int d = threadIdx.x;
    const int64_t t = id * 64 + d;
    if (id < 2) {
        const T v = (T)(id == 0 ? -gc.far : gc.far);
        phi0[t] = v;
        phi1[t] = v;
        return;
    }
    const uint32_t L = meta_cell[id];
    const uint32_t nx = (uint32_t)gc.n[0], ny = (uint32_t)gc.n[1];
    const uint32_t r = L / nx;
    const int cx = (int)(L - r * nx), cy = (int)(r % ny), cz = (int)(r / ny);
    const double p[3] = {gc.lower[0] + ((double)(4 * (int64_t)cx + (d & 3)) + 0.5) * gc.dx,
                         gc.lower[1] + ((double)(4 * (int64_t)cy + ((d >> 2) & 3)) + 0.5) * gc.dx,
                         gc.lower[2] + ((double)(4 * (int64_t)cz + (d >> 4)) + 0.5) * gc.dx};
    const uint32_t b0 = g.bin_off[L], b1 = g.bin_off[L + 1];
    double best = 0.0, sb = INFINITY;
    int bt = -1, breg = 0;
    double bq[3] = {0.0, 0.0, 0.0};
    for (uint32_t c0 = b0; c0 < b1; c0 += kMeshChunk) {
        const int cnt = (int)(b1 - c0 < (uint32_t)kMeshChunk ? b1 - c0 : (uint32_t)kMeshChunk);
        __syncthreads();  // previous chunk consumed
        if (d < cnt) {
            const int tri = (int)g.bin_tri[c0 + d];
            st[d] = tri;
            const int32_t* tv = g.mt + 3 * tri;
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int k = 0; k < 3; ++k) sv[d][3 * v + k] = g.mv[3 * tv[v] + k];
#pragma unroll
            for (int k = 0; k < 4; ++k) ss[d][k] = g.msph[4 * tri + k];
        }
        __syncthreads();
        for (int k = 0; k < cnt; ++k) {
            if (bt >= 0 && farther(ss[k], p, sb)) continue;
            double q[3];
            const int reg = tri_closest(&sv[k][0], &sv[k][3], &sv[k][6], p, q);
            const double e0 = p[0] - q[0], e1 = p[1] - q[1], e2 = p[2] - q[2];
            const double d2 = (e0 * e0 + e1 * e1) + e2 * e2;
            const int tri = st[k];
            if (bt < 0 || d2 < best || (d2 == best && tri < bt)) {
                best = d2;
                bt = tri;
                breg = reg;
                bq[0] = q[0]; bq[1] = q[1]; bq[2] = q[2];
                sb = sqrt(best);
            }
        }
    }
    double f = INFINITY;
    if (bt >= 0) {
        const double dd = sqrt(best);
        const double* N;
        if (breg == 0) N = g.mfn + 3 * bt;
        else if (breg <= 3) N = g.mvn + 3 * g.mt[3 * bt + breg - 1];
        else N = g.men + 9 * bt + 3 * (breg - 4);
        const double sgn = ((p[0] - bq[0]) * N[0] + (p[1] - bq[1]) * N[1]) + (p[2] - bq[2]) * N[2];
        f = sgn < 0.0 ? -dd : dd;
    }
    phi0[t] = (T)(gc.init_scale * f);
}

// ---------------------------------------------------------------- host ----

MeshDev mesh_prepare(const GridC& gc, const sg_geometry* geom, Geom& g, cudaStream_t s) {
    const int nv = geom->n_verts, nt = geom->n_tris;
    MeshHost h = mesh_normals(geom->verts, geom->tris, nv, nt);
    const int64_t ncell = (int64_t)gc.n[0] * gc.n[1] * gc.n[2];
    MeshDev m;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t sv = al(sizeof(double) * 3 * nv), st = al(sizeof(int32_t) * 3 * nt),
                 sfn = al(sizeof(double) * 3 * nt), sen = al(sizeof(double) * 9 * nt),
                 svn = al(sizeof(double) * 3 * nv), ssp = al(sizeof(double) * 4 * nt),
                 soff = al(sizeof(uint32_t) * (ncell + 1)),
                 scur = al(sizeof(uint32_t) * (ncell + 1));
    char* base = (char*)dalloc(sv + st + sfn + sen + svn + ssp + soff + scur, s);
    m.allocs.push_back(base);
    double* V = (double*)base;
    int32_t* T = (int32_t*)(base + sv);
    double* fn = (double*)(base + sv + st);
    double* en = (double*)(base + sv + st + sfn);
    double* vn = (double*)(base + sv + st + sfn + sen);
    double* sph = (double*)(base + sv + st + sfn + sen + svn);
    uint32_t* off = (uint32_t*)(base + sv + st + sfn + sen + svn + ssp);
    uint32_t* cur = (uint32_t*)(base + sv + st + sfn + sen + svn + ssp + soff);
    SG_CUDA(cudaMemcpyAsync(V, geom->verts, sizeof(double) * 3 * nv, cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(T, geom->tris, sizeof(int32_t) * 3 * nt, cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(fn, h.fn.data(), sizeof(double) * 3 * nt, cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(en, h.en.data(), sizeof(double) * 9 * nt, cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(vn, h.vn.data(), sizeof(double) * 3 * nv, cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(sph, h.sph.data(), sizeof(double) * 4 * nt, cudaMemcpyHostToDevice, s));
    BinC b;
    for (int k = 0; k < 3; ++k) {
        b.lower[k] = gc.lower[k];
        b.n[k] = gc.n[k];
    }
    b.cell = gc.cell;
    b.rb = 4.0 * gc.cell;
    SG_CUDA(cudaMemsetAsync(cur, 0, sizeof(uint32_t) * (ncell + 1), s));
    k_bin_count<<<(unsigned)ceil_div(nt, 128), 128, 0, s>>>(b, V, T, nt, cur);
    SG_LAUNCHED();
    size_t tmp_bytes = 0;
    SG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cur, off, (int)(ncell + 1), s));
    void* tmp = dalloc(tmp_bytes, s);
    SG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cur, off, (int)(ncell + 1), s));
    SG_CUDA(cudaFreeAsync(tmp, s));
    uint32_t total = 0;
    SG_CUDA(cudaMemcpyAsync(&total, off + ncell, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    uint32_t* tri = (uint32_t*)dalloc(sizeof(uint32_t) * std::max<uint32_t>(total, 1), s);
    m.allocs.push_back(tri);
    SG_CUDA(cudaMemsetAsync(cur, 0, sizeof(uint32_t) * (ncell + 1), s));
    k_bin_fill<<<(unsigned)ceil_div(nt, 128), 128, 0, s>>>(b, V, T, nt, off, cur, tri);
    SG_LAUNCHED();
    g.mesh_nt = nt;
    g.mesh_nv = nv;
    g.mv = V;
    g.mt = T;
    g.mfn = fn;
    g.men = en;
    g.mvn = vn;
    g.msph = sph;
    g.bin_off = off;
    g.bin_tri = tri;
    g.mesh_rb = b.rb;
    m.bin_entries = total;
    return m;
}

void mesh_release(MeshDev& m, cudaStream_t s) {
    for (void* p : m.allocs) cudaFreeAsync(p, s);
    m.allocs.clear();
}

void launch_tag_mesh(const GridC& gc, const Geom& g, int32_t W, uint32_t* core_w, uint32_t* neg_w,
                     uint32_t* known_w, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(gc.n[0], 256), (unsigned)gc.n[1], (unsigned)gc.n[2]);
    k_tag_mesh<<<grid, 256, 0, s>>>(gc, g, W, core_w, neg_w, known_w);
    SG_LAUNCHED();
}

void launch_phi_init_mesh(const GridC& gc, const Geom& g, const uint32_t* meta_cell,
                          int64_t n_pkg, int32_t dtype, void* phi0, void* phi1, cudaStream_t s) {
    const unsigned blocks = (unsigned)n_pkg;
    if (dtype == SG_F64)
        k_phi_init_mesh<double><<<blocks, 64, 0, s>>>(gc, g, meta_cell, n_pkg, (double*)phi0,
                                                     (double*)phi1);
    else
        k_phi_init_mesh<float><<<blocks, 64, 0, s>>>(gc, g, meta_cell, n_pkg, (float*)phi0,
                                                    (float*)phi1);
    SG_LAUNCHED();
}

}  // namespace sg
