// sg_relax.cu -- SPH particle relaxation against the level set (NEXT-2).
//
// "The SPH particle relaxation is a typical grid-particle coupling
// algorithm in which the integral field is interpolated by bi- or tri-linear
// interpolation to the particle's position and used in the form of surface
// force to drive the particle."  Force law and bounding: reading R-21
// (include/sg.h sg_relax).
//
// One relaxation step on the device:
//   k_rl_key     cell of every particle in a uniform cell-linked list of cell
//                size 2h, per-cell counts
//   k_rl_scan*   exclusive scan of the cell counts (block sums + one block)
//   k_rl_scatter particles copied into cell order (atomic cursors)
//   k_rl_force   pair sum over the 27 neighbour cells + trilinear G (the
//                kernel-gradient integral) through the package neighbour row
//                (Lst. 2), displacement, clamp -> new position
//   k_rl_bound   trilinear (phi, grad phi) at the new position, projection
//                of particles closer than surface_offset to the surface
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "sg_internal.cuh"

namespace sg {

struct RelaxC {
    double lower[3], upper[3];
    double cs, inv_cs;  // cell-list cell size h (pairs within 2h: +-2 cells)
    int32_t nc[3];      // cell-list cells per axis
    double h, two_h, sigma, vol;  // Wendland C2, particle volume dp^3
    double step_dp2, max_d, off;  // step dp^2, max_disp dp, surface_offset dp
};

// trilinear interpolation of C components of a package field at x (inside an
// active cell): corners through the containing package's neighbour row
// (Lst. 2, shifts in [-1, 4]).  cstride / pstride: element strides of a
// component / a package; dstride: stride of a data point.
template <class T, int C>
__device__ __forceinline__ void interp(const GridC& gc, const uint32_t* __restrict__ nb,
                                       uint32_t b, const double (&x)[3], const int (&c)[3],
                                       const T* __restrict__ f, int pstride, int dstride,
                                       int cstride, T (&out)[C]) {
    int s[3];
    T t[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double u = (x[k] - gc.lower[k]) / gc.dx - 0.5;
        const double a = floor(u);
        t[k] = (T)(u - a);
        s[k] = (int)a - 4 * c[k];
    }
#pragma unroll
    for (int e = 0; e < C; ++e) out[e] = T(0);
    const uint32_t* row = nb + (size_t)b * 27;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int bx = q & 1, by = (q >> 1) & 1, bz = q >> 2;
        const int sx = s[0] + bx, sy = s[1] + by, sz = s[2] + bz;
        const Shift hx = nb_shift(sx), hy = nb_shift(sy), hz = nb_shift(sz);
        const int d = hx.data + 4 * hy.data + 16 * hz.data;
        const size_t pk = __ldg(row + hx.off + 3 * hy.off + 9 * hz.off);
        const T w = ((bx ? t[0] : T(1) - t[0]) * (by ? t[1] : T(1) - t[1])) *
                    (bz ? t[2] : T(1) - t[2]);
        const T* p = f + pk * pstride + (size_t)d * dstride;
#pragma unroll
        for (int e = 0; e < C; ++e) out[e] += w * __ldg(p + e * cstride);
    }
}

// containing grid cell and its package (0/1 = far field); false if outside
// the owned domain
__device__ __forceinline__ bool locate(const GridC& gc, const uint32_t* __restrict__ bg,
                                       const double (&x)[3], int (&c)[3], uint32_t& b) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (!(x[k] >= gc.lower[k] && x[k] < gc.upper[k])) return false;
        c[k] = min((int)floor((x[k] - gc.lower[k]) / gc.cell), gc.n[k] - 1);
    }
    if (c[2] < gc.z_lo || c[2] >= gc.z_hi) return false;
    b = __ldg(bg + ((int64_t)(c[2] - gc.zs_lo) * gc.n[1] + c[1]) * gc.n[0] + c[0]);
    return true;
}

__device__ __forceinline__ int64_t rl_cell(const RelaxC& r, const double (&x)[3], bool& in) {
    int ci[3];
    in = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        in = in && x[k] >= r.lower[k] && x[k] < r.upper[k];
        ci[k] = min(max((int)floor((x[k] - r.lower[k]) * r.inv_cs), 0), r.nc[k] - 1);
    }
    return ((int64_t)ci[2] * r.nc[1] + ci[1]) * r.nc[0] + ci[0];
}

template <class T>
__global__ void k_rl_key(RelaxC r, int64_t n, const T* __restrict__ pos, int32_t* __restrict__ key,
                         int32_t* __restrict__ count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x[3] = {(double)pos[3 * i], (double)pos[3 * i + 1], (double)pos[3 * i + 2]};
    bool in;
    const int64_t c = rl_cell(r, x, in);
    key[i] = in ? (int32_t)c : -1;
    if (in) atomicAdd(count + c, 1);
}

// exclusive scan of int32 counts: 1024 per block, then the block sums
constexpr int kScanB = 1024;

__global__ void __launch_bounds__(kScanB) k_rl_scan_blocks(int32_t* __restrict__ v, int64_t n,
                                                           int32_t* __restrict__ bsum) {
    __shared__ int32_t s[kScanB];
    const int64_t i = (int64_t)blockIdx.x * kScanB + threadIdx.x;
    const int32_t x = i < n ? v[i] : 0;
    s[threadIdx.x] = x;
    __syncthreads();
    for (int o = 1; o < kScanB; o <<= 1) {
        const int32_t y = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0;
        __syncthreads();
        s[threadIdx.x] += y;
        __syncthreads();
    }
    if (i < n) v[i] = s[threadIdx.x] - x;  // exclusive within the block
    if (threadIdx.x == kScanB - 1) bsum[blockIdx.x] = s[kScanB - 1];
}

__global__ void __launch_bounds__(kScanB) k_rl_scan_sums(int32_t* __restrict__ bsum, int64_t nb) {
    __shared__ int32_t s[kScanB];
    int32_t carry = 0;
    for (int64_t base = 0; base < nb; base += kScanB) {
        const int64_t i = base + threadIdx.x;
        const int32_t x = i < nb ? bsum[i] : 0;
        s[threadIdx.x] = x;
        __syncthreads();
        for (int o = 1; o < kScanB; o <<= 1) {
            const int32_t y = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0;
            __syncthreads();
            s[threadIdx.x] += y;
            __syncthreads();
        }
        if (i < nb) bsum[i] = carry + s[threadIdx.x] - x;
        const int32_t tot = s[kScanB - 1];
        __syncthreads();
        carry += tot;
    }
}

__global__ void k_rl_scan_add(int32_t* __restrict__ v, int64_t n, const int32_t* __restrict__ bsum) {
    const int64_t i = (int64_t)blockIdx.x * kScanB + threadIdx.x;
    if (i < n) v[i] += bsum[blockIdx.x];
}

__device__ __forceinline__ void ld4(const float* p, float (&v)[4]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

template <class T>
__global__ void k_rl_scatter(int64_t n, const T* __restrict__ pos, const int32_t* __restrict__ key,
                             const int32_t* __restrict__ start, int32_t* __restrict__ cursor,
                             T* __restrict__ spos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || key[i] < 0) return;
    // slots < n < 2^31 (sg_relax checks); the x3 offsets in 64 bit
    const int64_t slot = start[key[i]] + atomicAdd(cursor + key[i], 1);
    // 4 values per particle: one vector load per pair candidate
    spos[4 * slot] = pos[3 * i];
    spos[4 * slot + 1] = pos[3 * i + 1];
    spos[4 * slot + 2] = pos[3 * i + 2];
    spos[4 * slot + 3] = T(0);
}

template <class T>
__global__ void __launch_bounds__(256) k_rl_force(GridC gc, RelaxC r, int64_t n,
                                                  const T* __restrict__ pos,
                                                  const int32_t* __restrict__ key,
                                                  const int32_t* __restrict__ start,
                                                  const int32_t* __restrict__ cnt,
                                                  const T* __restrict__ spos,
                                                  const uint32_t* __restrict__ bg,
                                                  const uint32_t* __restrict__ nb,
                                                  const T* __restrict__ G, T* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x[3] = {(double)pos[3 * i], (double)pos[3 * i + 1], (double)pos[3 * i + 2]};
    int c[3];
    uint32_t b = 0;
    if (key[i] < 0 || !locate(gc, bg, x, c, b)) {  // outside: unchanged
        out[3 * i] = pos[3 * i];
        out[3 * i + 1] = pos[3 * i + 1];
        out[3 * i + 2] = pos[3 * i + 2];
        return;
    }
    // pair sum  sum_j V grad W(x_i - x_j)
    const int k0 = key[i];
    const int cx = k0 % r.nc[0], cy = (k0 / r.nc[0]) % r.nc[1], cz = k0 / (r.nc[0] * r.nc[1]);
    T sx = T(0), sy = T(0), sz = T(0);
    const T xi = (T)x[0], yi = (T)x[1], zi = (T)x[2];
    const T inv_h = (T)(1.0 / r.h), two_h2 = (T)(r.two_h * r.two_h);
    const T coef = (T)(-5.0 * r.sigma / (r.h * r.h) * r.vol);  // W'(r)/r = coef (1 - q/2)^3
    // cells of size h: the partners within 2h lie in the 5 x 5 x 5 cells
    // around; the 5 cells of one (y, z) row are consecutive in the sorted
    // array, so each row is one contiguous range
    const int xa = max(cx - 2, 0), xb = min(cx + 2, r.nc[0] - 1);
    for (int dz = -2; dz <= 2; ++dz) {
        const int z = cz + dz;
        if (z < 0 || z >= r.nc[2]) continue;
        for (int dy = -2; dy <= 2; ++dy) {
            const int y = cy + dy;
            if (y < 0 || y >= r.nc[1]) continue;
            {
                const int64_t row = ((int64_t)z * r.nc[1] + y) * r.nc[0];
                const int32_t s0 = start[row + xa], s1 = start[row + xb] + cnt[row + xb];
#pragma unroll 4
                for (int64_t jj = s0; jj < s1; ++jj) {
                    T pj[4];
                    ld4(spos + 4 * jj, pj);
                    const T ex = xi - pj[0], ey = yi - pj[1], ez = zi - pj[2];
                    const T d2 = ex * ex + ey * ey + ez * ez;
                    if (d2 > T(0) && d2 < two_h2) {
                        const T q = sqrt(d2) * inv_h;
                        const T a = T(1) - T(0.5) * q;
                        const T f = coef * a * a * a;  // W'(|r|) / |r| * V  (q/h factor folded)
                        sx += f * ex;
                        sy += f * ey;
                        sz += f * ez;
                    }
                }
            }
        }
    }
    // surface force: G(x_i) interpolated from the grid (zero in the far field)
    T g[3] = {T(0), T(0), T(0)};
    if (b >= 2) interp<T, 3>(gc, nb, b, x, c, G, 192, 1, 64, g);
    T ax = T(-2) * (sx - g[0]), ay = T(-2) * (sy - g[1]), az = T(-2) * (sz - g[2]);
    T ddx = (T)r.step_dp2 * ax, ddy = (T)r.step_dp2 * ay, ddz = (T)r.step_dp2 * az;
    const T len = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    if (len > (T)r.max_d) {
        const T sc = (T)r.max_d / len;
        ddx *= sc;
        ddy *= sc;
        ddz *= sc;
    }
    out[3 * i] = xi + ddx;
    out[3 * i + 1] = yi + ddy;
    out[3 * i + 2] = zi + ddz;
}

template <class T>
__global__ void __launch_bounds__(256) k_rl_bound(GridC gc, RelaxC r, int64_t n,
                                                  const T* __restrict__ moved,
                                                  const uint32_t* __restrict__ bg,
                                                  const uint32_t* __restrict__ nb,
                                                  const T* __restrict__ pg, T* __restrict__ pos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x[3] = {(double)moved[3 * i], (double)moved[3 * i + 1], (double)moved[3 * i + 2]};
    int c[3];
    uint32_t b = 0;
    T v[4] = {T(0), T(0), T(0), T(0)};
    bool have = false;
    if (locate(gc, bg, x, c, b)) {
        if (b >= 2) {
            interp<T, 4>(gc, nb, b, x, c, pg, 256, 4, 1, v);  // (phi, grad phi)
        } else {
            v[0] = (T)(b == 0 ? -gc.far : gc.far);
        }
        have = true;
    }
    T px = moved[3 * i], py = moved[3 * i + 1], pz = moved[3 * i + 2];
    const T off = (T)r.off;
    if (have && v[0] > -off) {
        const T m2 = v[1] * v[1] + v[2] * v[2] + v[3] * v[3];
        if (m2 > T(0)) {
            const T s = (v[0] + off) / sqrt(m2);
            px -= s * v[1];
            py -= s * v[2];
            pz -= s * v[3];
        }
    }
    pos[3 * i] = px;
    pos[3 * i + 1] = py;
    pos[3 * i + 2] = pz;
}

template <class T>
static void relax_t(sg_grid* g, int64_t n, T* pos, const sg_relax_params* p, cudaStream_t s) {
    const GridC& gc = g->gc;
    RelaxC r{};
    r.h = p->h_ratio * p->dp;
    r.two_h = 2.0 * r.h;
    r.cs = r.h;
    r.inv_cs = 1.0 / r.cs;
    int64_t C = 1;
    for (int k = 0; k < 3; ++k) {
        r.lower[k] = gc.lower[k];
        r.upper[k] = gc.upper[k];
        r.nc[k] = std::max(1, (int)std::ceil((gc.upper[k] - gc.lower[k]) * r.inv_cs));
        C *= r.nc[k];
    }
    SG_ARG(C < (1LL << 31), "sg_relax: cell list too large (dp too small for the domain)");
    const double pi = 3.14159265358979323846;
    r.sigma = 21.0 / (16.0 * pi * r.h * r.h * r.h);
    r.vol = p->dp * p->dp * p->dp;
    r.step_dp2 = p->step * p->dp * p->dp;
    r.max_d = p->max_disp * p->dp;
    r.off = p->surface_offset * p->dp;

    const int64_t nsb = ceil_div(C, kScanB);
    int32_t* key = (int32_t*)dalloc(sizeof(int32_t) * n, s);
    int32_t* start = (int32_t*)dalloc(sizeof(int32_t) * C, s);
    int32_t* cnt = (int32_t*)dalloc(sizeof(int32_t) * C, s);
    int32_t* bsum = (int32_t*)dalloc(sizeof(int32_t) * nsb, s);
    T* spos = (T*)dalloc(sizeof(T) * 4 * n, s);
    T* moved = (T*)dalloc(sizeof(T) * 3 * n, s);
    const unsigned pb = (unsigned)ceil_div(n, 256);
    for (int it = 0; it < p->steps; ++it) {
        SG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * C, s));
        k_rl_key<T><<<pb, 256, 0, s>>>(r, n, pos, key, cnt);
        SG_LAUNCHED();
        SG_CUDA(cudaMemcpyAsync(start, cnt, sizeof(int32_t) * C, cudaMemcpyDeviceToDevice, s));
        k_rl_scan_blocks<<<(unsigned)nsb, kScanB, 0, s>>>(start, C, bsum);
        SG_LAUNCHED();
        k_rl_scan_sums<<<1, kScanB, 0, s>>>(bsum, nsb);
        SG_LAUNCHED();
        k_rl_scan_add<<<(unsigned)nsb, kScanB, 0, s>>>(start, C, bsum);
        SG_LAUNCHED();
        // cursors: reuse bsum-free scratch -> zeroed cnt copy
        int32_t* cursor = (int32_t*)dalloc(sizeof(int32_t) * C, s);
        SG_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * C, s));
        k_rl_scatter<T><<<pb, 256, 0, s>>>(n, pos, key, start, cursor, spos);
        SG_LAUNCHED();
        SG_CUDA(cudaFreeAsync(cursor, s));
        k_rl_force<T><<<pb, 256, 0, s>>>(gc, r, n, pos, key, start, cnt, spos, g->bg, g->nb,
                                         (const T*)g->gkint, moved);
        SG_LAUNCHED();
        k_rl_bound<T><<<pb, 256, 0, s>>>(gc, r, n, moved, g->bg, g->nb, (const T*)g->grad, pos);
        SG_LAUNCHED();
    }
    for (void* q : {(void*)key, (void*)start, (void*)cnt, (void*)bsum, (void*)spos, (void*)moved})
        SG_CUDA(cudaFreeAsync(q, s));
}

}  // namespace sg

using namespace sg;

extern "C" sg_status sg_relax(sg_grid* g, int64_t n, void* pos, const sg_relax_params* p,
                              void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_relax");
        SG_ARG(g != nullptr && p != nullptr, "sg_relax: null argument");
        SG_ARG(n >= 0 && (n == 0 || pos != nullptr), "sg_relax: bad particle buffer");
        // cell-list slots and prefix sums are int32
        SG_ARG(n < (1LL << 31), "sg_relax: at most 2^31 - 1 particles per call");
        SG_ARG(p->dp > 0.0 && p->h_ratio >= 0.5 && p->h_ratio <= 2.0 && p->steps >= 0 &&
                   p->max_disp >= 0.0 && p->surface_offset >= 0.0,
               "sg_relax: bad parameters");
        if (!g->has_grad || !g->has_kint)
            throw Error(SG_ERR_STATE, "sg_relax: needs sg_gradient(SG_GRAD | SG_KINT) first");
        if (n == 0 || p->steps == 0) return;
        SG_CUDA(cudaGetLastError());
        if (g->dtype == SG_F64)
            relax_t<double>(g, n, (double*)pos, p, (cudaStream_t)stream);
        else
            relax_t<float>(g, n, (float*)pos, p, (cudaStream_t)stream);
    });
}
