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

#include <cmath>
#include <cstring>
#include <vector>

#include "sg_internal.cuh"

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
__device__ __forceinline__ void st_row(float* p, const float (&r)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
}
__device__ __forceinline__ void st_row(double* p, const double (&r)[4]) {
    reinterpret_cast<double2*>(p)[0] = make_double2(r[0], r[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(r[2], r[3]);
}

// neighbour-table slot of the six face neighbours, Lst. 2 offsets (R-8):
// r = 0..5 -> -x, +x, -y, +y, -z, +z
__device__ __forceinline__ int face_slot(int r) {
    // slot = ox + 3 oy + 9 oz, o in {0,1,2}; centre = 13
    return r == 0 ? 12 : r == 1 ? 14 : r == 2 ? 10 : r == 3 ? 16 : r == 4 ? 4 : 22;
}

// The 7-point cross of one x-row: own row c, rows ym/yp/zm/zp and the two
// x-end values xm/xp.  Lst. 2 with shifts -1 and 4 (the only ones a
// radius-1 stencil produces): shift -1 -> (offset 0, data 3), 4 -> (2, 0).
template <class T>
struct Cross {
    T c[4], ym[4], yp[4], zm[4], zp[4];
    T xm, xp;
};

template <class T>
__device__ __forceinline__ bool load_cross(const T* __restrict__ in, const uint32_t* __restrict__ nb,
                                           int64_t pkg, bool valid, Cross<T>& x) {
    const int r = threadIdx.x & 15;
    const int j = r & 3, k = r >> 2;
    uint32_t f = 0;
    if (valid && r < 6) f = __ldg(nb + pkg * 27 + face_slot(r));
    const int base = threadIdx.x & 16;
    const uint32_t nxm = __shfl_sync(0xffffffffu, f, base + 0);
    const uint32_t nxp = __shfl_sync(0xffffffffu, f, base + 1);
    const uint32_t nym = __shfl_sync(0xffffffffu, f, base + 2);
    const uint32_t nyp = __shfl_sync(0xffffffffu, f, base + 3);
    const uint32_t nzm = __shfl_sync(0xffffffffu, f, base + 4);
    const uint32_t nzp = __shfl_sync(0xffffffffu, f, base + 5);
    if (!valid) return false;
    const T* P = in + pkg * 64;
    ld_row(P + 4 * r, x.c);
    ld_row(j > 0 ? P + 4 * (r - 1) : in + (int64_t)nym * 64 + 4 * (3 + 4 * k), x.ym);
    ld_row(j < 3 ? P + 4 * (r + 1) : in + (int64_t)nyp * 64 + 4 * (0 + 4 * k), x.yp);
    ld_row(k > 0 ? P + 4 * (r - 4) : in + (int64_t)nzm * 64 + 4 * (j + 12), x.zm);
    ld_row(k < 3 ? P + 4 * (r + 4) : in + (int64_t)nzp * 64 + 4 * j, x.zp);
    x.xm = __ldg(in + (int64_t)nxm * 64 + 4 * r + 3);
    x.xp = __ldg(in + (int64_t)nxp * 64 + 4 * r);
    return true;
}

template <class T>
struct StC {
    T inv_dx, dx2, cdx, inv_2dx;
};

__device__ __forceinline__ float rs_scale(float p, float dx2) { return p * rsqrtf(fmaf(p, p, dx2)); }
__device__ __forceinline__ double rs_scale(double p, double dx2) { return p / sqrt(p * p + dx2); }

// O7 (reading R-12): one Jacobi Godunov step at one data point
template <class T>
__device__ __forceinline__ T godunov(T p, T xm, T xp, T ym, T yp, T zm, T zp, const StC<T>& c) {
    if (p == T(0)) return p;
    const bool pos = p > T(0);
    T g2 = T(0);
    const T m[3] = {xm, ym, zm}, q[3] = {xp, yp, zp};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const T dm = (p - m[a]) * c.inv_dx;  // backward difference a
        const T dp = (q[a] - p) * c.inv_dx;  // forward difference b
        const T u = pos ? fmax(dm, T(0)) : fmin(dm, T(0));
        const T v = pos ? fmin(dp, T(0)) : fmax(dp, T(0));
        g2 += fmax(u * u, v * v);
    }
    const T s = rs_scale(p, c.dx2);
    return p - c.cdx * s * (sqrt(g2) - T(1));
}

// K5 -- reinitialisation sweep over packages [lo, hi)
template <class T>
__global__ void __launch_bounds__(256) k_reinit(const T* __restrict__ in, T* __restrict__ out,
                                                const uint32_t* __restrict__ nb, int64_t lo,
                                                int64_t hi, StC<T> c) {
    const int64_t pkg = lo + (((int64_t)blockIdx.x * 256 + threadIdx.x) >> 4);
    Cross<T> x;
    if (!load_cross(in, nb, pkg, pkg < hi, x)) return;
    T o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const T l = i > 0 ? x.c[i - 1] : x.xm;
        const T r = i < 3 ? x.c[i + 1] : x.xp;
        o[i] = godunov(x.c[i], l, r, x.ym[i], x.yp[i], x.zm[i], x.zp[i], c);
    }
    st_row(out + pkg * 64 + 4 * (threadIdx.x & 15), o);
}

// K6 -- gradient by Lst. 5 with the arithmetic-mean regulariser, divided by
// dx (R-13): (phi_{+1} - phi_{-1}) / (2 dx); optional unit normal.
// Layout [pkg][component][64].
template <class T>
__global__ void __launch_bounds__(256) k_gradient(const T* __restrict__ in, T* __restrict__ grad,
                                                  T* __restrict__ normal,
                                                  const uint32_t* __restrict__ nb, int64_t lo,
                                                  int64_t hi, StC<T> c) {
    const int64_t pkg = lo + (((int64_t)blockIdx.x * 256 + threadIdx.x) >> 4);
    Cross<T> x;
    if (!load_cross(in, nb, pkg, pkg < hi, x)) return;
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
    T* G = grad + pkg * 192 + 4 * r;
    if (grad) {
        st_row(G, gx);
        st_row(G + 64, gy);
        st_row(G + 128, gz);
    }
    if (normal) {
        T nx[4], ny[4], nz[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const T m = sqrt(gx[i] * gx[i] + gy[i] * gy[i] + gz[i] * gz[i]);
            const T inv = m > T(0) ? T(1) / m : T(0);
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

// Table 1 "stencil": 7-point Laplacian
template <class T>
__global__ void __launch_bounds__(256) k_laplace(const T* __restrict__ in, T* __restrict__ out,
                                                 const uint32_t* __restrict__ nb, int64_t lo,
                                                 int64_t hi, T inv_dx2) {
    const int64_t pkg = lo + (((int64_t)blockIdx.x * 256 + threadIdx.x) >> 4);
    Cross<T> x;
    if (!load_cross(in, nb, pkg, pkg < hi, x)) return;
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
// kernel.  Four packages per 256-thread block; each package stages its
// (4 + 2R)^3 neighbourhood of H(-phi) in shared memory (values fetched through
// the neighbour row with Lst. 2, shifts in [-R, 3 + R] within [-4, 7]), then
// every thread accumulates its point over the tap list (taps in shared
// memory, uniform across the block -> broadcast reads).

template <class T>
struct Tap {
    int32_t off;
    T w, gx, gy, gz;
};

__device__ __forceinline__ float heav(float u, float eps, float inv_eps) {
    if (u < -eps) return 0.f;
    if (u > eps) return 1.f;
    const float q = u * inv_eps;
    return 0.5f * (1.f + q + sinpif(q) * 0.318309886183790672f);
}
__device__ __forceinline__ double heav(double u, double eps, double inv_eps) {
    if (u < -eps) return 0.0;
    if (u > eps) return 1.0;
    const double q = u * inv_eps;
    return 0.5 * (1.0 + q + sinpi(q) * 0.318309886183790672);
}

template <class T>
__global__ void __launch_bounds__(256) k_kint(const T* __restrict__ in,
                                              const uint32_t* __restrict__ nb, int64_t lo,
                                              int64_t hi, const Tap<T>* __restrict__ taps,
                                              int32_t n_taps, int32_t R, T eps, T* __restrict__ K,
                                              T* __restrict__ G) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Tap<T>* s_tap = reinterpret_cast<Tap<T>*>(smem_raw);
    const int RS = 4 + 2 * R;
    const int vol = RS * RS * RS;
    T* s_h = reinterpret_cast<T*>(smem_raw + ((sizeof(Tap<T>) * n_taps + 15) & ~size_t(15)));
    for (int t = threadIdx.x; t < n_taps; t += blockDim.x) s_tap[t] = taps[t];

    const int lp = threadIdx.x >> 6;  // package slot in block
    const int tl = threadIdx.x & 63;  // data point in package
    const int64_t pkg = lo + (int64_t)blockIdx.x * 4 + lp;
    const bool valid = pkg < hi;
    T* H = s_h + lp * vol;
    const T inv_eps = T(1) / eps;
    if (valid) {
        const uint32_t* row = nb + pkg * 27;
        for (int q = tl; q < vol; q += 64) {
            const int lx = q % RS, ly = (q / RS) % RS, lz = q / (RS * RS);
            const int sx = lx - R, sy = ly - R, sz = lz - R;  // shifts in [-R, 3+R]
            const int ox = (sx + 4) >> 2, oy = (sy + 4) >> 2, oz = (sz + 4) >> 2;
            const int dx = sx + 4 - 4 * ox, dy = sy + 4 - 4 * oy, dz = sz + 4 - 4 * oz;
            const uint32_t pk = __ldg(row + ox + 3 * oy + 9 * oz);
            const T v = __ldg(in + (int64_t)pk * 64 + dx + 4 * dy + 16 * dz);
            H[q] = heav(-v, eps, inv_eps);
        }
    }
    __syncthreads();
    if (!valid) return;
    const int i = tl & 3, j = (tl >> 2) & 3, k = tl >> 4;
    const int ci = (i + R) + RS * ((j + R) + RS * (k + R));
    T acc = T(0), ax = T(0), ay = T(0), az = T(0);
    for (int t = 0; t < n_taps; ++t) {
        const Tap<T> tp = s_tap[t];
        const T h = H[ci + tp.off];
        acc += tp.w * h;
        ax += tp.gx * h;
        ay += tp.gy * h;
        az += tp.gz * h;
    }
    K[pkg * 64 + tl] = acc;
    T* g = G + pkg * 192 + tl;
    g[0] = ax;
    g[64] = ay;
    g[128] = az;
}

// singular packages (R-16): K = S / 0, G = 0; grad = normal = 0
template <class T>
__global__ void k_singular(T* K, T* G, T* grad, T* normal, T S) {
    const int t = threadIdx.x;  // 128 threads: two packages x 64
    if (K) K[t] = t < 64 ? S : T(0);
    for (int c = 0; c < 3; ++c) {
        const int idx = (t >> 6) * 192 + c * 64 + (t & 63);
        if (G) G[idx] = T(0);
        if (grad) grad[idx] = T(0);
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
    return c;
}

template <class T>
static void reinit_t(sg_grid* g, int32_t iters, double cfl, cudaStream_t s) {
    const int64_t lo = g->own_lo, hi = g->own_hi;
    const StC<T> c = stencil_consts<T>(g, cfl);
    for (int it = 0; it < iters; ++it) {
        if (hi > lo) {
            const unsigned blocks = (unsigned)ceil_div((hi - lo) * 16, 256);
            k_reinit<T><<<blocks, 256, 0, s>>>((const T*)g->phi[g->cur], (T*)g->phi[1 - g->cur],
                                               g->nb, lo, hi, c);
            SG_LAUNCHED();
        }
        g->cur = 1 - g->cur;
    }
}

void launch_reinit(sg_grid* g, int32_t iters, double cfl, cudaStream_t s) {
    if (g->dtype == SG_F64)
        reinit_t<double>(g, iters, cfl, s);
    else
        reinit_t<float>(g, iters, cfl, s);
}

// Wendland C2 weights (reading R-14), evaluated on the host in double:
// sigma = 21 / (16 pi h^3), q = r / h, W = sigma (1 - q/2)^4 (2q + 1),
// W' = -5 sigma q (1 - q/2)^3 / h; w[o] = W(|o| dx) dx^3,
// gw[o] = W'(|o| dx) (-o/|o|) dx^3 for |o| dx < 2h.
template <class T>
static std::vector<Tap<T>> make_taps(double h_ratio, double dx, int R, double* S) {
    const double pi = 3.14159265358979323846;
    const double h = h_ratio * dx;
    const double sigma = 21.0 / (16.0 * pi * h * h * h);
    const int RS = 4 + 2 * R;
    std::vector<Tap<T>> v;
    double sum = 0.0;
    for (int oz = -R; oz <= R; ++oz)
        for (int oy = -R; oy <= R; ++oy)
            for (int ox = -R; ox <= R; ++ox) {
                const double len = std::sqrt((double)(ox * ox + oy * oy + oz * oz));
                if (!(len * dx < 2.0 * h)) continue;
                const double q = len * dx / h;
                const double a = 1.0 - 0.5 * q;
                const double W = sigma * a * a * a * a * (2.0 * q + 1.0) * dx * dx * dx;
                const double dW = -5.0 * sigma * q * a * a * a / h * dx * dx * dx;
                Tap<T> t;
                t.off = ox + RS * (oy + RS * oz);
                t.w = (T)W;
                t.gx = (T)(len > 0 ? dW * (-ox / len) : 0.0);
                t.gy = (T)(len > 0 ? dW * (-oy / len) : 0.0);
                t.gz = (T)(len > 0 ? dW * (-oz / len) : 0.0);
                sum += W;
                v.push_back(t);
            }
    *S = sum;
    return v;
}

struct TapCache {
    double h_ratio = -1;
    void* dev = nullptr;
    int32_t n = 0;
    int32_t R = 0;
    double S = 0;
};

template <class T>
static void gradient_t(sg_grid* g, uint32_t fields, double h_ratio, cudaStream_t s) {
    const int64_t lo = g->own_lo, hi = g->own_hi;
    const T* phi = (const T*)g->phi[g->cur];
    const StC<T> c = stencil_consts<T>(g, 0.0);
    const size_t vec_bytes = (size_t)g->n_pkg * 192 * sizeof(T);
    if ((fields & SG_GRAD) && !g->grad) g->grad = g->alloc(vec_bytes, s);
    if ((fields & SG_NORMAL) && !g->normal) g->normal = g->alloc(vec_bytes, s);
    if (fields & (SG_GRAD | SG_NORMAL)) {
        T* gp = (fields & SG_GRAD) ? (T*)g->grad : nullptr;
        T* np = (fields & SG_NORMAL) ? (T*)g->normal : nullptr;
        if (hi > lo) {
            const unsigned blocks = (unsigned)ceil_div((hi - lo) * 16, 256);
            k_gradient<T><<<blocks, 256, 0, s>>>(phi, gp, np, g->nb, lo, hi, c);
            SG_LAUNCHED();
        }
        k_singular<T><<<1, 128, 0, s>>>(nullptr, nullptr, gp, np, T(0));
        SG_LAUNCHED();
        if (gp) g->has_grad = true;
        if (np) g->has_normal = true;
    }
    if (fields & SG_KINT) {
        // largest |o_k| of a tap: o_k < 2 h_ratio  ->  R = ceil(2 h_ratio) - 1
        const int R = (int)std::ceil(2.0 * h_ratio) - 1;
        double S = 0;
        std::vector<Tap<T>> taps = make_taps<T>(h_ratio, g->gc.dx, R, &S);
        if (!g->kint) g->kint = g->alloc((size_t)g->n_pkg * 64 * sizeof(T), s);
        if (!g->gkint) g->gkint = g->alloc(vec_bytes, s);
        Tap<T>* d_taps = (Tap<T>*)dalloc(sizeof(Tap<T>) * taps.size(), s);
        SG_CUDA(cudaMemcpyAsync(d_taps, taps.data(), sizeof(Tap<T>) * taps.size(),
                                cudaMemcpyHostToDevice, s));
        const int RS = 4 + 2 * R;
        const size_t smem = ((sizeof(Tap<T>) * taps.size() + 15) & ~size_t(15)) +
                            sizeof(T) * 4 * RS * RS * RS;
        auto kern = k_kint<T>;
        if (smem > 48 * 1024)
            SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
        if (hi > lo) {
            kern<<<(unsigned)ceil_div(hi - lo, 4), 256, smem, s>>>(
                phi, g->nb, lo, hi, d_taps, (int32_t)taps.size(), R, (T)g->gc.dx, (T*)g->kint,
                (T*)g->gkint);
            SG_LAUNCHED();
        }
        k_singular<T><<<1, 128, 0, s>>>((T*)g->kint, (T*)g->gkint, nullptr, nullptr, (T)S);
        SG_LAUNCHED();
        SG_CUDA(cudaFreeAsync(d_taps, s));
        g->has_kint = true;
        g->kernel_sum = S;
    }
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
    if (hi <= lo) return;
    if (op == 0) {
        const int64_t n4 = (hi - lo) * 16;
        k_add<T><<<(unsigned)ceil_div(n4, 256), 256, 0, s>>>((T*)g->phi[g->cur], n4, lo * 16,
                                                            (T)value);
    } else {
        const unsigned blocks = (unsigned)ceil_div((hi - lo) * 16, 256);
        k_laplace<T><<<blocks, 256, 0, s>>>((const T*)g->phi[g->cur], (T*)g->phi[1 - g->cur],
                                            g->nb, lo, hi, (T)(1.0 / (g->gc.dx * g->gc.dx)));
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
        SG_ARG(g != nullptr, "sg_reinit: null grid");
        SG_ARG(iters >= 0, "sg_reinit: iters must be >= 0");
        SG_ARG(cfl > 0.0 && cfl <= 0.5, "sg_reinit: cfl must be in (0, 0.5]");
        SG_CUDA(cudaGetLastError());
        launch_reinit(g, iters, cfl, (cudaStream_t)stream);
        g->has_grad = g->has_normal = g->has_kint = false;  // derived fields are stale
    });
}

extern "C" sg_status sg_gradient(sg_grid* g, uint32_t fields, double h_ratio, void* stream) {
    return guard([&] {
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
        SG_ARG(g != nullptr, "sg_table1: null grid");
        SG_ARG(op == 0 || op == 1, "sg_table1: op must be 0 (sequential) or 1 (stencil)");
        SG_CUDA(cudaGetLastError());
        launch_table1(g, op, value, (cudaStream_t)stream);
    });
}
