// sg_probe.cu -- grid-particle coupling (K8, reading R-15).
//
// Per particle: containing background cell (fp64 division + floor) ->
// background table -> far constant (inactive cell) or trilinear
// interpolation of phi (and grad phi) over the 8 data points around the
// position (see the phase comments of k_probe).  The corners lie at package-relative shifts in [-1, 4] of the
// containing package and are resolved through its neighbour row with
// NeighbourIndexShift (Lst. 2): "position-based random memory
// access of a data package and may be its neighbors".
//
// Host buffers: positions are staged H2D, probed and copied back D2H in
// chunks on two internal streams (double-buffered), so transfers of one chunk
// overlap the kernel / transfers of the other.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "sg_internal.cuh"

namespace sg {

// (x - lower) / d with the oracle's rounding: for a power-of-two spacing the
// division is a multiplication by the exact reciprocal.
__device__ __forceinline__ double qdiv(const GridC& gc, double v, bool cell) {
    if (gc.dyadic) return v * (cell ? gc.inv_cell : gc.inv_dx);
    return v / (cell ? gc.cell : gc.dx);
}

// Phase 1 (one thread per particle): positions staged through shared memory
// (coalesced), containing cell, background lookup; far-field and OOB
// particles are finished here.  Band particles are appended to a block list
// with their package id, corner shifts and weights.
// Phase 2 (eight lanes per band particle, one per trilinear corner): each
// lane resolves its corner with Lst. 2 on the package's neighbour row, loads
// phi and the three gradient components, and the eight weighted values are
// summed with xor-shuffles.  Outputs leave through shared memory, coalesced.
template <class T>
__global__ void __launch_bounds__(256) k_probe(GridC gc, const uint32_t* __restrict__ bg,
                                               const uint32_t* __restrict__ nb,
                                               const T* __restrict__ phi,
                                               const T* __restrict__ grad, int64_t n,
                                               const T* __restrict__ pos, T* __restrict__ out_phi,
                                               T* __restrict__ out_grad,
                                               unsigned long long* __restrict__ oob) {
    __shared__ T s_pos[256 * 3];
    __shared__ T s_phi[256];
    __shared__ T s_g[256 * 3];
    __shared__ uint32_t s_pk[256];
    __shared__ uint16_t s_who[256];
    __shared__ uint32_t s_sh[256];  // packed shifts s_k + 1 in [0, 4], 3 bits each
    __shared__ T s_t[256 * 3];
    __shared__ int s_cnt;
    const int64_t base = (int64_t)blockIdx.x * 256;
    const int m = (int)min((int64_t)256, n - base);
    {
        // three independent coalesced loads per thread, then the stores
        const T* src = pos + 3 * base;
        const int t0 = threadIdx.x;
        const T a0 = t0 < 3 * m ? src[t0] : T(0);
        const T a1 = t0 + 256 < 3 * m ? src[t0 + 256] : T(0);
        const T a2 = t0 + 512 < 3 * m ? src[t0 + 512] : T(0);
        s_pos[t0] = a0;
        s_pos[t0 + 256] = a1;
        s_pos[t0 + 512] = a2;
    }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();

    const int t = threadIdx.x;
    bool bad = false, band = false;
    uint32_t b = 0, sh = 0;
    T tt[3];
    if (t < m) {
        const double x[3] = {(double)s_pos[3 * t], (double)s_pos[3 * t + 1],
                             (double)s_pos[3 * t + 2]};
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 3; ++k)  // NaN fails both comparisons -> OOB
            ok = ok && (x[k] >= gc.lower[k]) && (x[k] < gc.upper[k]);
        int c[3] = {0, 0, 0};
        if (ok) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                c[k] = min((int)floor(qdiv(gc, x[k] - gc.lower[k], true)), gc.n[k] - 1);
            ok = c[2] >= gc.z_lo && c[2] < gc.z_hi;  // owned planes of a slab
        }
        T rphi = (T)gc.far;
        if (!ok) {
            bad = true;
        } else {
            b = __ldg(bg + ((int64_t)(c[2] - gc.zs_lo) * gc.n[1] + c[1]) * gc.n[0] + c[0]);
            if (b < 2) {
                rphi = (T)(b == 0 ? -gc.far : gc.far);
            } else {
                band = true;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double u = qdiv(gc, x[k] - gc.lower[k], false) - 0.5;
                    const double a = floor(u);
                    tt[k] = (T)(u - a);
                    sh |= (uint32_t)((int)a - 4 * c[k] + 1) << (3 * k);  // s_k in [-1, 3]
                }
            }
        }
        if (!band) {
            s_phi[t] = rphi;
            s_g[3 * t] = s_g[3 * t + 1] = s_g[3 * t + 2] = T(0);
        }
    }
    const unsigned lane = threadIdx.x & 31;
    const unsigned bal = __ballot_sync(0xffffffffu, band);
    int wbase = 0;
    if (lane == 0 && bal) wbase = atomicAdd(&s_cnt, __popc(bal));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (band) {
        const int idx = wbase + __popc(bal & ((1u << lane) - 1u));
        s_pk[idx] = b;
        s_who[idx] = (uint16_t)t;
        s_sh[idx] = sh;
        s_t[3 * idx] = tt[0];
        s_t[3 * idx + 1] = tt[1];
        s_t[3 * idx + 2] = tt[2];
    }
    if (oob) {
        const unsigned mb = __ballot_sync(0xffffffffu, bad);
        if (lane == 0 && mb) atomicAdd(oob, (unsigned long long)__popc(mb));
    }
    __syncthreads();

    // phase 2: 8 lanes per band particle
    const int cnt = s_cnt;
    const int corner = threadIdx.x & 7;
    const int bx = corner & 1, by = (corner >> 1) & 1, bz = corner >> 2;
    for (int q0 = 0; q0 < cnt; q0 += 32) {
        const int q = q0 + (threadIdx.x >> 3);
        const bool act = q < cnt;
        T v = T(0), g0 = T(0), g1 = T(0), g2 = T(0);
        if (act) {
            const uint32_t shq = s_sh[q];
            const int sx = (int)(shq & 7) - 1 + bx, sy = (int)((shq >> 3) & 7) - 1 + by,
                      sz = (int)(shq >> 6) - 1 + bz;  // corner shifts in [-1, 4]
            const int ox = (sx + 4) >> 2, oy = (sy + 4) >> 2, oz = (sz + 4) >> 2;
            const int d = (sx + 4 - 4 * ox) + 4 * (sy + 4 - 4 * oy) + 16 * (sz + 4 - 4 * oz);
            const int64_t pk = __ldg(nb + (int64_t)s_pk[q] * 27 + ox + 3 * oy + 9 * oz);
            const T tx = s_t[3 * q], ty = s_t[3 * q + 1], tz = s_t[3 * q + 2];
            const T w = ((bx ? tx : T(1) - tx) * (by ? ty : T(1) - ty)) * (bz ? tz : T(1) - tz);
            v = w * __ldg(phi + pk * 64 + d);
            if (grad) {
                const T* G = grad + pk * 192 + d;
                g0 = w * __ldg(G);
                g1 = w * __ldg(G + 64);
                g2 = w * __ldg(G + 128);
            }
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            v += __shfl_xor_sync(0xffffffffu, v, o);
            if (grad) {
                g0 += __shfl_xor_sync(0xffffffffu, g0, o);
                g1 += __shfl_xor_sync(0xffffffffu, g1, o);
                g2 += __shfl_xor_sync(0xffffffffu, g2, o);
            }
        }
        if (act && corner == 0) {
            const int p = s_who[q];
            s_phi[p] = v;
            s_g[3 * p] = g0;
            s_g[3 * p + 1] = g1;
            s_g[3 * p + 2] = g2;
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m; q += 256) out_phi[base + q] = s_phi[q];
    if (out_grad)
        for (int q = threadIdx.x; q < 3 * m; q += 256) out_grad[3 * base + q] = s_g[q];
}

template <class T>
static void probe_dev(const sg_grid* g, int64_t n, const void* pos, void* out_phi,
                      void* out_grad, unsigned long long* oob, cudaStream_t s) {
    if (n <= 0) return;
    const T* grad = out_grad ? (const T*)g->grad : nullptr;
    k_probe<T><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(
        g->gc, g->bg, g->nb, (const T*)g->phi[g->cur], grad, n, (const T*)pos, (T*)out_phi,
        (T*)out_grad, oob);
    SG_LAUNCHED();
}

static bool is_device_ptr(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct Staging {
    cudaStream_t st[2] = {nullptr, nullptr};
    cudaEvent_t ev = nullptr;
};

static Staging& staging() {
    static Staging S;
    static std::once_flag once;
    std::call_once(once, [] {
        SG_CUDA(cudaStreamCreateWithFlags(&S.st[0], cudaStreamNonBlocking));
        SG_CUDA(cudaStreamCreateWithFlags(&S.st[1], cudaStreamNonBlocking));
        SG_CUDA(cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming));
    });
    return S;
}

void launch_probe(const sg_grid* g, int64_t n, const void* pos, void* phi, void* grad,
                  unsigned long long* oob, cudaStream_t s) {
    const bool dev = is_device_ptr(pos) && is_device_ptr(phi) && is_device_ptr(grad);
    auto run = [&](int64_t m, const void* p, void* o, void* og, cudaStream_t st) {
        if (g->dtype == SG_F64)
            probe_dev<double>(g, m, p, o, og, oob, st);
        else
            probe_dev<float>(g, m, p, o, og, oob, st);
    };
    if (dev) {
        run(n, pos, phi, grad, s);
        return;
    }
    // host buffers: pipelined chunks through device staging buffers
    SG_ARG(!is_device_ptr(pos) && !is_device_ptr(phi) && (grad == nullptr || !is_device_ptr(grad)),
           "sg_probe: pos/phi/grad must be all device or all host pointers");
    Staging& S = staging();
    const int64_t chunk = std::min<int64_t>(n, (int64_t)1 << 22);
    const size_t es = (size_t)g->esz;
    char* buf[2];
    const size_t per = chunk * es * (3 + 1 + (grad ? 3 : 0));
    SG_CUDA(cudaEventRecord(S.ev, s));
    for (int b = 0; b < 2; ++b) {
        SG_CUDA(cudaStreamWaitEvent(S.st[b], S.ev, 0));
        buf[b] = (char*)dalloc(per, S.st[b]);
    }
    const char* hp = (const char*)pos;
    char* ho = (char*)phi;
    char* hg = (char*)grad;
    int64_t k = 0;
    for (int64_t off = 0; off < n; off += chunk, ++k) {
        const int b = (int)(k & 1);
        const int64_t m = std::min(chunk, n - off);
        cudaStream_t st = S.st[b];
        char* dp = buf[b];
        char* dphi = dp + chunk * es * 3;
        char* dg = dphi + chunk * es;
        SG_CUDA(cudaMemcpyAsync(dp, hp + off * 3 * es, m * 3 * es, cudaMemcpyHostToDevice, st));
        run(m, dp, dphi, grad ? dg : nullptr, st);
        SG_CUDA(cudaMemcpyAsync(ho + off * es, dphi, m * es, cudaMemcpyDeviceToHost, st));
        if (grad)
            SG_CUDA(cudaMemcpyAsync(hg + off * 3 * es, dg, m * 3 * es, cudaMemcpyDeviceToHost, st));
    }
    for (int b = 0; b < 2; ++b) {
        SG_CUDA(cudaFreeAsync(buf[b], S.st[b]));
        SG_CUDA(cudaStreamSynchronize(S.st[b]));
    }
}

}  // namespace sg

using namespace sg;

extern "C" sg_status sg_probe(const sg_grid* g, int64_t n, const void* pos, void* phi, void* grad,
                              unsigned long long* oob_count, void* stream) {
    return guard([&] {
        SG_ARG(g != nullptr, "sg_probe: null grid");
        SG_ARG(n >= 0, "sg_probe: n must be >= 0");
        if (n == 0) return;
        SG_ARG(pos != nullptr && phi != nullptr, "sg_probe: null pos or phi");
        if (grad != nullptr && !g->has_grad)
            throw Error(SG_ERR_STATE, "sg_probe: grad requested before sg_gradient(SG_GRAD)");
        SG_CUDA(cudaGetLastError());
        launch_probe(g, n, pos, phi, grad, oob_count, (cudaStream_t)stream);
    });
}
