// sg_probe.cu -- grid-particle coupling (K8, reading R-15).
//
// One thread per particle: containing background cell (fp64 division +
// floor) -> background table -> far constant (inactive cell) or
// trilinear interpolation of phi (and grad phi) over the 8 data points around
// the position.  The corners lie at package-relative shifts in [-1, 4] of the
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

template <class T>
__global__ void __launch_bounds__(256) k_probe(GridC gc, const uint32_t* __restrict__ bg,
                                               const uint32_t* __restrict__ nb,
                                               const T* __restrict__ phi,
                                               const T* __restrict__ grad, int64_t n,
                                               const T* __restrict__ pos, T* __restrict__ out_phi,
                                               T* __restrict__ out_grad,
                                               unsigned long long* __restrict__ oob) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    if (i < n) {
        const double x[3] = {(double)pos[3 * i], (double)pos[3 * i + 1], (double)pos[3 * i + 2]};
        int c[3];
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            // NaN fails both comparisons -> out of bounds
            ok = ok && (x[k] >= gc.lower[k]) && (x[k] < gc.upper[k]);
        }
        if (ok) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                c[k] = min((int)floor((x[k] - gc.lower[k]) / gc.cell), gc.n[k] - 1);
            ok = c[2] >= gc.z_lo && c[2] < gc.z_hi;  // owned planes of a slab
        }
        T rphi = (T)gc.far, g0 = T(0), g1 = T(0), g2 = T(0);
        if (!ok) {
            bad = true;
        } else {
            const uint32_t b =
                __ldg(bg + ((int64_t)(c[2] - gc.zs_lo) * gc.n[1] + c[1]) * gc.n[0] + c[0]);
            if (b < 2) {
                rphi = (T)(b == 0 ? -gc.far : gc.far);
            } else {
                int s[3];
                T t[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const double u = (x[k] - gc.lower[k]) / gc.dx - 0.5;
                    const double a = floor(u);
                    t[k] = (T)(u - a);
                    s[k] = (int)a - 4 * c[k];  // in [-1, 3]
                }
                const uint32_t* row = nb + (int64_t)b * 27;
                rphi = T(0);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int bx = q & 1, by = (q >> 1) & 1, bz = q >> 2;
                    const int sx = s[0] + bx, sy = s[1] + by, sz = s[2] + bz;  // [-1, 4]
                    const int ox = (sx + 4) >> 2, oy = (sy + 4) >> 2, oz = (sz + 4) >> 2;
                    const int d = (sx + 4 - 4 * ox) + 4 * (sy + 4 - 4 * oy) + 16 * (sz + 4 - 4 * oz);
                    const int64_t pk = __ldg(row + ox + 3 * oy + 9 * oz);
                    const T w = ((bx ? t[0] : T(1) - t[0]) * (by ? t[1] : T(1) - t[1])) *
                                (bz ? t[2] : T(1) - t[2]);
                    rphi += w * __ldg(phi + pk * 64 + d);
                    if (grad) {
                        const T* G = grad + pk * 192 + d;
                        g0 += w * __ldg(G);
                        g1 += w * __ldg(G + 64);
                        g2 += w * __ldg(G + 128);
                    }
                }
            }
        }
        out_phi[i] = rphi;
        if (out_grad) {
            out_grad[3 * i] = g0;
            out_grad[3 * i + 1] = g1;
            out_grad[3 * i + 2] = g2;
        }
    }
    if (oob) {
        const unsigned m = __ballot_sync(0xffffffffu, bad);
        if ((threadIdx.x & 31) == 0 && m) atomicAdd(oob, (unsigned long long)__popc(m));
    }
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
