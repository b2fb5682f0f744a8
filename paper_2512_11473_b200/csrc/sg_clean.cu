// sg_clean.cu -- small-feature cleaning (NEXT-3).
//
// "Very often the geometry which is originally generated for
// manufacturing includes many small features which are not necessary for
// computational fluid or solid dynamics (CFD or CSD) simulations and may lead
// to numerical instabilities if not cleaned.  In the present work, we
// reimplemented the level-set cleaning algorithms (only on the finest layer)
// in Ref. [yu2023level] so that it can be run on GPU."  The criterion of
// yu2023level is not restated in the paper; reading R-23 takes the stand-in
// of SPEC S:476-484 (include/sg.h sg_clean).
//
// One round = the kernel integral K (the SG_KINT path of sg_gradient), one
// marking pass (k_clean: raise every active point with -dx < phi < 0 and
// K < threshold S to +dx, block-reduced count), one host read of the count,
// and `reinit_iters` reinitialisation sweeps (sg_reinit's cached graph).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "sg_internal.cuh"

namespace sg {

template <class T>
__global__ void __launch_bounds__(256) k_clean(T* __restrict__ phi, const T* __restrict__ K,
                                               int64_t n_pkg, T dx, T kthr,
                                               unsigned long long* __restrict__ count) {
    const int64_t i = 128 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // skip 0 / 1
    bool raised = false;
    if (i < n_pkg * 64) {
        const T v = phi[i];
        if (v < T(0) && fabs(v) < dx && K[i] < kthr) {
            phi[i] = dx;
            raised = true;
        }
    }
    const int c = __syncthreads_count(raised);
    if (threadIdx.x == 0 && c) atomicAdd(count, (unsigned long long)c);
}

static unsigned long long* pinned_count() {
    static thread_local unsigned long long* p = nullptr;
    if (!p) SG_CUDA(cudaHostAlloc((void**)&p, sizeof(unsigned long long), cudaHostAllocDefault));
    return p;
}

static void check_call(sg_status st) {
    if (st != SG_OK) throw Error(st, sg_last_error());
}

}  // namespace sg

using namespace sg;

extern "C" sg_status sg_clean(sg_grid* g, double h_ratio, double threshold, int32_t reinit_iters,
                              double cfl, int32_t max_rounds, int32_t* rounds, int64_t* modified,
                              void* stream) {
    int32_t done = 0;
    std::vector<int64_t> mods;
    sg_status st = guard([&] {
        SG_ARG(g != nullptr, "sg_clean: null grid");
        SG_ARG(h_ratio >= 0.5 && h_ratio <= 2.0, "sg_clean: h_ratio must be in [0.5, 2]");
        SG_ARG(threshold >= 0.0 && threshold <= 1.0 && std::isfinite(threshold),
               "sg_clean: threshold must be in [0, 1]");
        SG_ARG(reinit_iters >= 0 && max_rounds >= 0, "sg_clean: negative count");
        SG_ARG(cfl > 0.0 && cfl <= 0.5, "sg_clean: cfl must be in (0, 0.5]");
        SG_ARG(g->gc.zs_lo == 0 && g->gc.zs_hi == g->gc.n[2] && g->id_base == 2,
               "sg_clean: single-domain grids only");
        mods.assign((size_t)max_rounds, 0);
    });
    if (st != SG_OK) return st;
    st = guard([&] {
        cudaStream_t s = (cudaStream_t)stream;
        unsigned long long* d_count = (unsigned long long*)dalloc(sizeof(unsigned long long), s);
        unsigned long long* h = pinned_count();
        const int64_t npts = (g->n_pkg - 2) * 64;
        for (int r = 0; r < max_rounds && npts > 0; ++r) {
            check_call(sg_gradient(g, SG_KINT, h_ratio, stream));
            SG_CUDA(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
            const unsigned nb = (unsigned)ceil_div(npts, 256);
            if (g->dtype == SG_F64)
                k_clean<double><<<nb, 256, 0, s>>>((double*)g->phi[g->cur], (const double*)g->kint,
                                                   g->n_pkg, g->gc.dx, threshold * g->kernel_sum,
                                                   d_count);
            else
                k_clean<float><<<nb, 256, 0, s>>>((float*)g->phi[g->cur], (const float*)g->kint,
                                                  g->n_pkg, (float)g->gc.dx,
                                                  (float)(threshold * g->kernel_sum), d_count);
            SG_LAUNCHED();
            SG_CUDA(cudaMemcpyAsync(h, d_count, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
            SG_CUDA(cudaStreamSynchronize(s));
            mods[(size_t)r] = (int64_t)*h;
            if (*h == 0) break;
            ++done;
            g->has_grad = g->has_normal = false;
            if (reinit_iters > 0) check_call(sg_reinit(g, reinit_iters, cfl, stream));
            else g->has_kint = false;
        }
        SG_CUDA(cudaFreeAsync(d_count, s));
    });
    if (rounds) *rounds = done;
    if (modified)
        for (int32_t r = 0; r < max_rounds; ++r) modified[r] = mods.empty() ? 0 : mods[(size_t)r];
    return st;
}
