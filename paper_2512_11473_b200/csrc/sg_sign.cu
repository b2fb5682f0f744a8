// sg_sign.cu -- sign-consistency correction (NEXT-3).
//
// "only the sign of level set for those data points very close to
// the surface is directly used, those at other locations are obtained by a
// two-step diffusion process from the near interface to the entire domain.
// The first coarse step is on the mesh cells and the second refined one is
// on the data packages."  Rule and trust sets: reading R-22 (include/sg.h
// sg_sign_correct).
//
// Both steps are bit-parallel Jacobi sweeps over (known, negative) bitmasks:
//   coarse  one thread per 32-cell word of the tagging bitmasks [z][y][W]:
//           x neighbours by shifts with the carry bit of the adjacent word,
//           y / z neighbours are the words one row / plane away; only words
//           next to the previous sweep's changes are visited (u8 stamps);
//   refined one thread per package, a u64 per mask (bit i + 4 j + 16 k, the
//           data layout): in-package neighbours by shifts, the face bits of
//           the 6 face-neighbour packages through the neighbour table (Lst. 2
//           slots 12/14, 10/16, 4/22); singular packages 0/1 are all-known,
//           all-negative / all-positive.
// The vote count of 6 face neighbours is a bit-sliced 3-bit adder, the
// majority a bit-sliced comparison: 32 (64) sites per thread, no branches.
// Convergence: each sweep raises a device flag if it signed anything; a sweep
// whose predecessor raised none returns at once, so sweeps are launched in
// growing batches and the host reads the flags once per batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "sg_internal.cuh"

namespace sg {

// ------------------------------------------------------- bit-sliced vote ---

template <class W>
__device__ __forceinline__ void full_add(W a, W b, W c, W& s, W& cy) {
    const W t = a ^ b;
    s = t ^ c;
    cy = (a & b) | (c & t);
}

// per bit lane: number of set bits among v[0..5], as 3 bit planes
template <class W>
__device__ __forceinline__ void count6(const W (&v)[6], W& c0, W& c1, W& c2) {
    W s1, k1, s2, k2;
    full_add(v[0], v[1], v[2], s1, k1);
    full_add(v[3], v[4], v[5], s2, k2);
    c0 = s1 ^ s2;
    const W k0 = s1 & s2;
    full_add(k1, k2, k0, c1, c2);
}

// per bit lane: A > B for 3-bit bit-sliced numbers
template <class W>
__device__ __forceinline__ W greater3(W a0, W a1, W a2, W b0, W b1, W b2) {
    return (a2 & ~b2) | (~(a2 ^ b2) & ((a1 & ~b1) | (~(a1 ^ b1) & (a0 & ~b0))));
}

// majority of the signed neighbours: lanes that turn negative / positive
template <class W>
__device__ __forceinline__ void majority(const W (&kn)[6], const W (&ng)[6], W& to_neg,
                                         W& to_pos) {
    W vn[6], vp[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        vn[d] = kn[d] & ng[d];
        vp[d] = kn[d] & ~ng[d];
    }
    W n0, n1, n2, p0, p1, p2;
    count6(vn, n0, n1, n2);
    count6(vp, p0, p1, p2);
    to_neg = greater3(n0, n1, n2, p0, p1, p2);
    to_pos = greater3(p0, p1, p2, n0, n1, n2);
}

// convergence flag of a sweep: one store per block that signed something,
// skipped once another block's store is visible (a single hot L2 line
// otherwise serialises thousands of stores per sweep)
__device__ __forceinline__ void raise_flag(bool changed, int* cur) {
    if (__syncthreads_or(changed) && threadIdx.x == 0) {
        if (*(volatile int*)cur == 0) *cur = 1;
    }
}

// persistent grid: a few resident blocks per SM, grid-stride loops
static unsigned sweep_blocks(int64_t items) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(items, 256), 8LL * sm_count()));
}

// ------------------------------------------------------------- coarse ----

// cell state: .x known bits, .y negative bits of one 32-cell word
// known bits: core cells, plus (refined layer, eval != nullptr) every valid
// cell that was not evaluated on this layer -- it carries its parent's
// corrected sign (on refined layers the correction is limited to the
// cells near the surface)
__global__ void __launch_bounds__(256) k_cell_pack(uint32_t nwords, const uint32_t* __restrict__ core,
                                                   const uint32_t* __restrict__ neg,
                                                   uint2* __restrict__ st,
                                                   const uint32_t* __restrict__ eval = nullptr,
                                                   int32_t nx = 0, uint32_t W = 1) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nwords) return;
    uint32_t k = core[t];
    if (eval) {
        const int tail = nx - 32 * (int)(t % W);
        const uint32_t valid = tail >= 32 ? 0xffffffffu : ((1u << tail) - 1u);
        k |= valid & ~eval[t];
    }
    st[t] = make_uint2(k, neg[t]);
}

__global__ void __launch_bounds__(256) k_cell_unpack(uint32_t nwords, const uint2* __restrict__ st,
                                                     uint32_t* __restrict__ neg) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nwords) neg[t] = st[t].y;
}

// One coarse sweep, frontier-restricted at word granularity: a 32-cell word
// is visited only if its u8 stamp says that it or one of the words whose
// cells touch its cells changed in the previous sweep, i.e.
// (u8)(stamp - sweep) <= 1 (every word is stamped 0 initially; a stamp of the
// next sweep written by another thread during this one also passes, and a
// stale stamp that aliases mod 256 only causes a harmless extra visit: the
// update is a pure function of the input buffer).  A skipped word cannot
// change and its output-buffer value is still current, because a word that
// changed is re-visited (and re-written) in the next sweep.
__global__ void __launch_bounds__(256) k_cell_sweep(int32_t nx, uint32_t W, uint32_t ny, uint32_t nz,
                                                    uint32_t nwords, int32_t sweep,
                                                    const uint2* __restrict__ in,
                                                    uint2* __restrict__ out,
                                                    uint8_t* __restrict__ stamp,
                                                    const int* __restrict__ prev,
                                                    int* __restrict__ cur) {
    if (prev && *prev == 0) return;  // converged: nothing to do (block-uniform)
    const uint8_t s8 = (uint8_t)sweep, n8 = (uint8_t)(sweep + 1);
    const uint32_t pl = W * ny;
    bool changed = false;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nwords;
         t += gridDim.x * blockDim.x) {
        if ((uint8_t)(stamp[t] - s8) > 1u) continue;
        const uint32_t row = t / W, q = t - row * W;
        const uint32_t z = row / ny, y = row - z * ny;
        const uint2 c = in[t];
        const uint2 zero = make_uint2(0u, 0u);
        const uint2 l = q > 0 ? in[t - 1] : zero;
        const uint2 r = q + 1 < W ? in[t + 1] : zero;
        const uint2 ym = y > 0 ? in[t - W] : zero;
        const uint2 yp = y + 1 < ny ? in[t + W] : zero;
        const uint2 zm = z > 0 ? in[t - pl] : zero;
        const uint2 zp = z + 1 < nz ? in[t + pl] : zero;
        uint32_t kk[6], nn[6];
        kk[0] = (c.x << 1) | (l.x >> 31);  // neighbour x - 1
        nn[0] = (c.y << 1) | (l.y >> 31);
        kk[1] = (c.x >> 1) | (r.x << 31);  // neighbour x + 1
        nn[1] = (c.y >> 1) | (r.y << 31);
        kk[2] = ym.x;
        nn[2] = ym.y;
        kk[3] = yp.x;
        nn[3] = yp.y;
        kk[4] = zm.x;
        nn[4] = zm.y;
        kk[5] = zp.x;
        nn[5] = zp.y;
        uint32_t tn, tp;
        majority(kk, nn, tn, tp);
        const int tail = nx - 32 * (int)q;  // valid cells in this word
        const uint32_t valid = tail >= 32 ? 0xffffffffu : ((1u << tail) - 1u);
        const uint32_t upd = ~c.x & (tn | tp) & valid;
        out[t] = make_uint2(c.x | upd, (c.y & ~upd) | (upd & tn));
        if (upd) {
            changed = true;
            stamp[t] = n8;
            if ((upd & 1u) && q > 0) stamp[t - 1] = n8;
            if ((upd >> 31) && q + 1 < W) stamp[t + 1] = n8;
            if (y > 0) stamp[t - W] = n8;
            if (y + 1 < ny) stamp[t + W] = n8;
            if (z > 0) stamp[t - pl] = n8;
            if (z + 1 < nz) stamp[t + pl] = n8;
        }
    }
    raise_flag(changed, cur);
}

// inactive cells' table entries from the corrected cell signs
__global__ void __launch_bounds__(256) k_bg_fix(uint32_t nx, int32_t ny, int32_t W, uint32_t ncell,
                                                const uint32_t* __restrict__ neg,
                                                uint32_t* __restrict__ bg) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const uint32_t b = bg[c];
    if (b >= 2u) return;
    const uint32_t row = c / nx;  // y + ny z
    const uint32_t x = c - row * nx;
    const uint32_t nb = (neg[(size_t)row * W + (x >> 5)] >> (x & 31)) & 1u;
    const uint32_t v = nb ? 0u : 1u;
    if (v != b) bg[c] = v;
}

// singular neighbour-table entries that refer to in-domain cells
__global__ void __launch_bounds__(256) k_nb_fix(GridC gc, int32_t W, int64_t n_pkg,
                                                const uint32_t* __restrict__ meta_cell,
                                                const uint32_t* __restrict__ neg,
                                                uint32_t* __restrict__ nbt,
                                                uint32_t* __restrict__ face) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t id = 2 + t / 27;
    if (id >= n_pkg) return;
    const int slot = (int)(t % 27);
    const uint32_t v = nbt[id * 27 + slot];
    if (v >= 2u) return;
    const uint32_t L = meta_cell[id];
    const int nx = gc.n[0], ny = gc.n[1];
    const int cx = (int)(L % (uint32_t)nx) + slot % 3 - 1;
    const int cy = (int)((L / (uint32_t)nx) % (uint32_t)ny) + (slot / 3) % 3 - 1;
    const int cz = (int)(L / ((uint32_t)nx * (uint32_t)ny)) + slot / 9 - 1;
    if (cx < 0 || cy < 0 || cz < 0 || cx >= nx || cy >= ny || cz >= gc.n[2]) return;  // R-6 kept
    const int64_t row = (int64_t)cy + (int64_t)ny * cz;
    const uint32_t ng = (neg[row * W + (cx >> 5)] >> (cx & 31)) & 1u;
    const uint32_t w = ng ? 0u : 1u;
    if (w != v) {
        nbt[id * 27 + slot] = w;
        const int fr = slot == 12 ? 0 : slot == 14 ? 1 : slot == 10 ? 2 : slot == 16 ? 3
                     : slot == 4 ? 4 : slot == 22 ? 5 : -1;
        if (fr >= 0) face[id * 8 + fr] = w;  // keep the face table in step
    }
}

// ------------------------------------------------------------ refined ----

// trusted points |phi| < tau keep their sign; singular packages all signed
template <class T>
__global__ void __launch_bounds__(256) k_pt_init(const T* __restrict__ phi, int64_t n_pkg, T tau,
                                                 uint64_t* __restrict__ kA, uint64_t* __restrict__ nA,
                                                 uint64_t* __restrict__ kB, uint64_t* __restrict__ nB) {
    const int lane = threadIdx.x & 31;
    const int64_t id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (id >= n_pkg) return;  // warp-uniform
    if (id < 2) {
        if (lane == 0) {
            kA[id] = kB[id] = ~0ull;
            nA[id] = nB[id] = id == 0 ? ~0ull : 0ull;
        }
        return;
    }
    const T a = phi[id * 64 + lane], b = phi[id * 64 + 32 + lane];
    const uint32_t klo = __ballot_sync(0xffffffffu, fabs(a) < tau);
    const uint32_t khi = __ballot_sync(0xffffffffu, fabs(b) < tau);
    const uint32_t nlo = __ballot_sync(0xffffffffu, a < T(0));
    const uint32_t nhi = __ballot_sync(0xffffffffu, b < T(0));
    if (lane == 0) {
        kA[id] = (uint64_t)klo | ((uint64_t)khi << 32);
        nA[id] = (uint64_t)nlo | ((uint64_t)nhi << 32);
    }
}

constexpr uint64_t kX0 = 0x1111111111111111ull, kX3 = 0x8888888888888888ull;
constexpr uint64_t kY0 = 0x000F000F000F000Full, kY3 = 0xF000F000F000F000ull;

__device__ __forceinline__ void face_shift(uint64_t own, const uint64_t (&f)[6], uint64_t (&o)[6]) {
    o[0] = ((own << 1) & ~kX0) | ((f[0] >> 3) & kX0);    // x - 1
    o[1] = ((own >> 1) & ~kX3) | ((f[1] << 3) & kX3);    // x + 1
    o[2] = ((own << 4) & ~kY0) | ((f[2] >> 12) & kY0);   // y - 1
    o[3] = ((own >> 4) & ~kY3) | ((f[3] << 12) & kY3);   // y + 1
    o[4] = (own << 16) | (f[4] >> 48);                   // z - 1
    o[5] = (own >> 16) | (f[5] << 48);                   // z + 1
}

__global__ void __launch_bounds__(256) k_pt_sweep(int64_t n_pkg, const uint32_t* __restrict__ nbt,
                                                  const uint64_t* __restrict__ kin,
                                                  const uint64_t* __restrict__ nin,
                                                  uint64_t* __restrict__ kout,
                                                  uint64_t* __restrict__ nout,
                                                  const int* __restrict__ prev,
                                                  int* __restrict__ cur) {
    if (prev && *prev == 0) return;
    bool changed = false;
    for (int64_t id = 2 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n_pkg;
         id += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t* row = nbt + id * 27;
        const int slot[6] = {12, 14, 10, 16, 4, 22};
        uint64_t fk[6], fn[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) {
            const uint32_t j = __ldg(row + slot[d]);
            fk[d] = kin[j];
            fn[d] = nin[j];
        }
        const uint64_t k = kin[id], n = nin[id];
        uint64_t kk[6], nn[6];
        face_shift(k, fk, kk);
        face_shift(n, fn, nn);
        uint64_t tn, tp;
        majority(kk, nn, tn, tp);
        const uint64_t upd = ~k & (tn | tp);
        kout[id] = k | upd;
        nout[id] = (n & ~upd) | (upd & tn);
        changed |= upd != 0ull;
    }
    raise_flag(changed, cur);
}

template <class T>
__global__ void __launch_bounds__(256) k_pt_apply(T* __restrict__ phi, int64_t n_pkg,
                                                  const uint64_t* __restrict__ kn,
                                                  const uint64_t* __restrict__ ng) {
    const int lane = threadIdx.x & 31;
    const int64_t id = 2 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (id >= n_pkg) return;
    const uint64_t k = kn[id], n = ng[id];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        if ((k >> i) & 1ull) {
            T* p = phi + id * 64 + i;
            const T a = fabs(*p);
            *p = ((n >> i) & 1ull) ? -a : a;
        }
    }
}

// ---------------------------------------------------------- host loop ----

static int* pinned_flags() {
    static thread_local int* p = nullptr;
    if (!p) SG_CUDA(cudaHostAlloc((void**)&p, 256 * sizeof(int), cudaHostAllocDefault));
    return p;
}

// Runs sweeps launch(j, prev_flag, cur_flag) in batches until one signs
// nothing or `cap` sweeps ran; returns the number of sweeps that signed
// something.  Sweep j reads buffer j % 2 and writes (j + 1) % 2, so the final
// state is in buffer (returned count) % 2.
template <class F>
static int run_sweeps(F&& launch, int cap, int* dflags, cudaStream_t s) {
    int* h = pinned_flags();
    int done = 0, signed_sweeps = 0, batch = 8;
    for (;;) {
        int n = batch;
        if (cap > 0) n = std::min(n, cap - done);
        if (n <= 0) break;
        SG_CUDA(cudaMemsetAsync(dflags, 0, sizeof(int) * (n + 1), s));
        for (int i = 0; i < n; ++i) launch(done + i, i == 0 ? nullptr : dflags + i, dflags + i + 1);
        SG_CUDA(cudaMemcpyAsync(h, dflags + 1, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
        SG_CUDA(cudaStreamSynchronize(s));
        int c = 0;
        while (c < n && h[c]) ++c;
        signed_sweeps += c;
        done += n;
        if (c < n) break;
        batch = std::min(2 * batch, 255);
    }
    return signed_sweeps;
}

// coarse flood on tagging bitmasks for the mesh build (see sg_internal.cuh)
int cell_flood(int32_t nx, int32_t W, int32_t ny, int32_t nz, const uint32_t* known, uint32_t* neg,
               cudaStream_t s) {
    const int64_t nwords = (int64_t)W * ny * nz;
    SG_ARG(nwords < (1LL << 31), "cell flood: too many cells");
    const size_t cw = sizeof(uint2) * (size_t)nwords;
    char* tmp = (char*)dalloc(2 * cw + 256 * sizeof(int) + (size_t)nwords, s);
    uint2* cs[2] = {(uint2*)tmp, (uint2*)(tmp + cw)};
    int* dflags = (int*)(tmp + 2 * cw);
    uint8_t* stamp = (uint8_t*)(dflags + 256);
    SG_CUDA(cudaMemsetAsync(stamp, 0, (size_t)nwords, s));
    const unsigned cb = (unsigned)ceil_div(nwords, 256);
    k_cell_pack<<<cb, 256, 0, s>>>((uint32_t)nwords, known, neg, cs[0]);
    SG_LAUNCHED();
    const unsigned cbs = sweep_blocks(nwords);
    const int sw = run_sweeps(
        [&](int j, const int* prev, int* cur) {
            k_cell_sweep<<<cbs, 256, 0, s>>>(nx, (uint32_t)W, (uint32_t)ny, (uint32_t)nz,
                                            (uint32_t)nwords, j, cs[j & 1], cs[(j + 1) & 1],
                                            stamp, prev, cur);
            SG_LAUNCHED();
        },
        0, dflags, s);
    k_cell_unpack<<<cb, 256, 0, s>>>((uint32_t)nwords, cs[sw & 1], neg);
    SG_LAUNCHED();
    SG_CUDA(cudaFreeAsync(tmp, s));
    return sw;
}

}  // namespace sg

using namespace sg;

extern "C" sg_status sg_sign_correct(sg_grid* g, double tau, int32_t max_sweeps, int32_t* sweeps,
                                     void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_sign_correct");
        SG_ARG(g != nullptr, "sg_sign_correct: null grid");
        SG_ARG(tau > 0.0 && std::isfinite(tau), "sg_sign_correct: tau must be > 0");
        SG_ARG(g->gc.zs_lo == 0 && g->gc.zs_hi == g->gc.n[2] && g->id_base == 2,
               "sg_sign_correct: single-domain grids only");
        cudaStream_t s = (cudaStream_t)stream;
        const GridC& gc = g->gc;
        const int32_t W = g->tag_W, ny = gc.n[1], nzt = g->zt_hi - g->zt_lo;
        const int64_t nwords = (int64_t)W * ny * nzt;
        const int64_t n_pkg = g->n_pkg;
        SG_ARG(nwords < (1LL << 31), "sg_sign_correct: too many cells");
        const size_t cw = sizeof(uint2) * (size_t)nwords, pw = sizeof(uint64_t) * (size_t)n_pkg;
        char* tmp = (char*)dalloc(2 * cw + 4 * pw + 256 * sizeof(int) + (size_t)nwords, s);
        uint2* cs[2] = {(uint2*)tmp, (uint2*)(tmp + cw)};
        uint64_t* pk[2] = {(uint64_t*)(tmp + 2 * cw), (uint64_t*)(tmp + 2 * cw + pw)};
        uint64_t* pn[2] = {(uint64_t*)(tmp + 2 * cw + 2 * pw), (uint64_t*)(tmp + 2 * cw + 3 * pw)};
        int* dflags = (int*)(tmp + 2 * cw + 4 * pw);
        uint8_t* stamp = (uint8_t*)(dflags + 256);
        SG_CUDA(cudaMemsetAsync(stamp, 0, (size_t)nwords, s));

        // coarse: core cells signed by f(centre), the rest unsigned
        const unsigned cb = (unsigned)ceil_div(nwords, 256);
        k_cell_pack<<<cb, 256, 0, s>>>((uint32_t)nwords, g->cell_core, g->cell_neg, cs[0],
                                       g->cell_eval, gc.n[0], (uint32_t)W);
        SG_LAUNCHED();
        const unsigned cbs = sweep_blocks(nwords);
        const int c_sweeps = run_sweeps(
            [&](int j, const int* prev, int* cur) {
                k_cell_sweep<<<cbs, 256, 0, s>>>(gc.n[0], (uint32_t)W, (uint32_t)ny, (uint32_t)nzt,
                                                (uint32_t)nwords, j, cs[j & 1], cs[(j + 1) & 1],
                                                stamp, prev, cur);
                SG_LAUNCHED();
            },
            max_sweeps, dflags, s);
        k_cell_unpack<<<cb, 256, 0, s>>>((uint32_t)nwords, cs[c_sweeps & 1], g->cell_neg);
        SG_LAUNCHED();
        k_bg_fix<<<(unsigned)ceil_div(g->ncell_stored, 256), 256, 0, s>>>(
            (uint32_t)gc.n[0], ny, W, (uint32_t)g->ncell_stored, g->cell_neg, g->bg);
        SG_LAUNCHED();
        if (n_pkg > 2) {
            k_nb_fix<<<(unsigned)ceil_div((n_pkg - 2) * 27, 256), 256, 0, s>>>(
                gc, W, n_pkg, g->meta_cell, g->cell_neg, g->nb, g->face);
            SG_LAUNCHED();
            tplan_invalidate(g, s);  // the face table changed
        }

        // refined: trusted points |phi| < tau, singular packages signed
        const unsigned wb = (unsigned)ceil_div(n_pkg * 32, 256);
        if (g->dtype == SG_F64)
            k_pt_init<double><<<wb, 256, 0, s>>>((const double*)g->phi[g->cur], n_pkg, tau, pk[0],
                                                 pn[0], pk[1], pn[1]);
        else
            k_pt_init<float><<<wb, 256, 0, s>>>((const float*)g->phi[g->cur], n_pkg, (float)tau,
                                                pk[0], pn[0], pk[1], pn[1]);
        SG_LAUNCHED();
        int p_sweeps = 0;
        if (n_pkg > 2) {
            const unsigned pb = sweep_blocks(n_pkg - 2);
            p_sweeps = run_sweeps(
                [&](int j, const int* prev, int* cur) {
                    k_pt_sweep<<<pb, 256, 0, s>>>(n_pkg, g->nb, pk[j & 1], pn[j & 1],
                                                  pk[(j + 1) & 1], pn[(j + 1) & 1], prev, cur);
                    SG_LAUNCHED();
                },
                max_sweeps, dflags, s);
            const unsigned ab = (unsigned)ceil_div((n_pkg - 2) * 32, 256);
            if (g->dtype == SG_F64)
                k_pt_apply<double><<<ab, 256, 0, s>>>((double*)g->phi[g->cur], n_pkg,
                                                      pk[p_sweeps & 1], pn[p_sweeps & 1]);
            else
                k_pt_apply<float><<<ab, 256, 0, s>>>((float*)g->phi[g->cur], n_pkg,
                                                     pk[p_sweeps & 1], pn[p_sweeps & 1]);
            SG_LAUNCHED();
        }
        SG_CUDA(cudaFreeAsync(tmp, s));
        g->has_grad = g->has_normal = g->has_kint = false;
        if (sweeps) {
            sweeps[0] = c_sweeps;
            sweeps[1] = p_sweeps;
        }
    });
}
