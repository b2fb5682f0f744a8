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
#include <cstdlib>
#include <mutex>

#include "sg_internal.cuh"

namespace sg {

__device__ __forceinline__ void ld_vec4(const float* p, float (&v)[4]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld_vec4(const double* p, double (&v)[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// Containing background cell of one coordinate and the domain test (R-15:
// fp64 division and floor).  Fast path (gc.idx32: fp32 positions, l_c a power
// of two, lower = 0, upper a float): x * 2^e is exact in fp32, so floor and the
// comparisons are bit-identical to the fp64 definition without fp64 work.
template <class T, bool I32 = false>
__device__ __forceinline__ bool cell_of(const GridC& gc, int k, T x, int& c);

// lower-corner data index a = floor(u), u = (x - lower)/dx - 1/2, and the
// fraction t = u - a (exact in fp32 on the fast path: u < 2^23)
template <class T, bool I32 = false>
__device__ __forceinline__ void corner_of(const GridC& gc, int k, T x, int& a, T& t);

// (x - lower) / d with the oracle's rounding: for a power-of-two spacing the
// division is a multiplication by the exact reciprocal.
__device__ __forceinline__ double qdiv(const GridC& gc, double v, bool cell) {
    if (gc.dyadic) return v * (cell ? gc.inv_cell : gc.inv_dx);
    return v / (cell ? gc.cell : gc.dx);
}

template <>
__device__ __forceinline__ bool cell_of<float, true>(const GridC& gc, int k, float x, int& c) {
    c = min(__float2int_rd(x * gc.inv_cellf), gc.n[k] - 1);
    return x >= 0.f && x < gc.upperf[k];  // NaN fails both
}
template <>
__device__ __forceinline__ bool cell_of<float, false>(const GridC& gc, int k, float x, int& c) {
    const double xd = (double)x;
    c = min((int)floor(qdiv(gc, xd - gc.lower[k], true)), gc.n[k] - 1);
    return xd >= gc.lower[k] && xd < gc.upper[k];
}
template <>
__device__ __forceinline__ bool cell_of<double, false>(const GridC& gc, int k, double x, int& c) {
    c = min((int)floor(qdiv(gc, x - gc.lower[k], true)), gc.n[k] - 1);
    return x >= gc.lower[k] && x < gc.upper[k];
}
// v = x / dx is exact (power-of-two scaling).  The definition's fraction
// t = (v - 1/2) - a is computed as v - (a + 1/2): a + 1/2 is exact, and the
// subtraction is exact for v >= 1/2 (the operands are within a factor 2, or
// v < 2 and ulp(v) <= 1/2), so t is the fp64 value rounded once -- also for
// v < 1/2 (a = -1, t = RN(v + 1/2)), where the fp32 u = v - 1/2 itself would
// be rounded (v < 1/4).  floor(u) is exact in every case.
template <>
__device__ __forceinline__ void corner_of<float, true>(const GridC& gc, int k, float x, int& a,
                                                       float& t) {
    const float v = x * gc.inv_dxf;
    const float fa = floorf(v - 0.5f);
    a = (int)fa;
    t = v - (fa + 0.5f);
}
template <>
__device__ __forceinline__ void corner_of<float, false>(const GridC& gc, int k, float x, int& a,
                                                        float& t) {
    const double u = qdiv(gc, (double)x - gc.lower[k], false) - 0.5;
    const double fa = floor(u);
    a = (int)fa;
    t = (float)(u - fa);
}
template <>
__device__ __forceinline__ void corner_of<double, false>(const GridC& gc, int k, double x, int& a,
                                                  double& t) {
    const double u = qdiv(gc, x - gc.lower[k], false) - 0.5;
    const double fa = floor(u);
    a = (int)fa;
    t = u - fa;
}

// Warp-centric, barrier-free: each warp owns a chunk of 128 consecutive
// particles (4 per lane, 4 independent lookup chains per lane in flight).
// Phase 1 (lane per particle): positions staged through the warp's shared
// region (coalesced loads, transposed), containing cell, background lookup;
// far-field and OOB particles are finished here; band particles are appended
// to the warp's list with package id, corner shifts and weights.
// Phase 2 (one lane per band particle of the compacted list): the lane
// resolves its 8 corners with Lst. 2 on the package's neighbour row and loads
// one (phi, grad) vector per corner from the interleaved gradient layout (or
// phi alone when no gradient is requested).  Results leave through the
// shared region, coalesced.
constexpr int kPW = 128;  // particles per warp chunk

template <class T>
struct __align__(16) ProbeSmem {
    static constexpr int kWB = sizeof(T) == 4 ? 8 : 4;  // warps per block
    __align__(16) T xs[kWB][3 * kPW];  // staged positions
    __align__(16) T io[kWB][4 * kPW];  // results: phi (128) + grad (384)
    uint32_t pk[kWB][kPW];  // band list: containing package
    uint8_t who[kWB][kPW];  // band list: particle slot in the chunk
};

// I32: the exact fp32 index fast path (gc.idx32); V: 16 B aligned caller
// buffers (vector staging of full fp32 chunks) -- both resolved at launch
// O32: (package, point, component) offsets of the gradient layout fit in 32
// bits (n_pkg * 256 < 2^32): 32-bit corner address arithmetic
template <class T, bool I32, bool V, bool Q = false, bool O32 = false>
__global__ void __launch_bounds__(32 * ProbeSmem<T>::kWB, 4)
k_probe(GridC gc, const uint32_t* __restrict__ bg,
                                               const uint32_t* __restrict__ nb,
                                               const T* __restrict__ phi,
                                               const T* __restrict__ pg, int64_t n,
                                               const T* __restrict__ pos, T* __restrict__ out_phi,
                                               T* __restrict__ out_grad,
                                               unsigned long long* __restrict__ oob,
                                               unsigned long long* __restrict__ queue) {
    __shared__ ProbeSmem<T> S;
    constexpr int kWB = ProbeSmem<T>::kWB;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nchunks = (n + kPW - 1) / kPW;
    // Chunk order.  Static (queue == NULL): warp (block b, w) takes chunks
    // 8 b + w, + stride, ... -- the 8 warps of a block work on 8 consecutive
    // chunks, sharing their packages in L1.  Queue (long particle streams
    // whose packages do not stay in L2): with a static stride the fast warps
    // (far-field chunks) run whole lattice planes ahead of the slow ones and
    // the packages sorted particles share are evicted before the next planes
    // come back to them; handing out groups of kGrab consecutive chunks from
    // a global counter keeps the chunks in flight a compact window (C5 probe
    // 17.5 -> 13.4 ms; on C2 it loses the cross-warp L1 sharing: 151 -> 181
    // us, so the launcher picks per call).  Lane 0 issues the atomic for the
    // next group one group ahead, hiding its latency.
    constexpr int kGrab = 4;
    const int64_t stride = (int64_t)gridDim.x * kWB;
    auto grab = [&]() {
        unsigned long long c = 0;
        if (Q && lane == 0) c = atomicAdd(queue, 1ull);
        return c;
    };
    auto bcast = [&](unsigned long long c) {
        return (int64_t)__shfl_sync(0xffffffffu, c, 0) * kGrab;
    };
    int64_t group = Q ? bcast(grab()) : 0;
    unsigned long long pend = grab();
    int in_group = 0;
    int64_t chunk = Q ? group : (int64_t)blockIdx.x * kWB + w;
    T* io = S.io[w];
    // far-field constants in the grid dtype (selects, no per-particle fp64)
    const T far_pos = (T)gc.far, far_neg = -far_pos;
    // stored background cells < 2^32 (sg_build): 32-bit cell index arithmetic
    const uint32_t n0 = (uint32_t)gc.n[0], plane = (uint32_t)gc.n[0] * (uint32_t)gc.n[1];
    // persistent warps: the positions of the next chunk are loaded while the
    // current chunk is processed (hides the DRAM latency of the stream)
    T v[12];
    // 16 B vector staging / write-back for fp32 full chunks when the caller's
    // buffers are 16 B aligned (chunk offsets are multiples of 512 B)
    bool vnext = false;
    auto load_chunk = [&](int64_t ch) {
        const int64_t b0 = ch * kPW;
        const int mm = (int)min((int64_t)kPW, n - b0);
        const T* src = pos + 3 * b0;
        vnext = sizeof(T) == 4 && V && mm == kPW;
        if constexpr (sizeof(T) == 4) {
            if (vnext) {
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const float4 a = __ldg(reinterpret_cast<const float4*>(src) + lane + 32 * u);
                    v[4 * u] = a.x; v[4 * u + 1] = a.y; v[4 * u + 2] = a.z; v[4 * u + 3] = a.w;
                }
                return;
            }
        }
#pragma unroll
        for (int u = 0; u < 12; ++u) {
            const int q = lane + 32 * u;
            v[u] = q < 3 * mm ? src[q] : T(0);
        }
    };
    if (chunk < nchunks) load_chunk(chunk);
    while (chunk < nchunks) {
    const int64_t base = chunk * kPW;
    const int m = (int)min((int64_t)kPW, n - base);
    T* xs = S.xs[w];
    const bool vcur = vnext;
    if constexpr (sizeof(T) == 4) {
        if (vcur) {
#pragma unroll
            for (int u = 0; u < 3; ++u)
                reinterpret_cast<float4*>(xs)[lane + 32 * u] =
                    make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
            // grad staging starts at zero (far-field / OOB particles keep it)
#pragma unroll
            for (int u = 0; u < 3; ++u)
                reinterpret_cast<float4*>(io + kPW)[lane + 32 * u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    if (!vcur) {
#pragma unroll
        for (int u = 0; u < 12; ++u) {
            xs[lane + 32 * u] = v[u];
            io[kPW + lane + 32 * u] = T(0);
        }
    }
    int64_t nxt;
    if constexpr (!Q) {
        nxt = chunk + stride;
    } else if (in_group + 1 < kGrab) {
        nxt = chunk + 1;
        ++in_group;
    } else {
        group = bcast(pend);
        pend = grab();
        nxt = group;
        in_group = 0;
    }
    if (nxt < nchunks) load_chunk(nxt);
    __syncwarp();
    T x[4][3];  // positions in the grid dtype; promoted to double where used
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k) x[j][k] = xs[3 * (lane + 32 * j) + k];

    // phase 1: four particles per lane (p = lane + 32 j)
    uint32_t b[4];
    bool ok[4];
    int c[4][3];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        ok[j] = lane + 32 * j < m;
        if constexpr (I32) {
            // exact fp32 path: with lower = 0 and x / l_c exact, x in
            // [0, upper) <=> floor(x / l_c) in [0, n) -- one unsigned compare
            // per axis (no clamp can apply); a NaN coordinate (converted to 0
            // by the floor) is caught by the sum, infinities fall out of range
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                c[j][k] = __float2int_rd(x[j][k] * gc.inv_cellf);
                ok[j] = ok[j] && (uint32_t)c[j][k] < (uint32_t)gc.n[k];
            }
            const float sum = (x[j][0] + x[j][1]) + x[j][2];
            ok[j] = ok[j] && sum == sum;
        } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) ok[j] = cell_of<T, I32>(gc, k, x[j][k], c[j][k]) && ok[j];
        }
        ok[j] = ok[j] && c[j][2] >= gc.z_lo && c[j][2] < gc.z_hi;  // owned planes of a slab
        b[j] = ok[j] ? __ldg(bg + ((uint32_t)(c[j][2] - gc.zs_lo) * plane + (uint32_t)c[j][1] * n0 +
                                   (uint32_t)c[j][0]))
                     : 1u;
    }
    int nband = 0;
    int nbad = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int p = lane + 32 * j;
        const bool inr = p < m;
        const bool band = ok[j] && b[j] >= 2;
        const unsigned bal = __ballot_sync(0xffffffffu, band);
        nbad += __popc(__ballot_sync(0xffffffffu, inr && !ok[j]));
        if (band) {
            const int idx = nband + __popc(bal & ((1u << lane) - 1u));
            S.pk[w][idx] = b[j];
            S.who[w][idx] = (uint8_t)p;
        } else if (inr) {
            io[p] = (!ok[j] || b[j] != 0) ? far_pos : far_neg;
        }
        nband += __popc(bal);
    }
    if (oob && lane == 0 && nbad) atomicAdd(oob, (unsigned long long)nbad);
    __syncwarp();

    // phase 2: one lane per band particle (compacted list), all 8 corners
    // resolved by the lane: 8 neighbour-row loads, then 8 vector loads of
    // (phi, grad) -- two dependent rounds with 8 loads each in flight
    for (int q0 = 0; q0 < nband; q0 += 32) {
        const int q = q0 + lane;
        if (q < nband) {
            const int p = S.who[w][q];
            const uint32_t* row = nb + (size_t)S.pk[w][q] * 27;
            // containing cell, lower corner data index a = floor(u),
            // u = (x - lower)/dx - 1/2, fractions t = u - a (R-15)
            int sv[3];
            T tv[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                int ck, a;
                if constexpr (I32) {
                    // in-domain band particle: the exact x / l_c has no clamp
                    // to apply (x < upper), as in cell_of<float, true>
                    ck = __float2int_rd(xs[3 * p + k] * gc.inv_cellf);
                } else {
                    cell_of<T, I32>(gc, k, xs[3 * p + k], ck);
                }
                corner_of<T, I32>(gc, k, xs[3 * p + k], a, tv[k]);
                sv[k] = a - 4 * ck;  // in [-1, 3]
            }
            const int s0x = sv[0], s0y = sv[1], s0z = sv[2];
            const uint32_t self = S.pk[w][q];
            uint32_t pk[8];
            int d[8];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const int sx = s0x + (cc & 1), sy = s0y + ((cc >> 1) & 1), sz = s0z + (cc >> 2);
                const Shift hx = nb_shift(sx), hy = nb_shift(sy), hz = nb_shift(sz);
                d[cc] = hx.data + 4 * hy.data + 16 * hz.data;
                // slot 13 (offset (1, 1, 1)) is the package itself (O5): a
                // corner inside the containing package needs no table load
                // (all eight for 27/64 of the band particles)
                const int slot = hx.off + 3 * hy.off + 9 * hz.off;
                pk[cc] = slot == 13 ? self : __ldg(row + slot);
            }
            const T tx = tv[0], ty = tv[1], tz = tv[2];
            T acc[4] = {T(0), T(0), T(0), T(0)};
            if (pg) {
                T v[8][4];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    if constexpr (O32)
                        ld_vec4(pg + (pk[cc] * 256u + 4u * (uint32_t)d[cc]), v[cc]);
                    else
                        ld_vec4(pg + ((size_t)pk[cc] * 64 + d[cc]) * 4, v[cc]);
                }
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const T wgt = (((cc & 1) ? tx : T(1) - tx) * ((cc & 2) ? ty : T(1) - ty)) *
                                  ((cc & 4) ? tz : T(1) - tz);
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[e] += wgt * v[cc][e];
                }
            } else {
                T v[8];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    if constexpr (O32)
                        v[cc] = __ldg(phi + (pk[cc] * 64u + (uint32_t)d[cc]));
                    else
                        v[cc] = __ldg(phi + (size_t)pk[cc] * 64 + d[cc]);
                }
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const T wgt = (((cc & 1) ? tx : T(1) - tx) * ((cc & 2) ? ty : T(1) - ty)) *
                                  ((cc & 4) ? tz : T(1) - tz);
                    acc[0] += wgt * v[cc];
                }
            }
            io[p] = acc[0];
            io[kPW + 3 * p] = acc[1];
            io[kPW + 3 * p + 1] = acc[2];
            io[kPW + 3 * p + 2] = acc[3];
        }
    }
    __syncwarp();
    // coalesced results
    bool done = false;
    if constexpr (sizeof(T) == 4) {
        if (vcur) {
            reinterpret_cast<float4*>(out_phi + base)[lane] = reinterpret_cast<const float4*>(io)[lane];
            if (out_grad) {
#pragma unroll
                for (int u = 0; u < 3; ++u)
                    reinterpret_cast<float4*>(out_grad + 3 * base)[lane + 32 * u] =
                        reinterpret_cast<const float4*>(io + kPW)[lane + 32 * u];
            }
            done = true;
        }
    }
    if (!done) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int p = lane + 32 * j;
            if (p < m) out_phi[base + p] = io[p];
        }
        if (out_grad) {
#pragma unroll
            for (int u = 0; u < 12; ++u) {
                const int q = lane + 32 * u;
                if (q < 3 * m) out_grad[3 * base + q] = io[kPW + q];
            }
        }
    }
    __syncwarp();  // io is restaged by the next chunk
    chunk = nxt;
    }
}

template <class T>
static void probe_dev(const sg_grid* g, int64_t n, const void* pos, void* out_phi,
                      void* out_grad, unsigned long long* oob, cudaStream_t s) {
    if (n <= 0) return;
    const T* grad = out_grad ? (const T*)g->grad : nullptr;
    constexpr int kWB = ProbeSmem<T>::kWB;
    const int rb = resident_blocks((const void*)k_probe<T, false, false>, 32 * kWB);
    const int64_t blocks = std::min<int64_t>(ceil_div(n, kPW * kWB), rb);
    const bool vec =
        ((uintptr_t)pos | (uintptr_t)out_phi | (uintptr_t)(out_grad ? out_grad : out_phi)) % 16 == 0;
    // in-order chunk queue for long streams (more than 256 chunks per
    // resident warp, e.g. C5's 899 M particles), static order otherwise
    // (SG_PROBE_QUEUE=0 / 1 forces the order; tests compare the two bitwise)
    static const int force_q = [] {
        const char* e = std::getenv("SG_PROBE_QUEUE");
        return e ? std::atoi(e) : -1;
    }();
    const bool q = force_q == 1 || (force_q != 0 && ceil_div(n, kPW) > 256 * blocks * kWB);
    auto kern = q ? k_probe<T, false, false, true> : k_probe<T, false, false>;
    if constexpr (sizeof(T) == 4) {
        const bool o32 = g->n_pkg * 256 < ((int64_t)1 << 32);
        if (g->gc.idx32 && vec && o32)
            kern = q ? k_probe<T, true, true, true, true> : k_probe<T, true, true, false, true>;
        else if (g->gc.idx32)
            kern = vec ? (q ? k_probe<T, true, true, true> : k_probe<T, true, true>)
                       : (q ? k_probe<T, true, false, true> : k_probe<T, true, false>);
        else if (vec)
            kern = q ? k_probe<T, false, true, true> : k_probe<T, false, true>;
    }
    unsigned long long* queue = nullptr;
    if (q) {
        queue = (unsigned long long*)dalloc(sizeof(unsigned long long), s);
        SG_CUDA(cudaMemsetAsync(queue, 0, sizeof(unsigned long long), s));
    }
    kern<<<(unsigned)blocks, 32 * kWB, 0, s>>>(g->gc, g->bg, g->nb, (const T*)g->phi[g->cur], grad,
                                               n, (const T*)pos, (T*)out_phi, (T*)out_grad, oob,
                                               queue);
    SG_LAUNCHED();
    if (queue) SG_CUDA(cudaFreeAsync(queue, s));
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

// host-buffer pipeline: an upload stream, a compute stream and a download
// stream over a ring of kRing device chunk buffers, so both copy engines
// stream continuously (a per-chunk upload only waits for its buffer's
// previous download)
constexpr int kRingMax = 8;
struct Staging {
    cudaStream_t up = nullptr, comp = nullptr, down = nullptr, down2 = nullptr;
    cudaEvent_t ev = nullptr;
    cudaEvent_t ev_up[kRingMax], ev_comp[kRingMax], ev_down[kRingMax], ev_down2[kRingMax];
};

// staging streams and event per host thread and device: concurrent host-
// buffer probes from two threads never share an event, and the streams
// belong to the device they stage for (a host-buffer probe returns after its
// staging streams drained, so one thread's calls never overlap)
static Staging& staging() {
    static thread_local std::vector<Staging> per_dev;
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    if ((int)per_dev.size() <= dev) per_dev.resize(dev + 1);
    Staging& S = per_dev[dev];
    if (!S.ev) {
        SG_CUDA(cudaStreamCreateWithFlags(&S.up, cudaStreamNonBlocking));
        SG_CUDA(cudaStreamCreateWithFlags(&S.comp, cudaStreamNonBlocking));
        SG_CUDA(cudaStreamCreateWithFlags(&S.down, cudaStreamNonBlocking));
        SG_CUDA(cudaStreamCreateWithFlags(&S.down2, cudaStreamNonBlocking));
        SG_CUDA(cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming));
        for (int b = 0; b < kRingMax; ++b) {
            SG_CUDA(cudaEventCreateWithFlags(&S.ev_up[b], cudaEventDisableTiming));
            SG_CUDA(cudaEventCreateWithFlags(&S.ev_comp[b], cudaEventDisableTiming));
            SG_CUDA(cudaEventCreateWithFlags(&S.ev_down[b], cudaEventDisableTiming));
            SG_CUDA(cudaEventCreateWithFlags(&S.ev_down2[b], cudaEventDisableTiming));
        }
    }
    return S;
}

// ------------------------------------------------- partitioned grids ----
// K9: particles binned to the rank that owns their
// background plane, exchanged, probed by the owner, results sent back and
// restored to the caller's order.  Binning is stable (within a destination
// the caller's order is kept), so the received batch of every owner is
// deterministic.

constexpr int kBinT = 4096;  // particles per binning tile (256 threads x 16)

struct BinC {
    GridC gc;
    int32_t nranks, self;
    int32_t cuts[SG_MAX_RANKS + 1];
};

// owner rank of a position: the containing background plane by the probe's
// own cell arithmetic (the fp64 definition, R-15); outside the domain or NaN
// -> this rank (the local probe returns (+far, 0) and counts it)
template <class T>
__device__ __forceinline__ int owner_of(const BinC& b, const T* x) {
    int c[3];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) ok = cell_of<T, false>(b.gc, k, x[k], c[k]) && ok;
    if (!ok) return b.self;
    int lo = 0, hi = b.nranks - 1;  // largest r with cuts[r] <= cz
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b.cuts[mid] <= c[2]) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <class T>
__global__ void __launch_bounds__(256) k_bin_count(BinC b, int64_t n, const T* __restrict__ pos,
                                                   int64_t* __restrict__ hist, int64_t ntiles) {
    __shared__ int h[SG_MAX_RANKS];
    for (int d = threadIdx.x; d < b.nranks; d += 256) h[d] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * kBinT;
    for (int q = 0; q < kBinT / 256; ++q) {
        const int64_t i = t0 + q * 256 + threadIdx.x;
        if (i < n) atomicAdd(&h[owner_of(b, pos + 3 * i)], 1);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < b.nranks; d += 256) hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

// exclusive scan of the destination-major tile counts (one block; a few
// hundred thousand entries at most), per-destination totals
__global__ void __launch_bounds__(1024) k_bin_scan(int64_t* __restrict__ v, int64_t m,
                                                   int32_t nranks, int64_t ntiles,
                                                   long long* __restrict__ totals) {
    __shared__ int64_t part[1024];
    const int64_t per = (m + 1023) / 1024;
    const int64_t a = min(m, (int64_t)threadIdx.x * per), e = min(m, a + per);
    int64_t sum = 0;
    for (int64_t i = a; i < e; ++i) sum += v[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int64_t add = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    int64_t run = part[threadIdx.x] - sum;
    for (int64_t i = a; i < e; ++i) {
        const int64_t c = v[i];
        v[i] = run;
        run += c;
    }
    __syncthreads();
    if (threadIdx.x < nranks) {
        const int d = threadIdx.x;
        const int64_t lo = v[(int64_t)d * ntiles];
        const int64_t hi = d + 1 < nranks ? v[(int64_t)(d + 1) * ntiles] : part[1023];
        totals[d] = ntiles ? hi - lo : 0;
    }
}

// stable scatter of the positions into destination order; perm[i] = slot
template <class T>
__global__ void __launch_bounds__(256) k_bin_scatter(BinC b, int64_t n, const T* __restrict__ pos,
                                                     const int64_t* __restrict__ off, int64_t ntiles,
                                                     T* __restrict__ sendpos,
                                                     uint32_t* __restrict__ perm) {
    __shared__ int64_t base[SG_MAX_RANKS];
    __shared__ int wcnt[8][SG_MAX_RANKS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = threadIdx.x; d < b.nranks; d += 256) base[d] = off[(int64_t)d * ntiles + blockIdx.x];
    const int64_t t0 = (int64_t)blockIdx.x * kBinT;
    for (int q = 0; q < kBinT / 256; ++q) {
        for (int k = threadIdx.x; k < 8 * SG_MAX_RANKS; k += 256) (&wcnt[0][0])[k] = 0;
        __syncthreads();
        const int64_t i = t0 + q * 256 + threadIdx.x;
        const bool valid = i < n;
        const int d = valid ? owner_of(b, pos + 3 * i) : -1;
        const unsigned same = __match_any_sync(0xffffffffu, d);
        const int rank_w = __popc(same & ((1u << lane) - 1u));
        if (valid && rank_w == 0) wcnt[warp][d] = __popc(same);
        __syncthreads();
        if (valid) {
            int64_t slot = base[d] + rank_w;
            for (int w = 0; w < warp; ++w) slot += wcnt[w][d];
            sendpos[3 * slot] = pos[3 * i];
            sendpos[3 * slot + 1] = pos[3 * i + 1];
            sendpos[3 * slot + 2] = pos[3 * i + 2];
            perm[i] = (uint32_t)slot;
        }
        __syncthreads();
        for (int dd = threadIdx.x; dd < b.nranks; dd += 256) {
            int64_t t = 0;
            for (int w = 0; w < 8; ++w) t += wcnt[w][dd];
            base[dd] += t;
        }
        __syncthreads();
    }
}

// results back to the caller's order
template <class T>
__global__ void k_unbin(int64_t n, const uint32_t* __restrict__ perm, const T* __restrict__ rphi,
                        const T* __restrict__ rgrad, T* __restrict__ phi, T* __restrict__ grad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t k = perm[i];
    phi[i] = rphi[k];
    if (grad) {
        grad[3 * i] = rgrad[3 * k];
        grad[3 * i + 1] = rgrad[3 * k + 1];
        grad[3 * i + 2] = rgrad[3 * k + 2];
    }
}

template <class T>
static void probe_partitioned_dev(const sg_grid* g, int64_t n, const T* pos, T* out_phi, T* out_grad,
                                  unsigned long long* oob, cudaStream_t s) {
    const int P = g->nranks, me = g->rank;
    SG_ARG(n < (1LL << 32), "sg_probe: at most 2^32 - 1 particles per rank on a partitioned grid");
    BinC b{};
    b.gc = g->gc;
    b.nranks = P;
    b.self = me;
    for (int r = 0; r <= P; ++r) b.cuts[r] = g->cuts[r];
    const int64_t ntiles = ceil_div(n, kBinT);
    const size_t es = sizeof(T);
    const bool want_grad = out_grad != nullptr;
    // scratch: hist/offsets | totals | send positions | perm | results
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    const size_t sz_h = al(sizeof(int64_t) * std::max<int64_t>(1, P * ntiles)),
                 sz_t = al(sizeof(long long) * (P + 1) * (P + 1)),
                 sz_p = al(es * 3 * std::max<int64_t>(n, 1)),
                 sz_m = al(sizeof(uint32_t) * std::max<int64_t>(n, 1)),
                 sz_r = al(es * 4 * std::max<int64_t>(n, 1));
    char* buf = (char*)dalloc(sz_h + sz_t + sz_p + sz_m + sz_r, s);
    int64_t* hist = (int64_t*)buf;
    // [0, P]: my totals per destination + my grad request; then [P][P + 1]
    long long* tot = (long long*)(buf + sz_h);
    T* sendpos = (T*)(buf + sz_h + sz_t);
    uint32_t* perm = (uint32_t*)(buf + sz_h + sz_t + sz_p);
    T* res = (T*)(buf + sz_h + sz_t + sz_p + sz_m);  // phi [n] | grad [3n]
    SG_CUDA(cudaMemsetAsync(tot, 0, sizeof(long long) * P, s));
    const long long flag = want_grad ? 1 : 0;
    SG_CUDA(cudaMemcpyAsync(tot + P, &flag, sizeof(flag), cudaMemcpyHostToDevice, s));
    if (ntiles) {
        k_bin_count<T><<<(unsigned)ntiles, 256, 0, s>>>(b, n, pos, hist, ntiles);
        SG_LAUNCHED();
        k_bin_scan<<<1, 1024, 0, s>>>(hist, P * ntiles, P, ntiles, tot);
        SG_LAUNCHED();
        k_bin_scatter<T><<<(unsigned)ntiles, 256, 0, s>>>(b, n, pos, hist, ntiles, sendpos, perm);
        SG_LAUNCHED();
    }
    // count matrix cnt[src][dst] and every rank's grad request (the one host
    // synchronisation): the owners probe grad for everybody if anybody asks,
    // so every rank takes the same exchange decisions
    comm_allgather(g->comm, tot, tot + P + 1, sizeof(long long) * (P + 1), s);
    std::vector<long long> all((size_t)P * (P + 1)), cnt((size_t)P * P);
    SG_CUDA(cudaMemcpyAsync(all.data(), tot + P + 1, sizeof(long long) * all.size(),
                            cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    bool any_grad = false;
    for (int r = 0; r < P; ++r) {
        for (int d = 0; d < P; ++d) cnt[(size_t)r * P + d] = all[(size_t)r * (P + 1) + d];
        any_grad = any_grad || all[(size_t)r * (P + 1) + P] != 0;
    }
    if (any_grad && !g->has_grad)  // raised on every rank alike (has_grad is collective)
        throw Error(SG_ERR_STATE, "sg_probe: grad requested before sg_gradient(SG_GRAD)");
    const bool want_grad_any = any_grad;
    std::vector<int64_t> soff(P + 1, 0), roff(P + 1, 0);
    for (int d = 0; d < P; ++d) soff[d + 1] = soff[d] + cnt[(size_t)me * P + d];
    for (int r = 0; r < P; ++r) roff[r + 1] = roff[r] + (r == me ? 0 : cnt[(size_t)r * P + me]);
    const int64_t R = roff[P];
    T* rphi = res;
    T* rgrad = res + n;
    // received batch: positions | phi | grad
    T* recv = R ? (T*)dalloc(es * 7 * R, s) : nullptr;
    T* recv_phi = recv + 3 * R;
    T* recv_grad = recv + 4 * R;
    std::vector<P2P> ops;
    for (int d = 0; d < P; ++d) {
        const int64_t c = cnt[(size_t)me * P + d];
        if (d != me && c) ops.push_back(P2P{d, true, sendpos + 3 * soff[d], (size_t)c * 3 * es});
    }
    for (int r = 0; r < P; ++r) {
        const int64_t c = r == me ? 0 : cnt[(size_t)r * P + me];
        if (c) ops.push_back(P2P{r, false, recv + 3 * roff[r], (size_t)c * 3 * es});
    }
    comm_group(g->comm, ops.data(), (int)ops.size(), s);
    // the owner's probes: this rank's own bucket in place, the received batch
    const int64_t mine = cnt[(size_t)me * P + me];
    if (mine)
        probe_dev<T>(g, mine, sendpos + 3 * soff[me], rphi + soff[me],
                     want_grad_any ? rgrad + 3 * soff[me] : nullptr, oob, s);
    if (R) probe_dev<T>(g, R, recv, recv_phi, want_grad_any ? recv_grad : nullptr, oob, s);
    ops.clear();
    for (int r = 0; r < P; ++r) {
        const int64_t c = r == me ? 0 : cnt[(size_t)r * P + me];
        if (!c) continue;
        ops.push_back(P2P{r, true, recv_phi + roff[r], (size_t)c * es});
        if (want_grad_any) ops.push_back(P2P{r, true, recv_grad + 3 * roff[r], (size_t)c * 3 * es});
    }
    for (int d = 0; d < P; ++d) {
        const int64_t c = cnt[(size_t)me * P + d];
        if (d == me || !c) continue;
        ops.push_back(P2P{d, false, rphi + soff[d], (size_t)c * es});
        if (want_grad_any) ops.push_back(P2P{d, false, rgrad + 3 * soff[d], (size_t)c * 3 * es});
    }
    comm_group(g->comm, ops.data(), (int)ops.size(), s);
    if (n) {
        k_unbin<T><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(n, perm, rphi, rgrad, out_phi,
                                                             want_grad ? out_grad : nullptr);
        SG_LAUNCHED();
    }
    if (recv) SG_CUDA(cudaFreeAsync(recv, s));
    SG_CUDA(cudaFreeAsync(buf, s));
}

static void probe_partitioned(const sg_grid* g, int64_t n, const void* pos, void* phi, void* grad,
                              unsigned long long* oob, cudaStream_t s) {
    const bool dev = is_device_ptr(pos) && is_device_ptr(phi) && is_device_ptr(grad);
    const size_t es = (size_t)g->esz;
    const void* dpos = pos;
    void* dphi = phi;
    void* dgrad = grad;
    char* stage = nullptr;
    if (!dev) {  // host buffers: whole-array staging
        SG_ARG(n == 0 || (!is_device_ptr(pos) && !is_device_ptr(phi) &&
                          (grad == nullptr || !is_device_ptr(grad))),
               "sg_probe: pos/phi/grad must be all device or all host pointers");
        stage = (char*)dalloc(std::max<size_t>(1, n * es * 7), s);
        dpos = stage;
        dphi = stage + n * es * 3;
        dgrad = grad ? stage + n * es * 4 : nullptr;
        if (n) SG_CUDA(cudaMemcpyAsync(stage, pos, n * es * 3, cudaMemcpyHostToDevice, s));
    }
    if (g->dtype == SG_F64)
        probe_partitioned_dev<double>(g, n, (const double*)dpos, (double*)dphi, (double*)dgrad, oob, s);
    else
        probe_partitioned_dev<float>(g, n, (const float*)dpos, (float*)dphi, (float*)dgrad, oob, s);
    if (!dev) {
        if (n) {
            SG_CUDA(cudaMemcpyAsync(phi, dphi, n * es, cudaMemcpyDeviceToHost, s));
            if (grad) SG_CUDA(cudaMemcpyAsync(grad, dgrad, n * es * 3, cudaMemcpyDeviceToHost, s));
        }
        SG_CUDA(cudaFreeAsync(stage, s));
        SG_CUDA(cudaStreamSynchronize(s));
    }
}

void launch_probe(const sg_grid* g, int64_t n, const void* pos, void* phi, void* grad,
                  unsigned long long* oob, cudaStream_t s) {
    if (g->partitioned()) {
        probe_partitioned(g, n, pos, phi, grad, oob, s);
        return;
    }
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
    // ~10 chunks of 0.25-2 M particles.  Measured on C4 (19.45 M particles,
    // 233 MB up + 311 MB down; profiles/r02/e2e_staging.jsonl): 0.6 M-particle
    // chunks 7.58 ms, 1 M 6.86 ms, 2 M 6.84 ms, 4 M (ring 3) 7.10 ms -- the
    // copy engines reach their concurrent rate with chunks of >= 1 M, while
    // the first upload before any kernel (fill) overlaps the caller's build /
    // reinit / gradient still running on its stream.  Chunks are multiples of
    // 4096 particles: host offsets that are only 16 B aligned (n / 10 =
    // 1,945,444 particles) cost 7.28 ms against 6.65-6.70 ms for 1.90 M /
    // 1.97 M / 2 M-particle chunks (profiles/r02/e2e_staging.jsonl).
    // (SG_PROBE_CHUNK / SG_PROBE_RING / SG_PROBE_DOWN1: experiment overrides)
    static const int64_t env_chunk = [] {
        const char* e = std::getenv("SG_PROBE_CHUNK");
        return e ? std::atoll(e) : 0LL;
    }();
    static const int env_ring = [] {
        const char* e = std::getenv("SG_PROBE_RING");
        return e ? std::max(2, std::min(kRingMax, std::atoi(e))) : 4;
    }();
    static const bool down1 = [] {
        const char* e = std::getenv("SG_PROBE_DOWN1");
        return e && e[0] == '1';
    }();
    const int kRing = env_ring;
    const int64_t chunk = env_chunk > 0 ? std::min<int64_t>(n, env_chunk) : std::min<int64_t>(
        n, std::max<int64_t>((int64_t)1 << 18,
                             std::min<int64_t>(ceil_div(ceil_div(n, 10), 4096) * 4096, (int64_t)1 << 21)));
    const size_t es = (size_t)g->esz;
    const size_t per = chunk * es * (3 + 1 + (grad ? 3 : 0));
    // the uploads of the positions do not depend on the grid: only the probe
    // kernels wait for the caller's stream (the build / reinit / gradient
    // still running there), so the first chunks' H2D overlap that work
    SG_CUDA(cudaEventRecord(S.ev, s));
    SG_CUDA(cudaStreamWaitEvent(S.comp, S.ev, 0));
    char* ring = (char*)dalloc(per * kRing, S.up);
    SG_CUDA(cudaEventRecord(S.ev_up[0], S.up));  // the ring exists on up
    SG_CUDA(cudaStreamWaitEvent(S.comp, S.ev_up[0], 0));
    SG_CUDA(cudaStreamWaitEvent(S.down, S.ev_up[0], 0));
    SG_CUDA(cudaStreamWaitEvent(S.down2, S.ev_up[0], 0));
    const char* hp = (const char*)pos;
    char* ho = (char*)phi;
    char* hg = (char*)grad;
    int64_t k = 0;
    for (int64_t off = 0; off < n; off += chunk, ++k) {
        const int b = (int)(k % kRing);
        const int64_t m = std::min(chunk, n - off);
        char* dp = ring + per * b;
        char* dphi = dp + chunk * es * 3;
        char* dg = dphi + chunk * es;
        // buffer b is free once the download of chunk k - kRing is done
        if (k >= kRing) {
            SG_CUDA(cudaStreamWaitEvent(S.up, S.ev_down[b], 0));
            SG_CUDA(cudaStreamWaitEvent(S.up, S.ev_down2[b], 0));
        }
        SG_CUDA(cudaMemcpyAsync(dp, hp + off * 3 * es, m * 3 * es, cudaMemcpyHostToDevice, S.up));
        SG_CUDA(cudaEventRecord(S.ev_up[b], S.up));
        SG_CUDA(cudaStreamWaitEvent(S.comp, S.ev_up[b], 0));
        run(m, dp, dphi, grad ? dg : nullptr, S.comp);
        SG_CUDA(cudaEventRecord(S.ev_comp[b], S.comp));
        // phi and grad come back on two download streams (two copy engines)
        SG_CUDA(cudaStreamWaitEvent(S.down, S.ev_comp[b], 0));
        SG_CUDA(cudaMemcpyAsync(ho + off * es, dphi, m * es, cudaMemcpyDeviceToHost, S.down));
        SG_CUDA(cudaEventRecord(S.ev_down[b], S.down));
        cudaStream_t d2 = down1 ? S.down : S.down2;
        SG_CUDA(cudaStreamWaitEvent(d2, S.ev_comp[b], 0));
        if (grad)
            SG_CUDA(cudaMemcpyAsync(hg + off * 3 * es, dg, m * 3 * es, cudaMemcpyDeviceToHost, d2));
        SG_CUDA(cudaEventRecord(S.ev_down2[b], d2));
    }
    SG_CUDA(cudaEventRecord(S.ev, S.down2));
    SG_CUDA(cudaStreamWaitEvent(S.down, S.ev, 0));
    SG_CUDA(cudaFreeAsync(ring, S.down));
    SG_CUDA(cudaStreamSynchronize(S.down));
}

}  // namespace sg

using namespace sg;

extern "C" sg_status sg_probe(const sg_grid* g, int64_t n, const void* pos, void* phi, void* grad,
                              unsigned long long* oob_count, void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_probe");
        SG_ARG(g != nullptr, "sg_probe: null grid");
        SG_ARG(n >= 0, "sg_probe: n must be >= 0");
        if (n == 0 && !g->partitioned()) return;  // (collective on a partition)
        SG_ARG(n == 0 || (pos != nullptr && phi != nullptr), "sg_probe: null pos or phi");
        if (grad != nullptr && !g->has_grad && !g->partitioned())
            throw Error(SG_ERR_STATE, "sg_probe: grad requested before sg_gradient(SG_GRAD)");
        SG_CUDA(cudaGetLastError());
        launch_probe(g, n, pos, phi, grad, oob_count, (cudaStream_t)stream);
    });
}
