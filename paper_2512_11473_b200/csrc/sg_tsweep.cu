// sg_tsweep.cu -- reinitialisation two sweeps at a time (K5 with temporal
// blocking; SURVEY 7 hard part 2).
//
// The paper's reinitialisation (O7 / reading R-12) is a chain of
// Jacobi sweeps over the packages (Lst. 4 package_for): sweep k+1
// of a data point reads sweep k of its six neighbours.  One sweep per kernel
// moves phi through HBM twice per sweep (read + write, 8.5 B per point with the
// face row), and on C3/C5 that is the whole cost.  Here one kernel does two
// sweeps: a CTA stages a tile of packages plus the part of their neighbourhood
// the two sweeps depend on in shared memory, does sweep 1 there (the tile and
// the neighbourhood rows the tile's sweep 2 reads), then sweep 2 of the tile,
// and writes the tile once.  Per pair of sweeps the tile is read and written
// once; the neighbourhood rows are extra reads.
//
// Which data a point of the tile depends on: after two sweeps, the points
// within L1 distance 2.  For a package P of the tile and a neighbour package
// H = P + o (o in {-1, 0, 1}^3, |o|_1 = 1 or 2: the 6 face and 12 edge
// neighbours; corners are at distance >= 3) the distance of H's x-row (j, k)
// from P is  [o_x != 0] + d(o_y, j) + d(o_z, k)  with d(+1, j) = j + 1,
// d(-1, j) = 4 - j, d(0, .) = 0 (the row's nearest point).  Rows at distance
// <= 2 are loaded; rows at distance <= 1 are updated in sweep 1 (sweep 2 of the
// tile reads exactly the distance-1 points).  A halo row's other points (and
// anything whose neighbour was not loaded) get meaningless sweep-1 values that
// nothing reads.  The arithmetic of every point is godunov_row
// (sg_godunov.cuh), the same inline code as the single sweep, so the result is
// bit-identical to two k_sweep launches.
//
// Tiles: the active packages sorted by the Morton code of their background
// cell (cub radix sort), cut into chunks of kTI; a chunk whose slots (2
// singular + packages + halo) exceed kTCap or whose first-sweep halo rows
// exceed kTComp is halved until it fits.  The plan (per tile: slot -> global
// id, slot -> six face-neighbour slots, halo row masks, first-sweep halo row
// list) is built once per grid on the device (one hash set per CTA) and
// reused by every reinit call; sg_sign_correct's table fix invalidates it.
//
// Measured (one B200, profiles/README.md): C2 24.7-26.9 us per sweep vs 15.1
// us for the single sweep, C3 274-292 vs 158 us (row-per-lane cp.async
// staging and this version: TMA bulk staging + two rows per lane; 64-package
// tiles at 3 CTAs / SM measure the same).  The thick band's tiles carry a
// large neighbourhood (1.7 halo packages per tile package at 96 packages per
// tile: 0.9 extra rows staged and 0.57 extra rows updated in sweep 1 per
// tile row); ncu (C2): 20 M warp instructions per two-sweep launch, 57 % of
// them the Godunov arithmetic itself, issue active 45 % (stalls: fixed
// latency of the arithmetic chains, shared-memory loads and the four
// barriers per tile), 16 warps per SM.  Kept as an opt-in path (SG_TSWEEP=1)
// with its
// bitwise tests (tests/test_tsweep_gpu.py).
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdlib>

#include "sg_godunov.cuh"
#include "sg_internal.cuh"

namespace sg {

constexpr int kTI = 96;        // packages per level-0 chunk
constexpr int kTCap = 384;     // slots per tile (2 singular + packages + halo)
constexpr int kTComp = 1280;   // first-sweep halo rows per tile
constexpr int kTT = 256;       // threads per tile CTA
constexpr int kHS = 2048;      // plan hash set (>= 19 kTI candidates)
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr uint32_t kInt = 0x80000000u;  // hash value flag: a package of the chunk
constexpr size_t kTSmem = (size_t)kTCap * (256 + 16 + 4);

static_assert(2 + kTI + 18 * kTI <= kHS, "plan hash set too small");
static_assert(kTCap <= 4096, "slots are 12-bit in the row list");

// -------------------------------------------------------------- plan ---

__device__ __forceinline__ uint32_t spread3(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void k_tp_keys(const uint32_t* __restrict__ meta_cell, int64_t n_act, uint32_t nx,
                          uint32_t ny, uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_act) return;
    const uint32_t c = meta_cell[2 + i];
    const uint32_t x = c % nx, y = (c / nx) % ny, z = c / (nx * ny);
    key[i] = spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
    val[i] = (uint32_t)(2 + i);
}

// the 18 face / edge relations o: neighbour-table slot and the row masks of
// H = P + o (bits 0..15: distance <= 1, bits 16..31: distance <= 2)
struct Rel {
    int slot;
    uint32_t mask;
};
__device__ __forceinline__ Rel relation(int q) {
    // enumerate o in {-1,0,1}^3 with |o|_1 in {1, 2}: 18 of the 27 slots
    int cnt = 0;
    for (int s = 0; s < 27; ++s) {
        const int ox = s % 3 - 1, oy = (s / 3) % 3 - 1, oz = s / 9 - 1;
        const int l1 = abs(ox) + abs(oy) + abs(oz);
        if (l1 < 1 || l1 > 2) continue;
        if (cnt++ != q) continue;
        uint32_t m = 0;
        for (int r = 0; r < 16; ++r) {
            const int j = r & 3, k = r >> 2;
            const int dy = oy == 1 ? j + 1 : (oy == -1 ? 4 - j : 0);
            const int dz = oz == 1 ? k + 1 : (oz == -1 ? 4 - k : 0);
            const int d = (ox != 0) + dy + dz;
            if (d <= 1) m |= 1u << r;
            if (d <= 2) m |= 1u << (16 + r);
        }
        return {s, m};
    }
    return {13, 0};
}

__device__ __forceinline__ int h_slot(uint32_t key) { return (int)((key * 2654435761u) >> 21); }

__device__ __forceinline__ int h_insert(uint32_t* hk, uint32_t key) {
    int h = h_slot(key);
    while (true) {
        const uint32_t prev = atomicCAS(&hk[h], kEmpty, key);
        if (prev == kEmpty || prev == key) return h;
        h = (h + 1) & (kHS - 1);
    }
}
__device__ __forceinline__ int h_find(const uint32_t* hk, uint32_t key) {
    int h = h_slot(key);
    while (true) {
        const uint32_t k = hk[h];
        if (k == key) return h;
        if (k == kEmpty) return -1;
        h = (h + 1) & (kHS - 1);
    }
}

struct TPlanDev {
    int4* cnt;
    uint32_t* ids;
    uint4* lf;
    uint16_t* m2;
    uint16_t* comp;
    uint32_t* ctr;
    int64_t t_cap;
};

// One CTA per level-0 chunk of kTI sorted packages; chunks that overflow a
// tile are halved on a CTA-local stack.  Tiles are numbered in emission order.
__global__ void __launch_bounds__(256) k_tp_plan(const uint32_t* __restrict__ sorted, int64_t n_act,
                                                 const uint32_t* __restrict__ nb,
                                                 const uint32_t* __restrict__ face, TPlanDev P) {
    __shared__ uint32_t hk[kHS], hv[kHS], hm[kHS];
    __shared__ uint32_t sid[kTCap];
    __shared__ long long st_a[32];
    __shared__ int st_n[32];
    __shared__ int sp, cur_n, s_t;
    __shared__ long long cur_a;
    __shared__ int wsum[8][2];
    __shared__ Rel rel[18];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid < 18) rel[tid] = relation(tid);
    if (tid == 0) {
        const long long a0 = (long long)blockIdx.x * kTI;
        st_a[0] = a0;
        st_n[0] = (int)min((long long)kTI, (long long)n_act - a0);
        sp = 1;
    }
    __syncthreads();
    while (true) {
        if (tid == 0) {
            if (sp > 0) {
                --sp;
                cur_a = st_a[sp];
                cur_n = st_n[sp];
            } else {
                cur_n = 0;
            }
        }
        __syncthreads();
        const int n = cur_n;
        const long long a = cur_a;
        if (n == 0) break;
        for (int h = tid; h < kHS; h += 256) {
            hk[h] = kEmpty;
            hv[h] = 0;
            hm[h] = 0;
        }
        __syncthreads();
        for (int i = tid; i < n; i += 256) hv[h_insert(hk, sorted[a + i])] = kInt | (uint32_t)(2 + i);
        __syncthreads();
        for (int p = tid; p < 18 * n; p += 256) {
            const int i = p / 18;
            const Rel R = rel[p - 18 * i];
            const uint32_t nid = __ldg(nb + (size_t)sorted[a + i] * 27 + R.slot);
            if (nid < 2) continue;
            const int h = h_insert(hk, nid);
            // chunk entries were flagged before the barrier above; a halo
            // entry's value is 0 until the compaction below
            if (!(hv[h] & kInt)) atomicOr(&hm[h], R.mask);
        }
        __syncthreads();
        // compaction of the halo entries (8 hash entries per thread, in order)
        int cH = 0, cC = 0;
        for (int e = 0; e < kHS / 256; ++e) {
            const int h = tid * (kHS / 256) + e;
            if (hk[h] != kEmpty && !(hv[h] & kInt)) {
                ++cH;
                cC += __popc(hm[h] & 0xffffu);
            }
        }
        int xH = cH, xC = cC;  // inclusive warp scan
        for (int d = 1; d < 32; d <<= 1) {
            const int tH = __shfl_up_sync(0xffffffffu, xH, d), tC = __shfl_up_sync(0xffffffffu, xC, d);
            if (lane >= d) {
                xH += tH;
                xC += tC;
            }
        }
        if (lane == 31) {
            wsum[wid][0] = xH;
            wsum[wid][1] = xC;
        }
        __syncthreads();
        int oH = xH - cH, oC = xC - cC, tH = 0, tC = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < wid) {
                oH += wsum[w][0];
                oC += wsum[w][1];
            }
            tH += wsum[w][0];
            tC += wsum[w][1];
        }
        if (2 + n + tH > kTCap || tC > kTComp) {
            if (tid == 0) {
                if (n == 1) {
                    atomicOr(P.ctr + 1, 2u);  // cannot happen: 2 + 1 + 18 slots, <= 288 rows
                } else {
                    st_a[sp] = a + n / 2;
                    st_n[sp] = n - n / 2;
                    st_a[sp + 1] = a;
                    st_n[sp + 1] = n / 2;
                    sp += 2;
                }
            }
            __syncthreads();
            continue;
        }
        if (tid == 0) {
            const uint32_t t = atomicAdd(P.ctr, 1u);
            if ((int64_t)t >= P.t_cap) atomicOr(P.ctr + 1, 1u);
            s_t = (int)t;
        }
        __syncthreads();
        const int64_t t = (uint32_t)s_t;
        if (t >= P.t_cap) continue;  // counted; the host re-plans with the total
        const int nS = 2 + n + tH;
        uint32_t* ids = P.ids + t * kTCap;
        uint16_t* m2 = P.m2 + t * kTCap;
        uint16_t* comp = P.comp + t * kTComp;
        for (int e = 0; e < kHS / 256; ++e) {
            const int h = tid * (kHS / 256) + e;
            if (hk[h] != kEmpty && !(hv[h] & kInt)) {
                const int slot = 2 + n + oH++;
                hv[h] = (uint32_t)slot;
                sid[slot] = hk[h];
                m2[slot] = (uint16_t)(hm[h] >> 16);
                for (uint32_t m = hm[h] & 0xffffu; m; m &= m - 1)
                    comp[oC++] = (uint16_t)((slot << 4) | (__ffs(m) - 1));
            }
        }
        for (int i = tid; i < n + 2; i += 256) sid[i] = i < 2 ? (uint32_t)i : sorted[a + i - 2];
        if (tid == 0) P.cnt[t] = make_int4(n, tH, tC, 0);
        __syncthreads();
        for (int s = tid; s < nS; s += 256) {
            const uint32_t gid = sid[s];
            ids[s] = gid;
            uint32_t l[6] = {0, 0, 0, 0, 0, 0};
            if (s >= 2)
                for (int r = 0; r < 6; ++r) {
                    const uint32_t f = __ldg(face + (size_t)gid * 8 + r);
                    if (f < 2) {
                        l[r] = f;
                    } else {
                        const int h = h_find(hk, f);
                        l[r] = h < 0 ? 0u : (hv[h] & 0xffffu);  // not staged: never read
                        // a tile package's face neighbours are all staged
                        // (6 of the 18 relations); checked, not assumed
                        if (s < 2 + n && h < 0) atomicOr(P.ctr + 1, 4u);
                    }
                    if (l[r] >= (uint32_t)nS) atomicOr(P.ctr + 1, 4u);
                }
            P.lf[t * kTCap + s] =
                make_uint4(l[0] | (l[1] << 16), l[2] | (l[3] << 16), l[4] | (l[5] << 16), 0u);
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------- sweeps ----

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void f4(const float4 v, float (&r)[4]) {
    r[0] = v.x;
    r[1] = v.y;
    r[2] = v.z;
    r[3] = v.w;
}

// sweep of x-row r of slot s from the staged rows (the cross of load_cross2 in
// sg_stencil.cu, with tile-local neighbour slots)
__device__ __forceinline__ float4 row_step(const float4* D, const uint4* LF, int s, int r,
                                           const StC<float>& c) {
    const int j = r & 3, k = r >> 2;
    const uint4 L = LF[s];
    const float4* P = D + s * 16;
    float cc[4], ym[4], yp[4], zm[4], zp[4], o[4];
    f4(P[r], cc);
    f4(j > 0 ? P[r - 1] : D[(L.y & 0xffffu) * 16 + 3 + 4 * k], ym);
    f4(j < 3 ? P[r + 1] : D[(L.y >> 16) * 16 + 4 * k], yp);
    f4(k > 0 ? P[r - 4] : D[(L.z & 0xffffu) * 16 + j + 12], zm);
    f4(k < 3 ? P[r + 4] : D[(L.z >> 16) * 16 + j], zp);
    const float xm = reinterpret_cast<const float*>(D + (L.x & 0xffffu) * 16 + r)[3];
    const float xp = reinterpret_cast<const float*>(D + (L.x >> 16) * 16 + r)[0];
    godunov_row(cc, xm, xp, ym, yp, zm, zp, c, o);
    return make_float4(o[0], o[1], o[2], o[3]);
}

// the two x-rows (j, k), (j, k + 2) of slot s (8 lanes per package, lane
// (j, k), k in {0, 1}): the cross of load_cross2 (sg_stencil.cu) from the
// staged slots, then the ReinitOp arithmetic -- bit-identical to k_sweep
__device__ __forceinline__ void pkg_step(const float4* D, const uint4* LF, int s, int j, int k,
                                         const StC<float>& c, float4& out0, float4& out1) {
    const uint4 L = LF[s];
    const int nxm = L.x & 0xffff, nxp = L.x >> 16, nym = L.y & 0xffff, nyp = L.y >> 16;
    const int nzm = L.z & 0xffff, nzp = L.z >> 16;
    const float4* P = D + s * 16;
    const int r0 = j + 4 * k, r1 = r0 + 8;
    float c0[4], c1[4], zlo[4], zmid[4], zhi[4], ym0[4], yp0[4], ym1[4], yp1[4], o0[4], o1[4];
    f4(P[r0], c0);
    f4(P[r1], c1);
    f4(P[r0 + 4], zmid);
    f4(k == 0 ? D[nzm * 16 + j + 12] : P[j], zlo);
    f4(k == 0 ? P[j + 12] : D[nzp * 16 + j], zhi);
    f4(j > 0 ? P[r0 - 1] : D[nym * 16 + 3 + 4 * k], ym0);
    f4(j < 3 ? P[r0 + 1] : D[nyp * 16 + 4 * k], yp0);
    f4(j > 0 ? P[r1 - 1] : D[nym * 16 + 3 + 4 * (k + 2)], ym1);
    f4(j < 3 ? P[r1 + 1] : D[nyp * 16 + 4 * (k + 2)], yp1);
    const float* Xm = reinterpret_cast<const float*>(D + nxm * 16);
    const float* Xp = reinterpret_cast<const float*>(D + nxp * 16);
    const float xm0 = Xm[4 * r0 + 3], xm1 = Xm[4 * r1 + 3], xp0 = Xp[4 * r0], xp1 = Xp[4 * r1];
    godunov_row(c0, xm0, xp0, ym0, yp0, zlo, zmid, c, o0);
    godunov_row(c1, xm1, xp1, ym1, yp1, zmid, zhi, c, o1);
    out0 = make_float4(o0[0], o0[1], o0[2], o0[3]);
    out1 = make_float4(o1[0], o1[1], o1[2], o1[3]);
}

// TMA bulk copy global -> shared, completing on an mbarrier (1-D, 16 B units)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned tx) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(b), "r"(parity)
        : "memory");
}

// Two Jacobi sweeps phi_in -> phi_out over every active package, one tile per
// CTA iteration (persistent: tile t = blockIdx.x + i * gridDim.x).  Shared
// memory: kTCap package slots of 64 floats, their face slots, ids, row masks.
// Staging: TMA bulk copies (one per tile package, one per run of consecutive
// staged rows of a halo package) completing on one mbarrier phase per tile;
// the next tile's plan rows are prefetched into registers during sweep 2.
__global__ void __launch_bounds__(kTT, 2) k_tsweep(const float* __restrict__ in,
                                                   float* __restrict__ out, TPlanDev P,
                                                   StC<float> c) {
    extern __shared__ __align__(128) unsigned char sm_raw[];
    float4* D = reinterpret_cast<float4*>(sm_raw);
    uint4* LF = reinterpret_cast<uint4*>(D + kTCap * 16);
    uint32_t* ID = reinterpret_cast<uint32_t*>(LF + kTCap);
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const int g8 = tid & 7, j = g8 & 3, k = g8 >> 2, grp = tid >> 3;  // 32 package groups
    const uint32_t nt = (uint32_t)min((long long)*(volatile uint32_t*)P.ctr, (long long)P.t_cap);
    if (tid == 0) {
        mbar_init(&bar, kTT);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    static_assert(kTCap <= 2 * kTT, "two plan slots per thread");
    constexpr int kPI = (kTI + 31) / 32;            // tile packages per 8-lane group
    constexpr int kHR = (kTComp + kTT - 1) / kTT;   // first-sweep halo rows per thread
    int4 cn = make_int4(0, 0, 0, 0);
    uint32_t pid[2] = {0, 0};
    uint4 plf[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    uint16_t pm2[2] = {0, 0};
    auto fetch = [&](uint32_t t) {
        cn = __ldg(P.cnt + t);
        const int nS = 2 + cn.x + cn.y;
        const size_t tb = (size_t)t * kTCap;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int s = tid + h * kTT;
            if (s < nS) {
                pid[h] = __ldg(P.ids + tb + s);
                plf[h] = __ldg(P.lf + tb + s);
                pm2[h] = __ldg(P.m2 + tb + s);
            }
        }
    };
    if (blockIdx.x < nt) fetch(blockIdx.x);
    unsigned phase = 0;
    for (uint32_t t = blockIdx.x; t < nt; t += gridDim.x) {
        const int nI = cn.x, nC = cn.z, nS = 2 + nI + cn.y;
        // stage: every thread arrives once with the bytes it issues
        uint32_t tx = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int s = tid + h * kTT;
            if (s < nS) {
                ID[s] = pid[h];
                LF[s] = plf[h];
                if (s < 2 + nI) {
                    tx += 256;
                } else {
                    for (uint32_t m = pm2[h]; m;) {  // runs of consecutive rows
                        const int r0 = __ffs(m) - 1;
                        const uint32_t run = ~(m >> r0);
                        const int len = run ? __ffs(run) - 1 : 16 - r0;
                        tx += 16u * len;
                        m &= ~(((1u << len) - 1u) << r0);
                    }
                }
            }
        }
        mbar_arrive_tx(&bar, tx);
        // the slots were written by threads (generic proxy) in the previous
        // tile; order those writes before the TMA (async proxy) overwrites
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int s = tid + h * kTT;
            if (s < nS) {
                const float* src = in + (size_t)pid[h] * 64;
                if (s < 2 + nI) {
                    bulk_g2s(D + s * 16, src, 256, &bar);
                } else {
                    for (uint32_t m = pm2[h]; m;) {
                        const int r0 = __ffs(m) - 1;
                        const uint32_t run = ~(m >> r0);
                        const int len = run ? __ffs(run) - 1 : 16 - r0;
                        bulk_g2s(D + s * 16 + r0, src + 4 * r0, 16u * len, &bar);
                        m &= ~(((1u << len) - 1u) << r0);
                    }
                }
            }
        }
        // the first-sweep halo row list, read while the stage is in flight
        uint32_t ce[kHR];
#pragma unroll
        for (int q = 0; q < kHR; ++q) {
            const int w = tid + kTT * q;
            ce[q] = w < nC ? __ldg(P.comp + (size_t)t * kTComp + w) : 0u;
        }
        __syncthreads();  // ID / LF visible
        mbar_wait(&bar, phase);
        phase ^= 1u;
        // sweep 1: tile packages (two rows per lane) and the halo rows at
        // distance 1 (one row per lane), kept in registers until every
        // thread has read its inputs
        float4 a0[kPI], a1[kPI], hr[kHR];
#pragma unroll
        for (int q = 0; q < kPI; ++q) {
            const int pi = grp + 32 * q;
            if (pi < nI) pkg_step(D, LF, 2 + pi, j, k, c, a0[q], a1[q]);
        }
#pragma unroll
        for (int q = 0; q < kHR; ++q) {
            const int w = tid + kTT * q;
            if (w < nC) hr[q] = row_step(D, LF, (int)(ce[q] >> 4), (int)(ce[q] & 15u), c);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kPI; ++q) {
            const int pi = grp + 32 * q;
            if (pi < nI) {
                D[(2 + pi) * 16 + j + 4 * k] = a0[q];
                D[(2 + pi) * 16 + j + 4 * k + 8] = a1[q];
            }
        }
#pragma unroll
        for (int q = 0; q < kHR; ++q) {
            const int w = tid + kTT * q;
            if (w < nC) D[(ce[q] >> 4) * 16 + (ce[q] & 15u)] = hr[q];
        }
        __syncthreads();
        if (t + gridDim.x < nt) fetch(t + gridDim.x);
        // sweep 2: the tile packages, straight to HBM
#pragma unroll
        for (int q = 0; q < kPI; ++q) {
            const int pi = grp + 32 * q;
            if (pi < nI) {
                float4 v0, v1;
                pkg_step(D, LF, 2 + pi, j, k, c, v0, v1);
                float4* O = reinterpret_cast<float4*>(out + (size_t)ID[2 + pi] * 64);
                O[j + 4 * k] = v0;
                O[j + 4 * k + 8] = v1;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------- host ----

// Opt-in (SG_TSWEEP=1, read at every call): measured slower than the
// single-sweep chain on C2 and C3 (profiles/README.md "two-sweep tiles").
static bool tsweep_enabled() {
    const char* e = std::getenv("SG_TSWEEP");
    return e && e[0] == '1';
}

static void plan_alloc(sg_grid* g, TPlan* tp, int64_t t_cap, cudaStream_t s) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t b_cnt = al(sizeof(int4) * t_cap), b_ids = al(sizeof(uint32_t) * kTCap * t_cap),
                 b_lf = al(sizeof(uint4) * kTCap * t_cap), b_m2 = al(sizeof(uint16_t) * kTCap * t_cap),
                 b_cp = al(sizeof(uint16_t) * kTComp * t_cap), b_ct = al(sizeof(uint32_t) * 2);
    char* p = (char*)g->alloc(b_cnt + b_ids + b_lf + b_m2 + b_cp + b_ct, s);
    tp->arena = p;
    tp->t_cap = t_cap;
    tp->cnt = (int4*)p;
    p += b_cnt;
    tp->ids = (uint32_t*)p;
    p += b_ids;
    tp->lf = (uint4*)p;
    p += b_lf;
    tp->m2 = (uint16_t*)p;
    p += b_m2;
    tp->comp = (uint16_t*)p;
    p += b_cp;
    tp->ctr = (uint32_t*)p;
}

static TPlanDev dev_view(const TPlan* tp) {
    return TPlanDev{tp->cnt, tp->ids, tp->lf, tp->m2, tp->comp, tp->ctr, tp->t_cap};
}

// Build the plan on stream s (one host synchronisation: the emitted tile count
// and the capacity flag).
static void tplan_build(sg_grid* g, TPlan* tp, cudaStream_t s) {
    const int64_t n_act = g->n_pkg - 2;
    uint32_t *kin = nullptr, *kout = nullptr, *vin = nullptr, *vout = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    int bits = 0;
    while ((1 << bits) < std::max({g->gc.n[0], g->gc.n[1], g->gc.n[2]})) ++bits;
    SG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, kout, vin, vout, (int)n_act, 0,
                                            3 * bits, s));
    char* scratch = (char*)dalloc(4 * ((sizeof(uint32_t) * n_act + 255) & ~(size_t)255) + tmp_bytes, s);
    const size_t step = (sizeof(uint32_t) * n_act + 255) & ~(size_t)255;
    kin = (uint32_t*)scratch;
    kout = (uint32_t*)(scratch + step);
    vin = (uint32_t*)(scratch + 2 * step);
    vout = (uint32_t*)(scratch + 3 * step);
    tmp = scratch + 4 * step;
    k_tp_keys<<<(unsigned)ceil_div(n_act, 256), 256, 0, s>>>(g->meta_cell, n_act, (uint32_t)g->gc.n[0],
                                                           (uint32_t)g->gc.n[1], kin, vin);
    SG_LAUNCHED();
    SG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, vout, (int)n_act, 0,
                                            3 * bits, s));
    const int64_t chunks = ceil_div(n_act, kTI);
    int64_t t_cap = chunks + chunks / 4 + 64;
    for (int attempt = 0; attempt < 2; ++attempt) {
        plan_alloc(g, tp, t_cap, s);
        SG_CUDA(cudaMemsetAsync(tp->ctr, 0, 2 * sizeof(uint32_t), s));
        k_tp_plan<<<(unsigned)chunks, 256, 0, s>>>(vout, n_act, g->nb, g->face, dev_view(tp));
        SG_LAUNCHED();
        uint32_t h[2] = {0, 0};
        SG_CUDA(cudaMemcpyAsync(h, tp->ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
        SG_CUDA(cudaStreamSynchronize(s));
        if (h[1] & 2u) throw Error(SG_ERR_STATE, "tile plan: a single package overflows a tile");
        if (h[1] & 4u) throw Error(SG_ERR_STATE, "tile plan: a face slot outside its tile");
        if (!(h[1] & 1u)) {
            tp->n_tiles = h[0];
            tp->state = 1;
            break;
        }
        g->release(tp->arena, s);  // too few tiles reserved: re-plan with the count
        tp->arena = nullptr;
        t_cap = h[0];
    }
    SG_CUDA(cudaFreeAsync(scratch, s));
    if (tp->state != 1) throw Error(SG_ERR_STATE, "tile plan: capacity");
}

// Whether reinit of g can run two sweeps per launch; builds the plan on first
// use.  fp32 grids over the whole domain (not partitioned, no ghost planes),
// background grid <= 1024^3 cells (30-bit Morton keys).
bool tsweep_ready(sg_grid* g, cudaStream_t s) {
    if (!tsweep_enabled() || g->dtype != SG_F32 || g->partitioned()) return false;
    if (g->own_lo != 2 || g->own_hi != g->n_pkg || g->n_pkg <= 2) return false;
    if (g->gc.zs_lo != 0 || g->gc.zs_hi != g->gc.n[2]) return false;
    for (int k = 0; k < 3; ++k)
        if (g->gc.n[k] > 1024) return false;
    if (!g->tplan) g->tplan = new TPlan();
    TPlan* tp = g->tplan;
    if (tp->state == 0) {
        try {
            tplan_build(g, tp, s);
        } catch (...) {
            if (tp->arena) g->release(tp->arena, s);
            tp->arena = nullptr;
            tp->state = -1;
            throw;
        }
    }
    return tp->state == 1;
}

const void* tsweep_key(const sg_grid* g) { return g->tplan ? g->tplan->arena : nullptr; }

// one launch = two sweeps phi[cur] -> phi[1 - cur]
void tsweep_launch(sg_grid* g, int cur, float inv_dx, float dx2, float cdx, float ncfl,
                   cudaStream_t s) {
    // per device (the attribute belongs to the current context); cheap, and
    // only called while a graph is captured or for eager launches
    SG_CUDA(cudaFuncSetAttribute(k_tsweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTSmem));
    const TPlan* tp = g->tplan;
    const int blocks = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)tp->n_tiles, resident_blocks((const void*)k_tsweep, kTT, kTSmem)));
    StC<float> c{};
    c.inv_dx = inv_dx;
    c.dx2 = dx2;
    c.cdx = cdx;
    c.ncfl = ncfl;
    k_tsweep<<<blocks, kTT, kTSmem, s>>>((const float*)g->phi[cur], (float*)g->phi[1 - cur],
                                         dev_view(tp), c);
    SG_CUDA(cudaGetLastError());  // counted by the caller (one per pass)
}

void tplan_invalidate(sg_grid* g, cudaStream_t s) {
    if (!g->tplan) return;
    if (g->tplan->arena) g->release(g->tplan->arena, s);
    *g->tplan = TPlan();
}

void tplan_release(sg_grid* g, cudaStream_t) {
    delete g->tplan;  // device memory: one of the grid's allocations
    g->tplan = nullptr;
}

}  // namespace sg
