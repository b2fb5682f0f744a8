// sg_build.cu -- sg_build (K1-K4), grid lifetime, info/view, slab helpers.
//
// Compiled with -fmad=false: the fp64 signed distance (sdf.cuh) and the
// position arithmetic must be the separately rounded operations of DESIGN.md
// "O1"/"O2" so that the core predicate and the initial phi are reproducible.
//
// Pipeline (steps 1-5 of the initialization, single layer):
//   K1 k_tag      : f at every background-cell centre -> core / sign bitmasks
//   K2 k_count    : inner tagging (26-neighbourhood dilation of 32-cell words),
//                   per-tile active counts
//      k_scan     : exclusive scan of tile counts (ordered compaction, R-1)
//      -- one D2H read of the package count (P:468-471 analogue) --
//      k_scatter  : block scan inside each tile -> ids 2.. in linear order;
//                   background table, meta (cell, category)
//      k_planes   : first package id per background plane (slab ranges)
//   K3 k_nb       : 27-neighbour package table
//   K4 k_phi_init : phi = init_scale * f at the 64 data points
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <chrono>
#include <cstring>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>

#include "sdf.cuh"
#include "sg_internal.cuh"

namespace sg {

std::atomic<uint64_t> g_launches{0};

static thread_local std::string t_last_error;

void set_last_error(const std::string& m) { t_last_error = m; }
void clear_last_error() { t_last_error.clear(); }

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    std::string m = std::string(cudaGetErrorName(e)) + " (" + cudaGetErrorString(e) + ") in " +
                    what + " at " + file + ":" + std::to_string(line);
    if (e == cudaErrorMemoryAllocation) throw Error(SG_ERR_OOM, m);
    throw Error(SG_ERR_CUDA, m);
}

namespace {
struct OccKey {
    const void* k;
    int dev, threads;
    size_t smem;
    bool operator==(const OccKey& o) const {
        return k == o.k && dev == o.dev && threads == o.threads && smem == o.smem;
    }
};
std::mutex g_occ_mu;
std::vector<std::pair<OccKey, int>> g_occ;
std::vector<int> g_sms;
}  // namespace

int sm_count() {
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_occ_mu);
    if ((int)g_sms.size() <= dev) g_sms.resize(dev + 1, 0);
    if (!g_sms[dev]) SG_CUDA(cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev));
    return g_sms[dev];
}

int resident_blocks(const void* kernel, int threads, size_t smem) {
    const int sms = sm_count();
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    const OccKey key{kernel, dev, threads, smem};
    {
        std::lock_guard<std::mutex> lk(g_occ_mu);
        for (auto& e : g_occ)
            if (e.first == key) return e.second;
    }
    int per = 0;
    SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem));
    const int r = std::max(1, sms * per);
    std::lock_guard<std::mutex> lk(g_occ_mu);
    g_occ.push_back({key, r});
    return r;
}

// the library's own stream-ordered pool per device: released memory stays
// in it (rebuilding a grid every step reuses it) without touching the
// device's default pool, which other code in the process may use
static std::mutex g_pool_mu;
static std::vector<cudaMemPool_t> g_pools;

static cudaMemPool_t lib_pool() {
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if ((int)g_pools.size() <= dev) g_pools.resize(dev + 1, nullptr);
    if (!g_pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool;
        SG_CUDA(cudaMemPoolCreate(&pool, &props));
        uint64_t thr = UINT64_MAX;
        SG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        g_pools[dev] = pool;
    }
    return g_pools[dev];
}

void* dalloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    if (bytes == 0) bytes = 256;
    SG_CUDA(cudaMallocFromPoolAsync(&p, bytes, lib_pool(), s));
    return p;
}

// ------------------------------------------------------------- kernels ---

constexpr int kTB = 256;  // threads (words) per compaction tile: 8192 cells

// Tag bitmasks: per tag plane z and row y, W = ceil(nx / 32) words; bit i of
// word q is cell x = 32 q + i.  core = |f(centre)| < l_c, neg = f(centre) < 0.
struct Bits {
    const uint32_t* core;
    const uint32_t* neg;
    int32_t W;
    int32_t zt_lo;
    FastDiv fdW;  // division by W (word index -> row, column)
    __device__ __forceinline__ int64_t idx(const GridC& gc, int z, int y, int q) const {
        return ((int64_t)(z - zt_lo) * gc.n[1] + y) * W + q;
    }
};

// K1 -- f at every background-cell centre of the tag planes [zt_lo, zt_hi)
// (O2: centre = lower + (c + 0.5) l_c); warp ballots pack the core and sign
// predicates into 32-cell words.
//
// Work unit: a block of 32 x 1 x 4 cells (one word in 4 consecutive planes);
// a lane evaluates one (x, y) column of 4 planes (the (x, y)-only terms of
// each primitive are shared, bit-identically).  A warp owns 32 such blocks
// along y.
// Lipschitz cull: the analytic f is a (union of) exact signed distance(s),
// hence 1-Lipschitz.  The cell centres of a block lie within
// R = |(15.5, 0, 1.5)| l_c of its centre c.  If |f(c)| > l_c + R + eps (eps far
// above the rounding of f), no cell of the block is core and every cell has
// the sign of f(c): the per-cell evaluation is skipped and the predicates are
// exactly those of the per-cell fp64 evaluation.  The 32 block-centre values
// of a warp are computed by its 32 lanes in parallel.
__global__ void __launch_bounds__(128, 4) k_tag_cull(GridC gc, Geom geom, int32_t zt_lo, int32_t zt_hi,
                                             int32_t W, int32_t cull,
                                             uint32_t* __restrict__ core_w,
                                             uint32_t* __restrict__ neg_w) {
    const int lane = threadIdx.x & 31;
    const int q = blockIdx.x;                                  // word (32 x-cells)
    const int y0 = 32 * blockIdx.y;                            // first row of the warp
    const int z0 = zt_lo + 4 * (4 * (int)blockIdx.z + (threadIdx.x >> 5));  // first plane
    if (z0 >= zt_hi) return;                                   // warp-uniform
    const double R = 15.572411502397436 * gc.cell;             // sqrt(15.5^2 + 1.5^2) l_c
    const double eps = 1e-9 * (gc.cell + fabs(gc.lower[0]) + fabs(gc.lower[1]) +
                               fabs(gc.lower[2]) + gc.upper[0] + gc.upper[1] + gc.upper[2]);
    bool skip_mine = false, neg_mine = false;
    // primitives of a union that provably exceed the minimum at every cell
    // of the block (1-Lipschitz, radius R from the centre) are not evaluated
    // there: the minimum over the rest is the same value, bit for bit
    uint32_t mask_mine = (geom.n >= 32 ? 0xFFFFFFFFu : (1u << geom.n) - 1u);
    if (cull) {
        const double bx = gc.lower[0] + (double)(32 * q + 16) * gc.cell;
        const double by = gc.lower[1] + ((double)(y0 + lane) + 0.5) * gc.cell;
        const double bz = gc.lower[2] + (double)(z0 + 2) * gc.cell;
        double fc;
        if (geom.n > 1 && !geom.n_leak) {
            double fi[SG_MAX_PRIMS];
            fc = 0.0;
            for (int i = 0; i < geom.n; ++i) {
                fi[i] = sd_prim(geom.kind[i], geom.p[i], bx, by, bz);
                fc = i == 0 ? fi[i] : fmin(fc, fi[i]);
            }
            mask_mine = 0u;
            for (int i = 0; i < geom.n; ++i)
                if (fi[i] - R <= fc + R + eps) mask_mine |= 1u << i;
        } else {
            fc = sd_eval(geom, bx, by, bz);
        }
        skip_mine = fabs(fc) > gc.cell + R + eps;
        neg_mine = fc < 0.0;
    }
    const uint32_t skip = __ballot_sync(0xffffffffu, skip_mine);
    const uint32_t negb = __ballot_sync(0xffffffffu, neg_mine);
    const int cx = 32 * q + lane;
    const bool in = cx < gc.n[0];
    const uint32_t valid = __ballot_sync(0xffffffffu, in);
    const int nrows = min(32, gc.n[1] - y0);
    for (int b = 0; b < nrows; ++b) {
        const int cy = y0 + b;
        uint32_t cw[4], nw[4];
        if ((skip >> b) & 1u) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                cw[k] = 0u;
                nw[k] = ((negb >> b) & 1u) ? valid : 0u;
            }
        } else {
            const double x = gc.lower[0] + ((double)cx + 0.5) * gc.cell;
            const double y = gc.lower[1] + ((double)cy + 0.5) * gc.cell;
            double z[4], f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) z[k] = gc.lower[2] + ((double)(z0 + k) + 0.5) * gc.cell;
            const uint32_t mask = __shfl_sync(0xffffffffu, mask_mine, b);
            if (in) sd_eval_col_mask<4>(geom, mask, x, y, z, f);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                cw[k] = __ballot_sync(0xffffffffu, in && fabs(f[k]) < gc.cell);
                nw[k] = __ballot_sync(0xffffffffu, in && f[k] < 0.0);
            }
        }
        if (lane < 4 && z0 + lane < zt_hi) {
            const int k = lane;
            const int64_t i = ((int64_t)(z0 + k - zt_lo) * gc.n[1] + cy) * W + q;
            core_w[i] = k == 0 ? cw[0] : k == 1 ? cw[1] : k == 2 ? cw[2] : cw[3];
            neg_w[i] = k == 0 ? nw[0] : k == 1 ? nw[1] : k == 2 ? nw[2] : nw[3];
        }
    }
}

// K1 of a refined layer (NEXT-4 multi-resolution: "For
// successive layers, only the cells covered by the coarse core cells will be
// evaluated"): a fine cell under a parent core cell is evaluated; any other
// takes its parent cell's sign.  Equal to full tagging: a fine core cell
// (|f| < l_f) has |f(parent centre)| < l_f + sqrt(3)/2 l_f < 2 l_f, a core
// parent; a non-core parent (|f| >= 2 l_f at its centre) has one sign over
// its whole cell (1-Lipschitz, half-diagonal sqrt(3) l_f).
__global__ void __launch_bounds__(256) k_tag_refine(GridC gc, Geom geom, int32_t W, ParentBits pb,
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
            const double f = sd_eval(geom, gc.lower[0] + ((double)cx + 0.5) * gc.cell,
                                     gc.lower[1] + ((double)cy + 0.5) * gc.cell,
                                     gc.lower[2] + ((double)cz + 0.5) * gc.cell);
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

// K1 without the cull (band-dense domains): a thread owns an (x, y) column of
// 4 planes, a warp 32 consecutive x-cells.
__global__ void __launch_bounds__(256) k_tag(GridC gc, Geom geom, int32_t zt_lo, int32_t zt_hi,
                                             int32_t W, uint32_t* __restrict__ core_w,
                                             uint32_t* __restrict__ neg_w) {
    const int cx = blockIdx.x * blockDim.x + threadIdx.x;
    const int cy = blockIdx.y;
    const int z0 = zt_lo + 4 * (int)blockIdx.z;
    const double x = gc.lower[0] + ((double)cx + 0.5) * gc.cell;
    const double y = gc.lower[1] + ((double)cy + 0.5) * gc.cell;
    double z[4], f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) z[k] = gc.lower[2] + ((double)(z0 + k) + 0.5) * gc.cell;
    if (cx < gc.n[0]) sd_eval_col<4>(geom, x, y, z, f);
    const int q = cx >> 5;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool in = cx < gc.n[0];
        const uint32_t cw = __ballot_sync(0xffffffffu, in && fabs(f[k]) < gc.cell);
        const uint32_t nw = __ballot_sync(0xffffffffu, in && f[k] < 0.0);
        if ((threadIdx.x & 31) == 0 && q < W && z0 + k < zt_hi) {
            const int64_t i = ((int64_t)(z0 + k - zt_lo) * gc.n[1] + cy) * W + q;
            core_w[i] = cw;
            neg_w[i] = nw;
        }
    }
}

__device__ __forceinline__ uint32_t valid_bits(const GridC& gc, int q, int W) {
    const int rem = gc.n[0] - 32 * (W - 1);  // cells in the last word of a row
    return (q < W - 1 || rem == 32) ? 0xffffffffu : ((1u << rem) - 1u);
}

// active = core dilated by the 26-neighbourhood (R-3, clipped to the domain):
// OR of the x-dilated words of the 3 x 3 rows around (y, z)
__device__ __forceinline__ uint32_t active_word(const GridC& gc, const Bits& b, int z, int y,
                                                int q) {
    uint32_t act = 0;
    for (int dz = -1; dz <= 1; ++dz) {
        const int zz = z + dz;
        if (zz < 0 || zz >= gc.n[2]) continue;
        for (int dy = -1; dy <= 1; ++dy) {
            const int yy = y + dy;
            if (yy < 0 || yy >= gc.n[1]) continue;
            const int64_t i = b.idx(gc, zz, yy, q);
            const uint32_t w = __ldg(b.core + i);
            const uint32_t wl = q > 0 ? __ldg(b.core + i - 1) : 0u;
            const uint32_t wr = q < b.W - 1 ? __ldg(b.core + i + 1) : 0u;
            act |= w | (w << 1) | (wl >> 31) | (w >> 1) | (wr << 31);
        }
    }
    return act & valid_bits(gc, q, b.W);
}

// the same for word t = (row, q) of a warp whose lanes hold consecutive
// words (every lane of the warp calls it; `in`: t is a word of the planes):
// the x-neighbour words of a row come from the neighbouring lanes by shuffle
// where those hold them (one load per row instead of three).  Bit-identical
// to active_word.
__device__ __forceinline__ uint32_t active_word_warp(const GridC& gc, const Bits& b, bool in,
                                                     int z, int y, int q) {
    const int lane = threadIdx.x & 31;
    uint32_t act = 0;
    // word index of (z, y, q) and the row / plane strides (the 3 x 3 rows
    // differ by constants)
    const int64_t i0 = in ? b.idx(gc, z, y, q) : 0;
    const int64_t pw = (int64_t)gc.n[1] * b.W;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
            const int zz = z + dz, yy = y + dy;
            const bool ok = in && zz >= 0 && zz < gc.n[2] && yy >= 0 && yy < gc.n[1];
            const int64_t i = ok ? i0 + dz * pw + dy * (int64_t)b.W : 0;
            const uint32_t w = ok ? __ldg(b.core + i) : 0u;
            // lane - 1 holds word (row, q - 1) when q > 0 (consecutive words)
            const uint32_t sl = __shfl_up_sync(0xffffffffu, w, 1);
            const uint32_t sr = __shfl_down_sync(0xffffffffu, w, 1);
            uint32_t wl = 0u, wr = 0u;
            if (ok && q > 0) wl = lane > 0 ? sl : __ldg(b.core + i - 1);
            if (ok && q < b.W - 1) wr = lane < 31 ? sr : __ldg(b.core + i + 1);
            act |= w | (w << 1) | (wl >> 31) | (w >> 1) | (wr << 31);
        }
    }
    return in ? act & valid_bits(gc, q, b.W) : 0u;
}

__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = w;  // inclusive
    }
    __syncthreads();
    total = s_warp[(blockDim.x >> 5) - 1];
    const int before = warp > 0 ? s_warp[warp - 1] : 0;
    return before + x - v;
}

// K2a -- active words of the stored planes + active count per tile of kTB words
__global__ void __launch_bounds__(kTB) k_count(GridC gc, Bits b, int64_t nwords,
                                               uint32_t* __restrict__ act_w,
                                               int32_t* __restrict__ tile_count,
                                               unsigned long long* __restrict__ n_core) {
    __shared__ int s_warp[32];
    const int64_t t = (int64_t)blockIdx.x * kTB + threadIdx.x;
    int cnt = 0, ncore = 0;
    // word t -> (row, q), row -> (y, z): invariant divisors (t < 2^32: the
    // stored planes' words)
    const bool in_t = t < nwords;
    const uint32_t row = b.fdW.div((uint32_t)t), rz = gc.fdy.div(row);
    const int q = (int)((uint32_t)t - row * (uint32_t)b.W);
    const int y = (int)(row - rz * (uint32_t)gc.n[1]);
    const int z = gc.zs_lo + (int)rz;
    const uint32_t act_all = active_word_warp(gc, b, in_t, z, y, q);
    if (in_t) {
        const uint32_t act = act_all;
        act_w[t] = act;
        cnt = __popc(act);
        ncore = __popc(__ldg(b.core + b.idx(gc, z, y, q)) & valid_bits(gc, q, b.W));
        // does an active cell lie on the domain boundary (so that some
        // neighbour-table entries need the out-of-domain rule R-6)?
        const int last = gc.n[0] - 1 - 32 * q;  // bit of x = nx - 1 in this word
        const bool edge = act && (y == 0 || y == gc.n[1] - 1 || z == 0 || z == gc.n[2] - 1 ||
                                  (q == 0 && (act & 1u)) ||
                                  (last < 32 && ((act >> last) & 1u)));
        if (edge) atomicOr(reinterpret_cast<unsigned int*>(n_core + 1), 1u);
    }
    // the tile's totals only (no prefixes needed here): one packed warp
    // reduction (each count <= 32 per thread, <= 8192 per tile: 16 bits)
    const unsigned packed = __reduce_add_sync(0xffffffffu, (unsigned)cnt | ((unsigned)ncore << 16));
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = (int)packed;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned sum = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += (unsigned)s_warp[w];
        tile_count[blockIdx.x] = (int)(sum & 0xffffu);
        const unsigned ctot = sum >> 16;
        if (ctot) atomicAdd(n_core, (unsigned long long)ctot);
    }
}

// K2b -- exclusive scan of tile counts (one block; each thread owns a
// contiguous segment).  out[n] = total.
__global__ void __launch_bounds__(1024) k_scan(const int32_t* __restrict__ cnt, int64_t n,
                                               int64_t* __restrict__ out,
                                               volatile long long* __restrict__ host,
                                               long long gen) {
    // one block: warp w owns a contiguous range of the counts, read 32 at a
    // time (coalesced); pass 1 sums the ranges, warp 0 scans the 32 sums,
    // pass 2 writes the exclusive prefix with warp scans and a running carry
    __shared__ long long s_tot[32], s_base[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t per = ((n + 31) / 32 + 31) & ~(int64_t)31;
    const int64_t b = min(n, (int64_t)w * per), e = min(n, b + per);
    long long sum = 0;
    for (int64_t i = b + lane; i < e; i += 32) sum += cnt[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) s_tot[w] = sum;
    __syncthreads();
    if (w == 0) {
        const long long v = s_tot[lane];
        long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        s_base[lane] = x - v;
    }
    __syncthreads();
    long long run = s_base[w];
    for (int64_t i0 = b; i0 < e; i0 += 32) {
        const int64_t i = i0 + lane;
        const long long v = i < e ? cnt[i] : 0;
        long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (i < e) out[i] = run + x - v;
        run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (threadIdx.x == 0) {
        const long long total = s_base[31] + s_tot[31];
        out[n] = total;
        // publish [active, core, boundary flag] to mapped pinned memory, the
        // generation last: the host polls it instead of a stream sync
        host[0] = total;
        host[1] = out[n + 1];
        host[2] = out[n + 2];
        __threadfence_system();
        host[3] = gen;
    }
}

// K2c -- ordered compaction (R-1): ids 2 + (active cells before) in linear
// cell order; background table (id, or 0/1 by sign) and meta (cell,
// category).  A thread owns one 32-cell word for the scan; the writes are
// done warp-cooperatively word by word (lane = bit), so every background-
// table store is a coalesced 128 B row segment.
__global__ void __launch_bounds__(kTB) k_scatter(GridC gc, Bits b, int64_t nwords,
                                                 const uint32_t* __restrict__ act_w,
                                                 const int64_t* __restrict__ tile_off,
                                                 uint32_t* __restrict__ bg,
                                                 uint32_t* __restrict__ meta_cell,
                                                 uint8_t* __restrict__ meta_cat, uint32_t cap) {
    __shared__ int s_warp[32];
    const int64_t t = (int64_t)blockIdx.x * kTB + threadIdx.x;
    const uint32_t act = t < nwords ? act_w[t] : 0u;
    int total;
    const int ex = block_excl_scan(__popc(act), s_warp, total);
    uint32_t core = 0, neg = 0, id0 = 0;
    int nbits = 0;
    int64_t off = 0, L0 = 0;
    if (t < nwords) {
        const uint32_t row = b.fdW.div((uint32_t)t), rz = gc.fdy.div(row);
        const int q = (int)((uint32_t)t - row * (uint32_t)b.W);
        const int y = (int)(row - rz * (uint32_t)gc.n[1]);
        const int z = gc.zs_lo + (int)rz;
        const int64_t wi = b.idx(gc, z, y, q);
        core = __ldg(b.core + wi);
        neg = __ldg(b.neg + wi);
        nbits = min(32, gc.n[0] - 32 * q);
        L0 = ((int64_t)z * gc.n[1] + y) * gc.n[0] + 32 * q;  // global linear cell
        off = L0 - (int64_t)gc.zs_lo * gc.plane;
        id0 = (uint32_t)(2 + tile_off[blockIdx.x] + ex);
    }
    // write-out: four rounds of 8 words per warp, lane l takes 8 consecutive
    // cells (8 (l & 3) ..) of word 8 round + l / 4 -> 32 B per lane, 1 KB per
    // warp store, two 16 B vector stores when the row start is 16 B aligned
    const int lane = threadIdx.x & 31;
    const int c0 = 8 * (lane & 3);
#pragma unroll
    for (int round = 0; round < 4; ++round) {
        const int src = 8 * round + (lane >> 2);
        const int nb_ = __shfl_sync(0xffffffffu, nbits, src);
        const uint32_t a = __shfl_sync(0xffffffffu, act, src);
        const uint32_t cw = __shfl_sync(0xffffffffu, core, src);
        const uint32_t nw = __shfl_sync(0xffffffffu, neg, src);
        const uint32_t i0 = __shfl_sync(0xffffffffu, id0, src);
        const int64_t o = __shfl_sync(0xffffffffu, off, src);
        const int64_t l0 = __shfl_sync(0xffffffffu, L0, src);
        if (c0 >= nb_) continue;
        uint32_t v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int b = c0 + i;
            const uint32_t m = 1u << b;
            if (a & m) {
                v[i] = i0 + __popc(a & (m - 1u));
                if (b < nb_ && v[i] < cap) {  // cap: the meta arrays' size
                    meta_cell[v[i]] = (uint32_t)(l0 + b);
                    meta_cat[v[i]] = (cw & m) ? 3 : 2;
                }
            } else {
                v[i] = (nw & m) ? 0u : 1u;
            }
        }
        uint32_t* dst = bg + o + c0;
        if (c0 + 8 <= nb_ && ((uintptr_t)dst & 15u) == 0) {
            reinterpret_cast<uint4*>(dst)[0] = make_uint4(v[0], v[1], v[2], v[3]);
            reinterpret_cast<uint4*>(dst)[1] = make_uint4(v[4], v[5], v[6], v[7]);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (c0 + i < nb_) dst[i] = v[i];
        }
    }
}

// first local package id of every stored plane; pf[planes] = n_pkg
__global__ void k_planes_init(int64_t* pf, int32_t planes, int64_t n_pkg, uint32_t* meta_cell,
                              uint8_t* meta_cat) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= planes) pf[i] = n_pkg;
    if (i < 2) {  // singular packages: no cell, category 0 / 1
        meta_cell[i] = 0xFFFFFFFFu;
        meta_cat[i] = (uint8_t)i;
    }
}

__global__ void k_planes(GridC gc, const uint32_t* __restrict__ meta_cell, int64_t n_pkg,
                         int64_t* __restrict__ pf) {
    const int64_t id = 2 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n_pkg) return;
    const int p = (int)(meta_cell[id] / (uint64_t)gc.plane) - gc.zs_lo;
    const int q = id == 2 ? -1 : (int)(meta_cell[id - 1] / (uint64_t)gc.plane) - gc.zs_lo;
    for (int z = q + 1; z <= p; ++z) pf[z] = id;
}

// Sign of f at a (virtual) cell centre outside the domain (R-6); rare, kept
// out of line so the neighbour-table kernel stays small.
__device__ __noinline__ uint32_t virtual_sign(double lx, double ly, double lz, double cell,
                                              const Geom* __restrict__ geom, int qx, int qy,
                                              int qz) {
    const double x = lx + ((double)qx + 0.5) * cell;
    const double y = ly + ((double)qy + 0.5) * cell;
    const double z = lz + ((double)qz + 0.5) * cell;
    return sd_eval(*geom, x, y, z) < 0.0 ? 0u : 1u;
}

// K3 -- neighbour table; a warp fills the rows of 4 packages (lane s < 27 =
// slot s; coalesced 108 B rows), the loads of the 4 packages batched.
// Neighbours outside the domain take the sign of f at the virtual cell centre
// (R-6); cells in the domain but outside the stored planes (beyond a ghost
// plane) take their sign bit (never dereferenced by owned-point stencils).
constexpr int kNbPW = 16;  // packages per warp

template <bool EDGE>
__global__ void __launch_bounds__(256) k_nb(GridC gc, const Geom* __restrict__ geom, Bits b,
                                            const uint32_t* __restrict__ bg,
                                            const uint32_t* __restrict__ meta_cell,
                                            int64_t n_pkg, uint32_t* __restrict__ nb,
                                            uint32_t* __restrict__ face) {
    const int64_t id0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kNbPW;
    const int s = threadIdx.x & 31;
    if (id0 >= n_pkg || s >= 27) return;
    const int ox = s % 3 - 1, oy = (s / 3) % 3 - 1, oz = s / 9 - 1;
    uint32_t L[kNbPW];
#pragma unroll
    for (int u = 0; u < kNbPW; ++u) {
        const int64_t id = id0 + u;
        L[u] = (id >= 2 && id < n_pkg) ? __ldg(meta_cell + id) : 0xFFFFFFFFu;
    }
    uint32_t v[kNbPW];
    const uint32_t nx = (uint32_t)gc.n[0], ny = (uint32_t)gc.n[1];
#pragma unroll
    for (int u = 0; u < kNbPW; ++u) {
        const int64_t id = id0 + u;
        v[u] = (uint32_t)id;  // far-field packages neighbour themselves
        if (id < 2 || id >= n_pkg) continue;
        const uint32_t r = gc.fdx.div(L[u]), rz = gc.fdy.div(r);
        const int qx = (int)(L[u] - r * nx) + ox, qy = (int)(r - rz * ny) + oy, qz = (int)rz + oz;
        if (EDGE &&
            (qx < 0 || qy < 0 || qz < 0 || qx >= gc.n[0] || qy >= gc.n[1] || qz >= gc.n[2])) {
            if (geom->mesh_nt) {  // mesh: sign of the nearest in-domain cell
                const int cx = min(max(qx, 0), gc.n[0] - 1), cy = min(max(qy, 0), gc.n[1] - 1);
                const int cz = min(max(qz, 0), gc.n[2] - 1);
                v[u] = ((__ldg(b.neg + b.idx(gc, cz, cy, cx >> 5)) >> (cx & 31)) & 1u) ? 0u : 1u;
            } else {
                v[u] = virtual_sign(gc.lower[0], gc.lower[1], gc.lower[2], gc.cell, geom, qx, qy,
                                    qz);
            }
        } else if (qz >= gc.zs_lo && qz < gc.zs_hi) {
            v[u] = __ldg(bg + (int64_t)(qz - gc.zs_lo) * gc.plane + (int64_t)qy * gc.n[0] + qx);
        } else {
            v[u] = ((__ldg(b.neg + b.idx(gc, qz, qy, qx >> 5)) >> (qx & 31)) & 1u) ? 0u : 1u;
        }
    }
    // face table entry of this slot: -x, +x, -y, +y, -z, +z (or a zero pad)
    const int fr = s == 12 ? 0 : s == 14 ? 1 : s == 10 ? 2 : s == 16 ? 3 : s == 4 ? 4 : s == 22 ? 5
                 : s < 2 ? 6 + s : -1;
#pragma unroll
    for (int u = 0; u < kNbPW; ++u)
        if (id0 + u < n_pkg) {
            nb[(id0 + u) * 27 + s] = v[u];
            if (fr >= 0) face[(id0 + u) * 8 + fr] = fr < 6 ? v[u] : 0u;
        }
}

// K4 -- initial level set at the 64 data points of every package:
// phi = init_scale * f(lower + (I + 0.5) dx) rounded to T (R-11, R-17);
// singular packages -far / +far in both buffers.  A thread owns one (i, j)
// column of a package (4 points sharing x and y).
// AX = 2: a thread owns the (i, j) column of 4 points along z (x, y shared);
// AX = 1: the (i, k) column along y (x, z shared) -- chosen for geometries
// whose expensive terms are shared along y (a torus about the y axis).
// The union mask of every package (the primitives that can attain the
// minimum somewhere in it; see k_phi_init), one thread per package and the
// primitives in a warp-uniform loop: no divergence between primitive kinds,
// which the per-lane evaluation inside k_phi_init had (C3: ~28 % of its
// instructions).
__global__ void __launch_bounds__(256) k_prim_mask(GridC gc, Geom geom,
                                                   const uint32_t* __restrict__ meta_cell,
                                                   int64_t n_pkg, uint32_t* __restrict__ mask) {
    const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n_pkg) return;
    if (id < 2) {
        mask[id] = 0u;
        return;
    }
    const uint32_t L = __ldg(meta_cell + id);
    const uint32_t nx = (uint32_t)gc.n[0], ny = (uint32_t)gc.n[1];
    const uint32_t r = gc.fdx.div(L), rz = gc.fdy.div(r);
    const int cx = (int)(L - r * nx), cy = (int)(r - rz * ny), cz = (int)rz;
    const double pcx = gc.lower[0] + ((double)cx + 0.5) * gc.cell;
    const double pcy = gc.lower[1] + ((double)cy + 0.5) * gc.cell;
    const double pcz = gc.lower[2] + ((double)cz + 0.5) * gc.cell;
    const double R = 2.598076211353316 * gc.dx;
    const double eps = 1e-9 * (gc.cell + fabs(gc.lower[0]) + fabs(gc.lower[1]) +
                               fabs(gc.lower[2]) + gc.upper[0] + gc.upper[1] + gc.upper[2]);
    double v[SG_MAX_PRIMS];
    double m = INFINITY;
    for (int i = 0; i < geom.n; ++i) {
        v[i] = sd_prim(geom.kind[i], geom.p[i], pcx, pcy, pcz);
        m = fmin(m, v[i]);
    }
    uint32_t k = 0;
    for (int i = 0; i < geom.n; ++i)
        if (v[i] - R <= m + R + eps) k |= 1u << i;
    mask[id] = k;
}

template <class T, int AX>
__global__ void __launch_bounds__(256) k_phi_init(GridC gc, Geom geom,
                                                  const uint32_t* __restrict__ meta_cell,
                                                  int64_t n_pkg, T* __restrict__ phi0,
                                                  T* __restrict__ phi1,
                                                  const uint32_t* __restrict__ pmask) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_pkg * 16) return;
    const int64_t id = t >> 4;
    const int col = (int)(t & 15);  // i + 4 j
    if (id < 2) {
        const T v = (T)(id == 0 ? -gc.far : gc.far);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            phi0[id * 64 + col + 16 * k] = v;
            phi1[id * 64 + col + 16 * k] = v;
        }
        return;
    }
    const uint32_t L = __ldg(meta_cell + id);
    const uint32_t nx = (uint32_t)gc.n[0], ny = (uint32_t)gc.n[1];
    const uint32_t r = gc.fdx.div(L), rz = gc.fdy.div(r);
    const int cx = (int)(L - r * nx), cy = (int)(r - rz * ny), cz = (int)rz;
    // column coordinates: (a, b) = (x, y) along z, or (x, z) along y
    const int64_t ix = 4 * (int64_t)cx + (col & 3);
    const int64_t ib = 4 * (int64_t)(AX == 2 ? cy : cz) + (col >> 2);
    const double x = gc.lower[0] + ((double)ix + 0.5) * gc.dx;
    const double bb = gc.lower[AX == 2 ? 1 : 2] + ((double)ib + 0.5) * gc.dx;
    const int cc = AX == 2 ? cz : cy;
    double w[4], f[4];  // the column's varying coordinate
#pragma unroll
    for (int k = 0; k < 4; ++k)
        w[k] = gc.lower[AX] + ((double)(4 * (int64_t)cc + k) + 0.5) * gc.dx;
    // the package's union mask (k_prim_mask; one primitive needs none)
    const uint32_t mask = geom.n > 1 ? __ldg(pmask + id) : 1u;
    if constexpr (AX == 2) {
        if (geom.n == 1) sd_eval_col<4>(geom, x, bb, w, f);
        else sd_eval_col_mask<4>(geom, mask, x, bb, w, f);
#pragma unroll
        for (int k = 0; k < 4; ++k) phi0[id * 64 + col + 16 * k] = (T)(gc.init_scale * f[k]);
    } else {
        sd_eval_coly_mask<4>(geom, mask, x, bb, w, f);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            phi0[id * 64 + (col & 3) + 4 * j + 16 * (col >> 2)] = (T)(gc.init_scale * f[j]);
    }
}

// per-plane active counts for slab balancing (planes [zc_lo, zc_lo + nplanes))
__global__ void __launch_bounds__(256) k_plane_count(GridC gc, Bits b, int32_t zc_lo,
                                                     int64_t nwords,
                                                     unsigned long long* __restrict__ counts) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nwords) return;
    const int q = (int)(t % b.W);
    const int64_t row = t / b.W;
    const int y = (int)(row % gc.n[1]);
    const int zl = (int)(row / gc.n[1]);
    const int c = __popc(active_word(gc, b, zc_lo + zl, y, q));
    if (c) atomicAdd(&counts[zl], (unsigned long long)c);
}

// ------------------------------------------------------------- helpers ---

static GridC make_gridc(const sg_desc* d) {
    GridC gc{};
    for (int k = 0; k < 3; ++k) {
        gc.lower[k] = d->lower[k];
        gc.n[k] = d->n[k];
        gc.upper[k] = d->lower[k] + (double)d->n[k] * d->cell;
    }
    gc.cell = d->cell;
    gc.dx = d->cell / 4.0;
    gc.init_scale = d->init_scale > 0.0 ? d->init_scale : 1.0;
    gc.far = d->far > 0.0 ? d->far : 4.0 * d->cell * std::max(1.0, gc.init_scale);
    gc.plane = (int64_t)d->n[0] * d->n[1];
    gc.inv_cell = 1.0 / d->cell;
    gc.inv_dx = 1.0 / gc.dx;
    int e = 0;
    gc.dyadic = std::frexp(d->cell, &e) == 0.5 ? 1 : 0;
    gc.idx32 = gc.dyadic && d->dtype == SG_F32;
    for (int k = 0; k < 3; ++k) {
        gc.upperf[k] = (float)gc.upper[k];
        gc.idx32 = gc.idx32 && d->lower[k] == 0.0 && (double)gc.upperf[k] == gc.upper[k] &&
                   d->n[k] < (1 << 20);
    }
    // SG_PROBE_IDX32=0 forces the general fp64 index path (tests compare the
    // two paths bit for bit)
    static const bool idx32_off = [] {
        const char* e = std::getenv("SG_PROBE_IDX32");
        return e && e[0] == '0';
    }();
    if (idx32_off) gc.idx32 = 0;
    gc.inv_cellf = (float)gc.inv_cell;
    gc.inv_dxf = (float)gc.inv_dx;
    gc.fdx = FastDiv((uint32_t)d->n[0]);
    gc.fdy = FastDiv((uint32_t)d->n[1]);
    return gc;
}

static void check_desc(const sg_desc* d, const sg_geometry* g) {
    SG_ARG(d != nullptr && g != nullptr, "sg_build: null desc or geometry");
    SG_ARG(d->pkg == SG_PKG, "sg_build: desc.pkg must be 4");
    SG_ARG(d->n[0] >= 1 && d->n[1] >= 1 && d->n[2] >= 1, "sg_build: n must be >= 1");
    SG_ARG(d->n[1] <= 65535 && d->n[2] <= 65535, "sg_build: n[1], n[2] must be <= 65535");
    SG_ARG((double)d->n[0] * d->n[1] * d->n[2] < 4294967295.0, "sg_build: more than 2^32-1 cells");
    SG_ARG(d->cell > 0.0 && std::isfinite(d->cell), "sg_build: cell must be > 0");
    SG_ARG(d->dtype == SG_F32 || d->dtype == SG_F64, "sg_build: unknown dtype");
    SG_ARG(d->init_scale >= 0.0 && d->far >= 0.0, "sg_build: negative init_scale or far");
    SG_ARG(g->n_prims >= 0 && g->n_prims <= SG_MAX_PRIMS && (g->n_prims == 0 || g->prims),
           "sg_build: need 0..16 primitives");
    if (g->n_tris > 0) {
        SG_ARG(g->n_prims == 0, "sg_build: a mesh geometry takes no primitives");
        SG_ARG(g->verts != nullptr && g->tris != nullptr && g->n_verts >= 3,
               "sg_build: mesh needs vertices and triangles");
        for (int64_t i = 0; i < 3LL * g->n_tris; ++i)
            SG_ARG(g->tris[i] >= 0 && g->tris[i] < g->n_verts, "sg_build: triangle index out of range");
        return;
    }
    int n_union = 0;
    for (int i = 0; i < g->n_prims; ++i) {
        SG_ARG(g->prims[i].kind >= SG_SPHERE && g->prims[i].kind <= SG_LEAK,
               "sg_build: unknown primitive kind");
        if (g->prims[i].kind == SG_LEAK) {
            const double* l = g->prims[i].p;
            SG_ARG(l[3] >= 0.0 && l[4] >= 0.0, "sg_build: leak radius and margin must be >= 0");
        } else {
            ++n_union;
        }
    }
    SG_ARG(n_union >= 1, "sg_build: need at least one non-leak primitive (or a mesh)");
}

// union primitives in their given order; SG_LEAK entries to the post-op list
static Geom make_geom(const sg_geometry* g) {
    Geom ge{};
    for (int i = 0; i < g->n_prims; ++i) {
        if (g->prims[i].kind == SG_LEAK) {
            for (int j = 0; j < 5; ++j) ge.leak[ge.n_leak][j] = g->prims[i].p[j];
            ++ge.n_leak;
        } else {
            ge.kind[ge.n] = g->prims[i].kind;
            for (int j = 0; j < 12; ++j) ge.p[ge.n][j] = g->prims[i].p[j];
            ++ge.n;
        }
    }
    return ge;
}

static void launch_tag(const GridC& gc, const Geom& geom, int32_t zt_lo, int32_t zt_hi,
                       int32_t W, uint32_t* core_w, uint32_t* neg_w, cudaStream_t s) {
    if (zt_hi <= zt_lo) return;
    // the cull pays where the band is a small fraction of the domain
    const int quads = (int)ceil_div(zt_hi - zt_lo, 4);
    // SG_TAG_CULL=0/1 forces the variant (tests); default by domain size
    static const int force = [] {
        const char* e = getenv("SG_TAG_CULL");
        return e ? atoi(e) : -1;
    }();
    // (leak balls flip signs inside a block: the cull's block-uniform sign
    // does not hold there, so leaky geometries always take the plain kernel)
    const bool cull = geom.n_leak == 0 &&
                      (force >= 0 ? force == 1
                                  : (double)gc.n[0] * gc.n[1] * gc.n[2] >= (double)(1 << 25));
    if (cull) {
        dim3 grid((unsigned)W, (unsigned)ceil_div(gc.n[1], 32), (unsigned)ceil_div(quads, 4));
        k_tag_cull<<<grid, 128, 0, s>>>(gc, geom, zt_lo, zt_hi, W, 1, core_w, neg_w);
    } else {
        dim3 grid((unsigned)ceil_div(gc.n[0], 256), (unsigned)gc.n[1], (unsigned)quads);
        k_tag<<<grid, 256, 0, s>>>(gc, geom, zt_lo, zt_hi, W, core_w, neg_w);
    }
    SG_LAUNCHED();
}

// pinned host landing buffer of the build's package-count read-back (one
// per host thread)
// mapped pinned landing buffer of the build's package-count read-back (one
// per host thread): k_scan writes [active, core, boundary, generation]
struct Published {
    volatile long long* host = nullptr;
    long long* dev = nullptr;
    long long gen = 0;
};
static Published& pinned_counts() {
    static thread_local Published p;
    if (!p.host) {
        void* h = nullptr;
        SG_CUDA(cudaHostAlloc(&h, 4 * sizeof(long long), cudaHostAllocMapped));
        std::memset(h, 0, 4 * sizeof(long long));
        void* d = nullptr;
        SG_CUDA(cudaHostGetDevicePointer(&d, h, 0));
        p.host = (volatile long long*)h;
        p.dev = (long long*)d;
    }
    return p;
}

// wait until k_scan has published generation `gen` (spin with pause; after
// 1 s fall back to a stream sync, which also surfaces kernel errors)
static void wait_published(const Published& p, long long gen, cudaStream_t s) {
    auto t0 = std::chrono::steady_clock::now();
    for (uint64_t it = 0; p.host[3] != gen; ++it) {
        if ((it & 1023) == 1023 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::seconds(1)) {
            SG_CUDA(cudaStreamSynchronize(s));
            if (p.host[3] != gen) throw Error(SG_ERR_CUDA, "sg_build: count read-back lost");
            break;
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    std::atomic_thread_fence(std::memory_order_acquire);
}

// library-internal side stream (one per process, non-blocking)
static cudaStream_t side_stream() {
    static cudaStream_t st = nullptr;
    static std::once_flag once;
    std::call_once(once, [] { SG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); });
    return st;
}

static int check_device() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) throw_cuda(e, "cudaGetDevice (no CUDA device?)", __FILE__, __LINE__);
    return dev;
}

}  // namespace sg

using namespace sg;

// ------------------------------------------------------------------- ABI ---

// frees everything a failed build allocated (stream-ordered, errors ignored)
struct BuildGuard {
    sg_grid* g;
    cudaStream_t s;
    std::vector<void*> tmp;
    MeshDev* md = nullptr;
    bool done = false;
    ~BuildGuard() {
        if (done) return;
        for (void* p : tmp) cudaFreeAsync(p, s);
        if (md)
            for (void* p : md->allocs) cudaFreeAsync(p, s);
        if (g) {
            for (auto& a : g->allocs) {
                if (g->has_allocator)
                    g->allocator.free(a.first, a.second, (void*)s, g->allocator.ctx);
                else
                    cudaFreeAsync(a.first, s);
            }
            if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
            if (g->ev_b) cudaEventDestroy(g->ev_b);
            if (g->ev_x) cudaEventDestroy(g->ev_x);
        }
    }
};

static void plane_counts(const sg_desc* desc, const sg_geometry* geom, int32_t z_lo, int32_t z_hi,
                         int64_t* counts, cudaStream_t s);

// Size hints for repeated builds of the same input.  A whole-domain build
// needs its package count on the host to size the arena and the launches
// after the compaction scan -- the one host synchronisation, a pipeline
// bubble of tens of microseconds (the GPU idles while the host wakes up,
// allocates and launches).  When the same (desc, geometry) was built before
// in this process, the counts of that build (package count, core count,
// boundary flag) size everything instead; every kernel still runs, the
// published counts are read once all the build's work is queued, and a
// mismatch (impossible for a deterministic build of the same input, but
// checked) discards the grid and builds again without the hint.  Mesh,
// slab, partitioned and refined builds always synchronise.  SG_BUILD_HINT=0
// disables hints.
struct HintMiss {};
static std::mutex g_hint_mu;
static std::vector<std::pair<uint64_t, std::array<int64_t, 3>>> g_hints;  // small LRU

static uint64_t build_key(const sg_desc* d, const Geom& g) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* p, size_t n) {
        const unsigned char* b = (const unsigned char*)p;
        for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    };
    mix(d->lower, sizeof(d->lower));
    mix(&d->cell, sizeof(d->cell));
    mix(d->n, sizeof(d->n));
    mix(&d->dtype, sizeof(d->dtype));
    mix(&d->far, sizeof(d->far));
    mix(&d->init_scale, sizeof(d->init_scale));
    mix(&g.n, sizeof(g.n));
    mix(&g.n_leak, sizeof(g.n_leak));
    mix(g.kind, sizeof(int32_t) * g.n);
    mix(g.p, sizeof(g.p[0]) * g.n);
    mix(g.leak, sizeof(g.leak[0]) * g.n_leak);
    int dev = 0;
    cudaGetDevice(&dev);
    mix(&dev, sizeof(dev));
    return h;
}
static bool hint_get(uint64_t k, int64_t (&c)[3]) {
    // SG_BUILD_HINT_SKEW=d (tests): every hint is off by d packages, so the
    // mismatch path (rebuild) and the arena bound of k_scatter run
    static const int64_t skew = [] {
        const char* e = std::getenv("SG_BUILD_HINT_SKEW");
        return e ? (int64_t)std::atoll(e) : 0LL;
    }();
    std::lock_guard<std::mutex> lk(g_hint_mu);
    for (auto& e : g_hints)
        if (e.first == k) {
            for (int i = 0; i < 3; ++i) c[i] = e.second[i];
            c[0] = std::max<int64_t>(0, c[0] + skew);
            return true;
        }
    return false;
}
static void hint_put(uint64_t k, const int64_t (&c)[3]) {
    std::lock_guard<std::mutex> lk(g_hint_mu);
    for (auto it = g_hints.begin(); it != g_hints.end(); ++it)
        if (it->first == k) {
            g_hints.erase(it);
            break;
        }
    if (g_hints.size() >= 32) g_hints.erase(g_hints.begin());
    g_hints.push_back({k, {c[0], c[1], c[2]}});
}
static void hint_drop(uint64_t k) {
    std::lock_guard<std::mutex> lk(g_hint_mu);
    for (auto it = g_hints.begin(); it != g_hints.end(); ++it)
        if (it->first == k) {
            g_hints.erase(it);
            return;
        }
}
static bool hints_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SG_BUILD_HINT");
        return !(e && e[0] == '0');
    }();
    return on;
}

static void build_once(const sg_desc* desc, const sg_geometry* geom, const sg_slab* slab,
                       const sg_grid* parent, void* stream, sg_grid** out,
                       const sg_comm* comm, const sg_allocator* allocator, bool allow_hint);

static void build_impl(const sg_desc* desc, const sg_geometry* geom, const sg_slab* slab,
                       const sg_grid* parent, void* stream, sg_grid** out,
                       const sg_comm* comm = nullptr, const sg_allocator* allocator = nullptr) {
    try {
        build_once(desc, geom, slab, parent, stream, out, comm, allocator, hints_enabled());
    } catch (const HintMiss&) {
        build_once(desc, geom, slab, parent, stream, out, comm, allocator, false);
    }
}

static void build_once(const sg_desc* desc, const sg_geometry* geom, const sg_slab* slab,
                       const sg_grid* parent, void* stream, sg_grid** out,
                       const sg_comm* comm, const sg_allocator* allocator, bool allow_hint) {
    {
        SG_ARG(out != nullptr, "sg_build: null out");
        *out = nullptr;
        check_desc(desc, geom);
        const int dev = check_device();
        cudaStream_t s = (cudaStream_t)stream;
        auto g = std::make_unique<sg_grid>();
        if (allocator) {
            SG_ARG(allocator->alloc && allocator->free, "sg_build: allocator needs alloc and free");
            g->has_allocator = true;
            g->allocator = *allocator;
        }
        BuildGuard guard_mem{g.get(), s};
        // partition over a communicator: per-plane counts of a uniform plane
        // range per rank, all-gathered -- the one host synchronisation of a
        // partitioned build; the plan then fixes this rank's package count
        sg_slab comm_slab{};
        int64_t known_npkg = -1;
        if (comm) {
            SG_ARG(slab == nullptr && parent == nullptr, "sg_build: comm excludes slab / parent");
            SG_ARG(geom->n_tris == 0, "sg_build: mesh geometries are single-domain only");
            const int P = comm_size(comm), r = comm_rank(comm), nz = desc->n[2];
            SG_ARG(nz >= P, "sg_build: fewer background planes than ranks");
            g->comm = comm;
            g->rank = r;
            g->nranks = P;
            g->cuts.assign(P + 1, 0);
            if (P > 1) {
                const int maxper = (int)ceil_div(nz, P);
                int64_t* buf = (int64_t*)dalloc(sizeof(int64_t) * maxper * (P + 1), s);
                guard_mem.tmp.push_back(buf);
                const int lo = (int)((int64_t)r * nz / P), hi = (int)((int64_t)(r + 1) * nz / P);
                SG_CUDA(cudaMemsetAsync(buf, 0, sizeof(int64_t) * maxper, s));
                plane_counts(desc, geom, lo, hi, buf, s);
                comm_allgather(comm, buf, buf + maxper, sizeof(int64_t) * maxper, s);
                std::vector<int64_t> all((size_t)P * maxper), counts(nz);
                SG_CUDA(cudaMemcpyAsync(all.data(), buf + maxper, sizeof(int64_t) * all.size(),
                                        cudaMemcpyDeviceToHost, s));
                SG_CUDA(cudaStreamSynchronize(s));
                SG_CUDA(cudaFreeAsync(buf, s));
                guard_mem.tmp.pop_back();
                for (int q = 0; q < P; ++q) {
                    const int ql = (int)((int64_t)q * nz / P), qh = (int)((int64_t)(q + 1) * nz / P);
                    for (int z = ql; z < qh; ++z) counts[z] = all[(size_t)q * maxper + (z - ql)];
                }
                slab_plan(counts.data(), nz, P, r, &g->plan, g->cuts.data());
                comm_slab = sg_slab{g->plan.z_lo, g->plan.z_hi, g->plan.id_base};
                slab = &comm_slab;
                known_npkg = g->plan.n_pkg;
                int lo_prio = 0, hi_prio = 0;
                SG_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
                SG_CUDA(cudaStreamCreateWithPriority(&g->comm_stream, cudaStreamNonBlocking, hi_prio));
                SG_CUDA(cudaEventCreateWithFlags(&g->ev_b, cudaEventDisableTiming));
                SG_CUDA(cudaEventCreateWithFlags(&g->ev_x, cudaEventDisableTiming));
            } else {
                g->cuts[1] = nz;
            }
        }
        g->desc = *desc;
        g->device = dev;
        g->gc = make_gridc(desc);
        g->geom = make_geom(geom);
        g->dtype = desc->dtype;
        g->esz = desc->dtype == SG_F64 ? 8 : 4;
        GridC& gc = g->gc;
        const int nz = desc->n[2];
        if (slab) {
            SG_ARG(slab->z_lo >= 0 && slab->z_lo < slab->z_hi && slab->z_hi <= nz,
                   "sg_build: slab planes outside the domain");
            SG_ARG(slab->id_base >= 2, "sg_build: slab.id_base must be >= 2");
            gc.z_lo = slab->z_lo;
            gc.z_hi = slab->z_hi;
            g->id_base = slab->id_base;
        } else {
            gc.z_lo = 0;
            gc.z_hi = nz;
            g->id_base = 2;
        }
        gc.zs_lo = std::max(0, gc.z_lo - 1);
        gc.zs_hi = std::min(nz, gc.z_hi + 1);
        const int32_t zt_lo = std::max(0, gc.zs_lo - 1), zt_hi = std::min(nz, gc.zs_hi + 1);
        const int64_t ncs = gc.plane * (gc.zs_hi - gc.zs_lo);
        g->ncell_stored = ncs;

        // K1: tag planes = stored planes + one on each side (inner tagging
        // of a stored boundary plane needs the core flags beyond it)
        const int32_t W = (int32_t)ceil_div(gc.n[0], 32);
        const int64_t tag_words = (int64_t)W * gc.n[1] * (zt_hi - zt_lo);
        const int64_t nwords = (int64_t)W * gc.n[1] * (gc.zs_hi - gc.zs_lo);
        const int64_t n_tiles = ceil_div(nwords, kTB);
        // the tag bitmasks stay with the grid (sign correction); one scratch
        // block: active words | tile counts | tile offsets + [core count,
        // boundary flag] (contiguous: one D2H copy)
        auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t sz_tag = al(sizeof(uint32_t) * 2 * tag_words),
                     sz_act = al(sizeof(uint32_t) * nwords), sz_cnt = al(sizeof(int32_t) * n_tiles),
                     sz_off = al(sizeof(int64_t) * (n_tiles + 3));
        uint32_t* core_w = (uint32_t*)g->alloc(sz_tag, s);
        uint32_t* neg_w = core_w + tag_words;
        g->cell_core = core_w;
        g->cell_neg = neg_w;
        g->tag_W = W;
        g->zt_lo = zt_lo;
        g->zt_hi = zt_hi;
        char* scratch = (char*)dalloc(sz_act + sz_cnt + sz_off, s);
        guard_mem.tmp.push_back(scratch);
        uint32_t* act_w = (uint32_t*)scratch;
        int32_t* tile_count = (int32_t*)(scratch + sz_act);
        int64_t* tile_off = (int64_t*)(scratch + sz_act + sz_cnt);
        unsigned long long* d_core = (unsigned long long*)(tile_off + n_tiles + 1);
        SG_CUDA(cudaMemsetAsync(d_core, 0, 2 * sizeof(unsigned long long), s));
        const bool mesh = geom->n_tris > 0;
        MeshDev md;
        guard_mem.md = &md;
        if (parent) {
            const ParentBits pb{parent->cell_core, parent->cell_neg, parent->tag_W};
            // cells evaluated here (under a parent core cell): the sign
            // correction of a refined layer revisits only these
            g->cell_eval = (uint32_t*)g->alloc(sizeof(uint32_t) * tag_words, s);
            if (mesh) {
                md = mesh_prepare(gc, geom, g->geom, s);
                launch_tag_refine_mesh(gc, g->geom, W, pb, core_w, neg_w, g->cell_eval, s);
            } else {
                dim3 grid((unsigned)ceil_div(gc.n[0], 256), (unsigned)gc.n[1], (unsigned)gc.n[2]);
                k_tag_refine<<<grid, 256, 0, s>>>(gc, g->geom, W, pb, core_w, neg_w, g->cell_eval);
                SG_LAUNCHED();
            }
        } else if (mesh) {
            // NEXT-4: exact distances near the surface from per-cell triangle
            // bins; signs of the cells beyond the bin radius by the coarse
            // sign flood, seeded by the cells within it
            SG_ARG(slab == nullptr, "sg_build: mesh geometries need a single-domain grid");
            md = mesh_prepare(gc, geom, g->geom, s);
            uint32_t* known_w = (uint32_t*)dalloc(sizeof(uint32_t) * tag_words, s);
            launch_tag_mesh(gc, g->geom, W, core_w, neg_w, known_w, s);
            cell_flood(gc.n[0], W, gc.n[1], zt_hi - zt_lo, known_w, neg_w, s);
            SG_CUDA(cudaFreeAsync(known_w, s));
        } else {
            launch_tag(gc, g->geom, zt_lo, zt_hi, W, core_w, neg_w, s);
        }
        const Bits bits{core_w, neg_w, W, zt_lo, FastDiv((uint32_t)W)};
        k_count<<<(unsigned)n_tiles, kTB, 0, s>>>(gc, bits, nwords, act_w, tile_count, d_core);
        SG_LAUNCHED();
        Published& pub = pinned_counts();
        const long long gen = ++pub.gen;
        k_scan<<<1, 1024, 0, s>>>(tile_count, n_tiles, tile_off, pub.dev, gen);
        SG_LAUNCHED();

        // the single host synchronisation: package count, core count and the
        // domain-boundary flag in one 24 B copy into pinned memory.  A
        // partitioned build knows its count from the all-gathered plane
        // counts: it enqueues everything first and reads the published
        // values at the end (they are long done by then), taking the
        // boundary-safe neighbour kernel since the flag is not known yet.
        int64_t counts[3] = {known_npkg - 2, 0, 1};
        const bool hintable = allow_hint && known_npkg < 0 && !slab && !parent && !mesh;
        const uint64_t hkey = hintable ? build_key(desc, g->geom) : 0;
        const bool hinted = hintable && hint_get(hkey, counts);
        if (known_npkg < 0 && !hinted) {
            wait_published(pub, gen, s);
            counts[0] = (int64_t)pub.host[0];
            counts[1] = (int64_t)pub.host[1];
            counts[2] = (int64_t)pub.host[2];
            if (hintable) hint_put(hkey, counts);
        }
        const int64_t n_active = counts[0];
        SG_ARG(n_active + 2 < 4294967295LL, "sg_build: more than 2^32-3 packages");
        // the stencil kernels address data points with 32-bit element offsets
        // (a grid this large would not fit its fields in 180 GB anyway)
        SG_ARG((n_active + 2) * 64 < ((int64_t)1 << 32),
               "sg_build: more than 2^32 stored data points on one device");
        g->n_pkg = n_active + 2;
        g->n_core = counts[1];
        g->n_inner = n_active - counts[1];
        const int64_t n_pkg = g->n_pkg;

        // one arena for every array of the grid (a single stream-ordered
        // allocation right after the host sync keeps the device busy)
        const int32_t planes = gc.zs_hi - gc.zs_lo;
        const size_t sz_bg = al(sizeof(uint32_t) * ncs), sz_mc = al(sizeof(uint32_t) * n_pkg),
                     sz_mk = al((size_t)n_pkg), sz_nb = al(sizeof(uint32_t) * 27 * n_pkg),
                     sz_fc = al(sizeof(uint32_t) * 8 * n_pkg),
                     sz_pf = al(sizeof(int64_t) * (planes + 1)),
                     sz_phi = al((size_t)g->esz * 64 * n_pkg);
        char* arena =
            (char*)g->alloc(sz_bg + sz_mc + sz_mk + sz_nb + sz_fc + sz_pf + 2 * sz_phi, s);
        g->bg = (uint32_t*)arena;
        arena += sz_bg;
        g->meta_cell = (uint32_t*)arena;
        arena += sz_mc;
        g->meta_cat = (uint8_t*)arena;
        arena += sz_mk;
        g->nb = (uint32_t*)arena;
        arena += sz_nb;
        g->face = (uint32_t*)arena;
        arena += sz_fc;
        g->plane_first = (int64_t*)arena;
        arena += sz_pf;
        g->phi[0] = arena;
        g->phi[1] = arena + sz_phi;

        k_scatter<<<(unsigned)n_tiles, kTB, 0, s>>>(gc, bits, nwords, act_w, tile_off, g->bg,
                                                    g->meta_cell, g->meta_cat, (uint32_t)n_pkg);
        SG_LAUNCHED();
        k_planes_init<<<(unsigned)ceil_div(planes + 1, 256), 256, 0, s>>>(
            g->plane_first, planes, n_pkg, g->meta_cell, g->meta_cat);
        SG_LAUNCHED();
        if (n_active > 0) {
            k_planes<<<(unsigned)ceil_div(n_active, 256), 256, 0, s>>>(gc, g->meta_cell, n_pkg,
                                                                       g->plane_first);
            SG_LAUNCHED();
        }
        Geom* d_geom = nullptr;
        if (counts[2]) {
            d_geom = (Geom*)dalloc(sizeof(Geom), s);
            guard_mem.tmp.push_back(d_geom);
            SG_CUDA(cudaMemcpyAsync(d_geom, &g->geom, sizeof(Geom), cudaMemcpyHostToDevice, s));
        }
        // K3 (integer / L2 gathers) on a side stream concurrently with K4
        // (fp64 ALU): they only share read-only inputs
        cudaStream_t side = side_stream();
        static thread_local cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
        if (!ev_fork) {
            SG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
            SG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        }
        SG_CUDA(cudaEventRecord(ev_fork, s));
        SG_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
        const unsigned nbb = (unsigned)ceil_div(ceil_div(n_pkg, kNbPW) * 32, 256);
        if (counts[2])  // band touches the domain boundary: out-of-domain rule needed
            k_nb<true><<<nbb, 256, 0, side>>>(gc, d_geom, bits, g->bg, g->meta_cell, n_pkg, g->nb,
                                              g->face);
        else
            k_nb<false><<<nbb, 256, 0, side>>>(gc, d_geom, bits, g->bg, g->meta_cell, n_pkg, g->nb,
                                               g->face);
        SG_LAUNCHED();
        SG_CUDA(cudaEventRecord(ev_join, side));
        const unsigned pb = (unsigned)ceil_div(n_pkg * 16, 256);
        if (mesh) {
            launch_phi_init_mesh(gc, g->geom, g->meta_cell, n_pkg, g->dtype, g->phi[0], g->phi[1], s);
        } else {
            // y-columns when the geometry has a torus about the y axis and
            // nothing whose shared terms need z-columns
            bool ycol = false, zcol = false;
            for (int i = 0; i < g->geom.n; ++i) {
                ycol = ycol || g->geom.kind[i] == SG_TORUS_Y;
                zcol = zcol || g->geom.kind[i] == SG_TORUS_Z || g->geom.kind[i] == SG_TRIPRISM_Z;
            }
            const bool ax1 = ycol && !zcol && std::getenv("SG_PHI_ZCOL_ONLY") == nullptr;
            uint32_t* pmask = nullptr;  // union masks (unions only)
            if (g->geom.n > 1) {
                pmask = (uint32_t*)dalloc(sizeof(uint32_t) * n_pkg, s);
                guard_mem.tmp.push_back(pmask);
                k_prim_mask<<<(unsigned)ceil_div(n_pkg, 256), 256, 0, s>>>(gc, g->geom, g->meta_cell,
                                                                          n_pkg, pmask);
                SG_LAUNCHED();
            }
            if (g->dtype == SG_F64) {
                auto kern = ax1 ? k_phi_init<double, 1> : k_phi_init<double, 2>;
                kern<<<pb, 256, 0, s>>>(gc, g->geom, g->meta_cell, n_pkg, (double*)g->phi[0],
                                        (double*)g->phi[1], pmask);
            } else {
                auto kern = ax1 ? k_phi_init<float, 1> : k_phi_init<float, 2>;
                kern<<<pb, 256, 0, s>>>(gc, g->geom, g->meta_cell, n_pkg, (float*)g->phi[0],
                                        (float*)g->phi[1], pmask);
            }
            SG_LAUNCHED();
            if (pmask) {
                SG_CUDA(cudaFreeAsync(pmask, s));
                guard_mem.tmp.pop_back();
            }
        }
        SG_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
        g->cur = 0;

        if (hinted) {  // everything is queued: the counts are long published
            wait_published(pub, gen, s);
            if ((int64_t)pub.host[0] != counts[0] || (int64_t)pub.host[1] != counts[1] ||
                (int64_t)pub.host[2] != counts[2]) {
                hint_drop(hkey);
                throw HintMiss{};  // the guard frees this attempt's memory
            }
        }
        // owned id range: whole domain -> [2, n_pkg); slab -> plane ranges
        if (known_npkg >= 0) {
            g->own_lo = g->plan.own_lo;
            g->own_hi = g->plan.own_hi;
            wait_published(pub, gen, s);
            if ((int64_t)pub.host[0] != n_active)
                throw Error(SG_ERR_STATE, "sg_build: partition count differs from the build's");
            g->n_core = (int64_t)pub.host[1];
            g->n_inner = n_active - g->n_core;
        } else if (gc.zs_lo == gc.z_lo && gc.zs_hi == gc.z_hi) {
            g->own_lo = 2;
            g->own_hi = n_pkg;
        } else {
            std::vector<int64_t> pf(planes + 1);
            SG_CUDA(cudaMemcpyAsync(pf.data(), g->plane_first, sizeof(int64_t) * (planes + 1),
                                    cudaMemcpyDeviceToHost, s));
            SG_CUDA(cudaStreamSynchronize(s));
            g->own_lo = pf[gc.z_lo - gc.zs_lo];
            g->own_hi = pf[gc.z_hi - gc.zs_lo];
        }

        SG_CUDA(cudaFreeAsync(scratch, s));
        if (d_geom) SG_CUDA(cudaFreeAsync(d_geom, s));
        if (mesh) {
            mesh_release(md, s);
            g->geom.mesh_nt = 0;  // device mesh arrays are gone
        }

        guard_mem.done = true;
        *out = g.release();
    }
}

extern "C" sg_status sg_build(const sg_desc* desc, const sg_geometry* geom, const sg_slab* slab,
                              void* stream, sg_grid** out) {
    return guard([&] {
        NvtxRange nvtx_("sg_build"); build_impl(desc, geom, slab, nullptr, stream, out); });
}

extern "C" sg_status sg_build_ex(const sg_desc* desc, const sg_geometry* geom,
                                 const sg_build_opts* opts, void* stream, sg_grid** out) {
    return guard([&] {
        NvtxRange nvtx_("sg_build_ex");
        const sg_build_opts o = opts ? *opts : sg_build_opts{nullptr, nullptr, nullptr};
        build_impl(desc, geom, o.slab, nullptr, stream, out, o.comm, o.allocator);
    });
}

extern "C" sg_status sg_pool_trim(void) {
    return guard([&] {
        cudaMemPool_t pool = lib_pool();
        SG_CUDA(cudaDeviceSynchronize());
        SG_CUDA(cudaMemPoolTrimTo(pool, 0));
    });
}

extern "C" sg_status sg_build_refined(const sg_grid* parent, const sg_geometry* geom, void* stream,
                                      sg_grid** out) {
    return guard([&] {
        NvtxRange nvtx_("sg_build_refined");
        SG_ARG(parent != nullptr && geom != nullptr, "sg_build_refined: null argument");
        SG_ARG(parent->gc.zs_lo == 0 && parent->gc.zs_hi == parent->gc.n[2] && parent->id_base == 2,
               "sg_build_refined: single-domain parent grids only");
        sg_desc d = parent->desc;
        d.cell = 0.5 * parent->desc.cell;
        for (int k = 0; k < 3; ++k) {
            SG_ARG(parent->desc.n[k] <= (1 << 30), "sg_build_refined: grid too large");
            d.n[k] = 2 * parent->desc.n[k];
        }
        // a default far field scales with the layer's cell size (R-4)
        build_impl(&d, geom, nullptr, parent, stream, out);
    });
}

static void free_grid(sg_grid* g, cudaStream_t s, bool async) {
    tplan_release(g, s);
    for (auto& a : g->allocs) {
        if (g->has_allocator)
            g->allocator.free(a.first, a.second, (void*)s, g->allocator.ctx);
        else if (async)
            cudaFreeAsync(a.first, s);
        else
            cudaFree(a.first);
    }
    g->allocs.clear();
    if (g->comm_stream) {
        if (async) {
            // the comm stream's last exchange must finish before the memory
            // it touches is reused on s
            cudaEventRecord(g->ev_x, g->comm_stream);
            cudaStreamWaitEvent(s, g->ev_x, 0);
        }
        cudaStreamDestroy(g->comm_stream);
    }
    if (g->ev_b) cudaEventDestroy(g->ev_b);
    if (g->ev_x) cudaEventDestroy(g->ev_x);
    delete g;
}

extern "C" void sg_destroy(sg_grid* grid) {
    if (!grid) return;
    cudaDeviceSynchronize();
    free_grid(grid, 0, false);
}

extern "C" sg_status sg_destroy_async(sg_grid* grid, void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_destroy_async");
        if (!grid) return;
        free_grid(grid, (cudaStream_t)stream, true);
        SG_CUDA(cudaGetLastError());
    });
}

extern "C" sg_status sg_info(const sg_grid* g, sg_info_t* info) {
    return guard([&] {
        SG_ARG(g && info, "sg_info: null argument");
        std::memset(info, 0, sizeof(*info));
        info->n_pkg = g->n_pkg;
        info->n_core = g->n_core;
        info->n_inner = g->n_inner;
        info->id_base = g->id_base;
        info->dtype = g->dtype;
        info->z_lo = g->gc.z_lo;
        info->z_hi = g->gc.z_hi;
        info->zs_lo = g->gc.zs_lo;
        info->zs_hi = g->gc.zs_hi;
        info->dx = g->gc.dx;
        info->far = g->gc.far;
        info->kernel_sum = g->kernel_sum;
        info->has_grad = g->has_grad;
        info->has_normal = g->has_normal;
        info->has_kint = g->has_kint;
        info->phi_cur = g->cur;
        info->device_bytes = g->bytes();
        info->own_lo = g->own_lo;
        info->own_hi = g->own_hi;
        info->rank = g->rank;
        info->nranks = g->nranks;
    });
}

extern "C" sg_status sg_view(const sg_grid* g, int32_t what, sg_view_t* v) {
    return guard([&] {
        SG_ARG(g && v, "sg_view: null argument");
        std::memset(v, 0, sizeof(*v));
        v->shape[0] = v->shape[1] = v->shape[2] = 1;
        const int fdt = g->dtype == SG_F64 ? 1 : 0;
        auto set = [&](void* p, int ndim, int64_t a, int64_t b, int64_t c, int es, int dt) {
            v->ptr = p;
            v->ndim = ndim;
            v->shape[0] = a;
            v->shape[1] = b;
            v->shape[2] = c;
            v->elem_size = es;
            v->dtype = dt;
        };
        switch (what) {
        case SG_VIEW_BG: set(g->bg, 1, g->ncell_stored, 1, 1, 4, 2); break;
        case SG_VIEW_META_CELL: set(g->meta_cell, 1, g->n_pkg, 1, 1, 4, 2); break;
        case SG_VIEW_META_CAT: set(g->meta_cat, 1, g->n_pkg, 1, 1, 1, 3); break;
        case SG_VIEW_NB: set(g->nb, 2, g->n_pkg, 27, 1, 4, 2); break;
        case SG_VIEW_FACE: set(g->face, 2, g->n_pkg, 8, 1, 4, 2); break;
        case SG_VIEW_PHI: set(g->phi[g->cur], 2, g->n_pkg, 64, 1, g->esz, fdt); break;
        case SG_VIEW_PHI_NEXT: set(g->phi[1 - g->cur], 2, g->n_pkg, 64, 1, g->esz, fdt); break;
        case SG_VIEW_GRAD: set(g->has_grad ? g->grad : nullptr, 3, g->n_pkg, 64, 4, g->esz, fdt); break;
        case SG_VIEW_NORMAL:
            set(g->has_normal ? g->normal : nullptr, 3, g->n_pkg, 3, 64, g->esz, fdt);
            break;
        case SG_VIEW_KINT: set(g->has_kint ? g->kint : nullptr, 2, g->n_pkg, 64, 1, g->esz, fdt); break;
        case SG_VIEW_GKINT:
            set(g->has_kint ? g->gkint : nullptr, 3, g->n_pkg, 3, 64, g->esz, fdt);
            break;
        case SG_VIEW_PLANE_FIRST:
            set(g->plane_first, 1, g->gc.zs_hi - g->gc.zs_lo + 1, 1, 1, 8, 4);
            break;
        case SG_VIEW_CELL_CORE:
            set(g->cell_core, 3, g->zt_hi - g->zt_lo, g->gc.n[1], g->tag_W, 4, 2);
            break;
        case SG_VIEW_CELL_NEG:
            set(g->cell_neg, 3, g->zt_hi - g->zt_lo, g->gc.n[1], g->tag_W, 4, 2);
            break;
        default: throw Error(SG_ERR_ARG, "sg_view: unknown selector");
        }
    });
}

extern "C" sg_status sg_balanced_cuts(const int64_t* counts, int32_t nz, int32_t nranks,
                                      int32_t* cuts) {
    return guard([&] {
        SG_ARG(counts && cuts, "sg_balanced_cuts: null argument");
        SG_ARG(nranks >= 1 && nz >= nranks, "sg_balanced_cuts: need 1 <= nranks <= nz");
        std::vector<int64_t> pre(nz + 1, 0);
        for (int z = 0; z < nz; ++z) pre[z + 1] = pre[z] + counts[z];
        const int64_t total = pre[nz];
        cuts[0] = 0;
        cuts[nranks] = nz;
        for (int r = 1; r < nranks; ++r) {
            // smallest z with prefix(z) >= r * total / nranks (exact integer
            // comparison: prefix * nranks >= r * total)
            int z = 0;
            while (z < nz && pre[z] * nranks < (int64_t)r * total) ++z;
            // every slab keeps at least one plane
            z = std::max(z, cuts[r - 1] + 1);
            z = std::min(z, nz - (nranks - r));
            cuts[r] = z;
        }
    });
}

static void plane_counts(const sg_desc* desc, const sg_geometry* geom, int32_t z_lo, int32_t z_hi,
                         int64_t* counts, cudaStream_t s) {
    {
        if (z_hi == z_lo) return;
        GridC gc = make_gridc(desc);
        const Geom ge = make_geom(geom);
        const int32_t zt_lo = std::max(0, z_lo - 1), zt_hi = std::min(desc->n[2], z_hi + 1);
        const int32_t W = (int32_t)ceil_div(gc.n[0], 32);
        const int64_t tag_words = (int64_t)W * gc.n[1] * (zt_hi - zt_lo);
        uint32_t* core_w = (uint32_t*)dalloc(sizeof(uint32_t) * 2 * tag_words, s);
        launch_tag(gc, ge, zt_lo, zt_hi, W, core_w, core_w + tag_words, s);
        const Bits bits{core_w, core_w + tag_words, W, zt_lo, FastDiv((uint32_t)W)};
        SG_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (z_hi - z_lo), s));
        const int64_t nwords = (int64_t)W * gc.n[1] * (z_hi - z_lo);
        k_plane_count<<<(unsigned)ceil_div(nwords, 256), 256, 0, s>>>(gc, bits, z_lo, nwords,
                                                                      (unsigned long long*)counts);
        SG_LAUNCHED();
        SG_CUDA(cudaFreeAsync(core_w, s));
    }
}

extern "C" sg_status sg_plane_counts(const sg_desc* desc, const sg_geometry* geom, int32_t z_lo,
                                     int32_t z_hi, int64_t* counts, void* stream) {
    return guard([&] {
        NvtxRange nvtx_("sg_plane_counts");
        check_desc(desc, geom);
        SG_ARG(geom->n_tris == 0, "sg_plane_counts: mesh geometries are single-domain only");
        SG_ARG(counts != nullptr, "sg_plane_counts: null counts");
        SG_ARG(z_lo >= 0 && z_lo <= z_hi && z_hi <= desc->n[2], "sg_plane_counts: bad plane range");
        check_device();
        plane_counts(desc, geom, z_lo, z_hi, counts, (cudaStream_t)stream);
    });
}

extern "C" const char* sg_last_error(void) { return t_last_error.c_str(); }
extern "C" int32_t sg_abi_version(void) { return SG_ABI_VERSION; }

extern "C" int32_t sg_neighbour_index_shift(const int32_t* shift, int32_t* offset, int32_t* data) {
    if (!shift) return -1;
    int32_t slot = 0, mul = 1;
    for (int k = 0; k < 3; ++k) {
        if (shift[k] < -SG_PKG || shift[k] > 2 * SG_PKG - 1) return -1;
        const Shift h = nb_shift(shift[k]);
        if (offset) offset[k] = h.off;
        if (data) data[k] = h.data;
        slot += mul * h.off;
        mul *= 3;
    }
    return slot;
}
extern "C" uint64_t sg_launch_count(void) { return g_launches.load(); }
