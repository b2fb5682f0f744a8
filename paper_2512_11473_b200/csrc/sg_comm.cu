// sg_comm.cu -- communicators of the z-slab partition (BASELINE
// north_star: "Packages are partitioned across the 8xB200 box in z-slabs of
// the background grid, with NCCL halo exchange of boundary packages over
// NVLink each reinitialization iteration and particles binned to their owning
// rank").  The paper itself runs on one device.
//
// Two backends behind one internal interface (all-gather, grouped
// point-to-point), both stream-ordered:
//   * NCCL, loaded at run time (dlopen "libnccl.so.2": the copy PyTorch
//     already loaded is reused; no link-time dependency), one process per
//     GPU -- the production path over NVLink / NVSwitch;
//   * an in-process group ("local"): nranks communicators on one device,
//     driven by one host thread each, exchanging by device-to-device copies
//     with the same matching rules (the k-th send from a to b meets the k-th
//     receive of b from a; a group posts all its sends before it blocks on
//     a receive).  It runs every multi-GPU path of the library on one GPU, so
//     the 1-vs-P bitwise tests exercise the real schedule.
// Also here: the slab plan (cuts, id base, owned and halo ranges) and the
// ghost-plane exchange of a partitioned grid.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "sg_internal.cuh"

namespace sg {

// ------------------------------------------------------------- NCCL ------

struct Nccl {
    void* h = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGetErrorString) getErrorString = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclCommGetAsyncError) getAsyncError = nullptr;
    std::string err;
};

static Nccl& nccl() {
    static Nccl N;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            N.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (N.h) break;
        }
        if (!N.h) {
            const char* e = dlerror();
            N.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        bool ok = true;
        auto sym = [&](auto& f, const char* n) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(N.h, n));
            if (!f) {
                ok = false;
                N.err += std::string(" missing ") + n;
            }
        };
        sym(N.getUniqueId, "ncclGetUniqueId");
        sym(N.commInitRank, "ncclCommInitRank");
        sym(N.commDestroy, "ncclCommDestroy");
        sym(N.getErrorString, "ncclGetErrorString");
        sym(N.allGather, "ncclAllGather");
        sym(N.send, "ncclSend");
        sym(N.recv, "ncclRecv");
        sym(N.groupStart, "ncclGroupStart");
        sym(N.groupEnd, "ncclGroupEnd");
        sym(N.getAsyncError, "ncclCommGetAsyncError");
        if (!ok) {
            dlclose(N.h);
            N.h = nullptr;
        }
    });
    if (!N.h) throw Error(SG_ERR_NCCL, N.err);
    return N;
}

#define SG_NCCL(x)                                                                      \
    do {                                                                                \
        ncclResult_t r_ = (x);                                                          \
        if (r_ != ncclSuccess)                                                          \
            throw ::sg::Error(SG_ERR_NCCL, std::string(#x) + ": " + nccl().getErrorString(r_)); \
    } while (0)

// ------------------------------------------------------- local group -----

struct LocalGroup {
    int n = 0;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    // all-gather rendezvous per call sequence number
    struct AG {
        std::vector<const void*> src;
        std::vector<cudaEvent_t> ready, done;
        int posted = 0, copied = 0, left = 0;
    };
    std::map<uint64_t, AG> ag;
    std::vector<uint64_t> ag_seq;  // per rank
    // point-to-point mailboxes keyed (src, dst, k-th message)
    struct Post {
        const void* src = nullptr;
        size_t bytes = 0;
        cudaEvent_t ready = nullptr, done = nullptr;
        bool matched = false;
    };
    std::map<std::tuple<int, int, uint64_t>, Post> mail;
    std::vector<uint64_t> send_seq, recv_seq;  // [src * n + dst]
};

}  // namespace sg

struct sg_comm {
    int kind = SG_COMM_NCCL;
    int rank = 0, nranks = 1, device = 0;
    ncclComm_t nc = nullptr;
    std::shared_ptr<sg::LocalGroup> grp;
};

namespace sg {

int comm_rank(const sg_comm* c) { return c ? c->rank : 0; }
int comm_size(const sg_comm* c) { return c ? c->nranks : 1; }
int comm_kind(const sg_comm* c) { return c ? c->kind : SG_COMM_LOCAL; }

// SG_COMM_TRACE=1: one stderr line per collective step (debugging hangs)
static bool trace() {
    static const bool t = [] {
        const char* e = std::getenv("SG_COMM_TRACE");
        return e && e[0] == '1';
    }();
    return t;
}

static cudaEvent_t new_event() {
    cudaEvent_t e;
    SG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
}

void comm_allgather(const sg_comm* c, const void* src, void* dst, size_t bytes, cudaStream_t s) {
    if (c->nranks == 1) {
        if (bytes) SG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (c->kind == SG_COMM_NCCL) {
        SG_NCCL(nccl().allGather(src, dst, bytes, ncclUint8, c->nc, s));
        return;
    }
    LocalGroup& G = *c->grp;
    const int me = c->rank, n = G.n;
    std::unique_lock<std::mutex> lk(G.mu);
    const uint64_t seq = G.ag_seq[me]++;
    if (trace()) fprintf(stderr, "[sg comm] rank %d allgather #%llu %zu B\n", me, (unsigned long long)seq, bytes);
    LocalGroup::AG& a = G.ag[seq];
    if (a.src.empty()) {
        a.src.assign(n, nullptr);
        a.ready.assign(n, nullptr);
        a.done.assign(n, nullptr);
    }
    a.src[me] = src;
    a.ready[me] = new_event();
    SG_CUDA(cudaEventRecord(a.ready[me], s));
    ++a.posted;
    G.cv.notify_all();
    G.cv.wait(lk, [&] { return a.posted == n; });
    for (int r = 0; r < n; ++r) {
        SG_CUDA(cudaStreamWaitEvent(s, a.ready[r], 0));
        if (bytes)
            SG_CUDA(cudaMemcpyAsync((char*)dst + (size_t)r * bytes, a.src[r], bytes,
                                    cudaMemcpyDeviceToDevice, s));
    }
    a.done[me] = new_event();
    SG_CUDA(cudaEventRecord(a.done[me], s));
    ++a.copied;
    G.cv.notify_all();
    // the sources stay untouched until every rank has copied them
    G.cv.wait(lk, [&] { return a.copied == n; });
    for (int r = 0; r < n; ++r) SG_CUDA(cudaStreamWaitEvent(s, a.done[r], 0));
    if (++a.left == n) {
        for (int r = 0; r < n; ++r) {
            cudaEventDestroy(a.ready[r]);
            cudaEventDestroy(a.done[r]);
        }
        G.ag.erase(seq);
    }
}

void comm_group(const sg_comm* c, const P2P* ops, int nops, cudaStream_t s) {
    if (nops == 0) return;
    for (int i = 0; i < nops; ++i)
        SG_ARG(ops[i].peer >= 0 && ops[i].peer < c->nranks && ops[i].peer != c->rank && ops[i].bytes,
               "comm_group: bad peer or empty transfer");
    if (c->kind == SG_COMM_NCCL) {
        Nccl& N = nccl();
        SG_NCCL(N.groupStart());
        for (int i = 0; i < nops; ++i) {
            const P2P& o = ops[i];
            if (o.send)
                SG_NCCL(N.send(o.buf, o.bytes, ncclUint8, o.peer, c->nc, s));
            else
                SG_NCCL(N.recv(o.buf, o.bytes, ncclUint8, o.peer, c->nc, s));
        }
        SG_NCCL(N.groupEnd());
        return;
    }
    LocalGroup& G = *c->grp;
    const int me = c->rank, n = G.n;
    std::unique_lock<std::mutex> lk(G.mu);
    std::vector<std::tuple<int, int, uint64_t>> mine;
    if (trace())
        for (int i = 0; i < nops; ++i)
            fprintf(stderr, "[sg comm] rank %d %s peer %d %zu B seq %llu\n", me,
                    ops[i].send ? "send" : "recv", ops[i].peer, ops[i].bytes,
                    (unsigned long long)(ops[i].send ? G.send_seq[me * n + ops[i].peer]
                                                     : G.recv_seq[ops[i].peer * n + me]));
    // 1. post every send (the data is ready when the stream reaches here)
    for (int i = 0; i < nops; ++i) {
        if (!ops[i].send) continue;
        const auto key = std::make_tuple(me, ops[i].peer, G.send_seq[me * n + ops[i].peer]++);
        LocalGroup::Post& p = G.mail[key];
        p.src = ops[i].buf;
        p.bytes = ops[i].bytes;
        p.ready = new_event();
        SG_CUDA(cudaEventRecord(p.ready, s));
        mine.push_back(key);
    }
    G.cv.notify_all();
    // 2. receives: wait for the matching send, copy after its ready event
    for (int i = 0; i < nops; ++i) {
        if (ops[i].send) continue;
        const auto key = std::make_tuple(ops[i].peer, me, G.recv_seq[ops[i].peer * n + me]++);
        G.cv.wait(lk, [&] { return G.mail.count(key) && G.mail[key].ready != nullptr; });
        LocalGroup::Post& p = G.mail[key];
        if (p.bytes != ops[i].bytes)
            throw Error(SG_ERR_NCCL, "local comm: send / receive sizes differ");
        SG_CUDA(cudaStreamWaitEvent(s, p.ready, 0));
        SG_CUDA(cudaMemcpyAsync(ops[i].buf, p.src, p.bytes, cudaMemcpyDeviceToDevice, s));
        p.done = new_event();
        SG_CUDA(cudaEventRecord(p.done, s));
        p.matched = true;
        G.cv.notify_all();
    }
    // 3. a send completes when its receiver's copy has (buffer reusable)
    for (const auto& key : mine) {
        G.cv.wait(lk, [&] { return G.mail[key].matched; });
        LocalGroup::Post& p = G.mail[key];
        SG_CUDA(cudaStreamWaitEvent(s, p.done, 0));
        cudaEventDestroy(p.ready);
        cudaEventDestroy(p.done);
        G.mail.erase(key);
    }
}

// ------------------------------------------------------------ the plan ---

void slab_plan(const int64_t* counts, int32_t nz, int32_t nranks, int32_t rank, sg_plan_t* p,
               int32_t* cuts_out) {
    SG_ARG(counts && p, "sg_slab_plan: null argument");
    SG_ARG(nranks >= 1 && nranks <= SG_MAX_RANKS && nz >= nranks,
           "sg_slab_plan: need 1 <= nranks <= min(nz, SG_MAX_RANKS)");
    SG_ARG(rank >= 0 && rank < nranks, "sg_slab_plan: rank outside [0, nranks)");
    std::vector<int32_t> cuts(nranks + 1);
    if (sg_balanced_cuts(counts, nz, nranks, cuts.data()) != SG_OK)
        throw Error(SG_ERR_ARG, sg_last_error());
    std::vector<int64_t> pre(nz + 1, 0);
    for (int z = 0; z < nz; ++z) {
        SG_ARG(counts[z] >= 0, "sg_slab_plan: negative count");
        pre[z + 1] = pre[z] + counts[z];
    }
    std::memset(p, 0, sizeof(*p));
    p->z_lo = cuts[rank];
    p->z_hi = cuts[rank + 1];
    p->zs_lo = std::max(0, p->z_lo - 1);
    p->zs_hi = std::min(nz, p->z_hi + 1);
    p->id_base = 2 + pre[p->zs_lo];
    p->n_pkg = 2 + pre[p->zs_hi] - pre[p->zs_lo];
    // local id of the first package of plane z (stored planes only)
    auto first = [&](int z) { return 2 + pre[z] - pre[p->zs_lo]; };
    p->own_lo = first(p->z_lo);
    p->own_hi = first(p->z_hi);
    if (rank > 0) {
        p->send_lo[0] = first(p->z_lo);
        p->send_lo[1] = first(p->z_lo + 1);
        p->recv_lo[0] = first(p->z_lo - 1);
        p->recv_lo[1] = first(p->z_lo);
    }
    if (rank < nranks - 1) {
        p->send_hi[0] = first(p->z_hi - 1);
        p->send_hi[1] = first(p->z_hi);
        p->recv_hi[0] = first(p->z_hi);
        p->recv_hi[1] = first(p->z_hi + 1);
    }
    if (cuts_out) std::copy(cuts.begin(), cuts.end(), cuts_out);
}

// ghost planes of a partitioned grid: the first owned plane goes to rank - 1
// (its ghost-above plane), the last one to rank + 1; whole background planes
// are contiguous local id ranges, so the buffers are sent in place
void halo_exchange(const sg_grid* g, void* field, size_t per_pkg, cudaStream_t s) {
    if (!g->partitioned()) return;
    const sg_plan_t& p = g->plan;
    char* f = (char*)field;
    P2P ops[4];
    int n = 0;
    auto add = [&](int peer, bool send, const int64_t* r) {
        const size_t b = (size_t)(r[1] - r[0]) * per_pkg;
        if (b) ops[n++] = P2P{peer, send, f + (size_t)r[0] * per_pkg, b};
    };
    if (g->rank > 0) {
        add(g->rank - 1, true, p.send_lo);
        add(g->rank - 1, false, p.recv_lo);
    }
    if (g->rank < g->nranks - 1) {
        add(g->rank + 1, true, p.send_hi);
        add(g->rank + 1, false, p.recv_hi);
    }
    comm_group(g->comm, ops, n, s);
}

}  // namespace sg

using namespace sg;

extern "C" sg_status sg_comm_unique_id(void* id) {
    return guard([&] {
        SG_ARG(id != nullptr, "sg_comm_unique_id: null id");
        static_assert(sizeof(ncclUniqueId) == SG_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        SG_NCCL(nccl().getUniqueId(&u));
        std::memcpy(id, &u, sizeof(u));
    });
}

extern "C" sg_status sg_comm_create(const void* id, int32_t rank, int32_t nranks, sg_comm** out) {
    return guard([&] {
        NvtxRange nvtx_("sg_comm_create");
        SG_ARG(id && out, "sg_comm_create: null argument");
        *out = nullptr;
        SG_ARG(nranks >= 1 && nranks <= SG_MAX_RANKS && rank >= 0 && rank < nranks,
               "sg_comm_create: need 0 <= rank < nranks <= SG_MAX_RANKS");
        auto c = std::make_unique<sg_comm>();
        c->kind = SG_COMM_NCCL;
        c->rank = rank;
        c->nranks = nranks;
        SG_CUDA(cudaGetDevice(&c->device));
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        SG_NCCL(nccl().commInitRank(&c->nc, nranks, u, rank));
        *out = c.release();
    });
}

extern "C" sg_status sg_comm_create_local(int32_t nranks, sg_comm** comms) {
    return guard([&] {
        NvtxRange nvtx_("sg_comm_create_local");
        SG_ARG(comms != nullptr, "sg_comm_create_local: null comms");
        SG_ARG(nranks >= 1 && nranks <= SG_MAX_RANKS, "sg_comm_create_local: bad nranks");
        auto grp = std::make_shared<LocalGroup>();
        grp->n = nranks;
        SG_CUDA(cudaGetDevice(&grp->device));
        grp->ag_seq.assign(nranks, 0);
        grp->send_seq.assign((size_t)nranks * nranks, 0);
        grp->recv_seq.assign((size_t)nranks * nranks, 0);
        for (int r = 0; r < nranks; ++r) {
            sg_comm* c = new sg_comm;
            c->kind = SG_COMM_LOCAL;
            c->rank = r;
            c->nranks = nranks;
            c->device = grp->device;
            c->grp = grp;
            comms[r] = c;
        }
    });
}

extern "C" sg_status sg_comm_info(const sg_comm* c, int32_t* rank, int32_t* nranks, int32_t* kind) {
    return guard([&] {
        SG_ARG(c != nullptr, "sg_comm_info: null comm");
        if (rank) *rank = c->rank;
        if (nranks) *nranks = c->nranks;
        if (kind) *kind = c->kind;
    });
}

extern "C" sg_status sg_comm_check(const sg_comm* c) {
    return guard([&] {
        SG_ARG(c != nullptr, "sg_comm_check: null comm");
        if (c->kind != SG_COMM_NCCL || !c->nc) return;
        ncclResult_t r = ncclSuccess;
        SG_NCCL(nccl().getAsyncError(c->nc, &r));
        if (r != ncclSuccess && r != ncclInProgress)
            throw Error(SG_ERR_NCCL, std::string("NCCL async error: ") + nccl().getErrorString(r));
    });
}

extern "C" void sg_comm_destroy(sg_comm* c) {
    if (!c) return;
    if (c->kind == SG_COMM_NCCL && c->nc) {
        try {
            nccl().commDestroy(c->nc);
        } catch (...) {
        }
    }
    delete c;
}

extern "C" sg_status sg_slab_plan(const int64_t* counts, int32_t nz, int32_t nranks, int32_t rank,
                                  sg_plan_t* plan, int32_t* cuts) {
    return guard([&] { slab_plan(counts, nz, nranks, rank, plan, cuts); });
}
