// exchange.cu -- ghost-multipole exchange between ranks.
//
// Paper analogue: octree nodes are distributed along a space-filling curve
// and each node's kernels need "all sub-grids of all neighboring
// nodes as a halo", delivered by HPX channels/parcels
// (P:L632-660).  Here one process drives one GPU; per level, each rank sends
// to each peer only the cells of its owned nodes that lie inside the staging
// window of a node owned by that peer (the parent-aligned halo of width
// 2 * parent_reach cells), as prepared records (mass; + X, Q2, Q3 for refined
// nodes), with one NCCL group of send/recv pairs over NVLink.
#include "internal.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <dlfcn.h>
#include <map>

#include <nccl.h>
#include <string>

using namespace octo;

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            if (e_ == cudaErrorMemoryAllocation) return fail(h, OCTO_ENOMEM, #call);           \
            return fail(h, OCTO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
        }                                                                                      \
    } while (0)
#define NC_(call)                                                                              \
    do {                                                                                       \
        ncclResult_t r_ = (call);                                                              \
        if (r_ != ncclSuccess) return fail(h, OCTO_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

int octo::parent_reach(double theta)
{
    const double r = 1.0 / theta;
    const double R2 = r * r;
    int pm = 0;
    for (int p = 0; p <= 8; p++)
        if ((double)(p * p) < R2) pm = p;
    return pm;
}

extern "C" int octo_fmm_nccl_unique_id(uint8_t *out128)
{
    if (!out128) return OCTO_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return OCTO_ENCCL;
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
    return OCTO_OK;
}

int octo::exchange_init(octo_fmm *h)
{
    if (h->cfg.flags & OCTO_EXTERNAL_BOOTSTRAP) {   // no NCCL: the caller's allgather bootstraps the puts
        if (!h->xput) return fail(h, OCTO_EINVAL, "OCTO_EXTERNAL_BOOTSTRAP needs the one-sided transport (OCTO_XCHG=nccl set)");
        return OCTO_OK;
    }
    ncclUniqueId id;
    std::memcpy(&id, h->cfg.nccl_unique_id, sizeof(id));
    ncclComm_t comm;
    NC_(ncclCommInitRank(&comm, h->cfg.nranks, id, h->cfg.rank));
    h->nccl_comm = comm;
    return OCTO_OK;
}

void octo::exchange_destroy(octo_fmm *h)
{
    exchange_destroy_plan(h);
    if (h->nccl_comm) ncclCommDestroy((ncclComm_t)h->nccl_comm);
    h->nccl_comm = nullptr;
}

void octo::exchange_free_level(Level &lv)
{
    for (auto &p : lv.peers) {
        void *ptrs[] = {p.d_send_leaf, p.d_send_ref, p.d_recv_leaf, p.d_recv_ref};
        for (void *x : ptrs)
            if (x) cudaFree(x);
    }
    lv.peers.clear();
}

// ---------------------------------------------------------------------------
// host plan: which cells go from each rank to each peer (host logic only)
// ---------------------------------------------------------------------------
// Cells of node B needed by a node A at offset o = ijk_A - ijk_B: along each
// axis, o = +1 -> B cells [8-w, 8), o = -1 -> [0, w), o = 0 -> [0, 8), with w =
// 2 * parent_reach (the staging window of A, kernels.cuh).
static void mark_box(uint8_t *mask, int ox, int oy, int oz, int w)
{
    int lo[3], hi[3];
    const int o[3] = {ox, oy, oz};
    for (int a = 0; a < 3; a++) {
        lo[a] = o[a] > 0 ? 8 - w : 0;
        hi[a] = o[a] < 0 ? w : 8;
    }
    for (int z = lo[2]; z < hi[2]; z++)
        for (int y = lo[1]; y < hi[1]; y++)
            for (int x = lo[0]; x < hi[0]; x++) mask[x + 8 * y + 64 * z] = 1;
}

static uint64_t morton(int32_t i, int32_t j, int32_t k)
{
    auto spread = [](uint64_t v) {
        v &= 0x1FFFFF;
        v = (v | (v << 32)) & 0x1F00000000FFFFull;
        v = (v | (v << 16)) & 0x1F0000FF0000FFull;
        v = (v | (v << 8)) & 0x100F00F00F00F00Full;
        v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
        v = (v | (v << 2)) & 0x1249249249249249ull;
        return v;
    };
    return spread(i) | (spread(j) << 1) | (spread(k) << 2);
}

// Exported for the CPU tests (no CUDA needed): the per-peer send and receive
// cell lists of `rank` for one level.  Lists are (node index in this rank's
// list) * 512 + cell, ordered canonically (Morton order of the node, then
// cell index) so sender and receiver agree without communication.
// out arrays may be NULL to query sizes; counts[peer*4 + {0..3}] =
// {send_leaf, send_ref, recv_leaf, recv_ref}.
extern "C" int octo_fmm_exchange_plan(double theta, int32_t rank, int32_t nranks, int64_t n, const int32_t *ijk,
                                      const uint8_t *refined, const int32_t *nb, const int32_t *owner,
                                      int64_t *counts, int32_t **lists /* [nranks*4] or NULL */)
{
    if (!ijk || !refined || !nb || !owner || !counts || nranks < 1) return OCTO_EINVAL;
    const int w = 2 * octo::parent_reach(theta);
    std::vector<std::vector<int32_t>> L(4 * (size_t)nranks);
    // order nodes by Morton key of ijk
    std::vector<int64_t> order(n);
    for (int64_t q = 0; q < n; q++) order[q] = q;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return morton(ijk[3 * a], ijk[3 * a + 1], ijk[3 * a + 2]) < morton(ijk[3 * b], ijk[3 * b + 1], ijk[3 * b + 2]);
    });
    std::vector<uint8_t> mask(512);
    for (int64_t oi = 0; oi < n; oi++) {
        const int64_t B = order[oi];
        const int ob = owner[B];
        // for each peer p != ob: cells of B needed by nodes owned by p adjacent to B
        for (int p = 0; p < nranks; p++) {
            if (p == ob) continue;
            if (p != rank && ob != rank) continue;   // only pairs involving this rank
            std::fill(mask.begin(), mask.end(), 0);
            bool any = false;
            for (int s = 0; s < 27; s++) {
                if (s == 13) continue;
                const int32_t A = nb[B * 27 + s];
                if (A < 0 || owner[A] != p) continue;
                mark_box(mask.data(), s % 3 - 1, (s / 3) % 3 - 1, s / 9 - 1, w);
                any = true;
            }
            if (!any) continue;
            // sender = ob, receiver = p
            const bool send = (ob == rank);
            const int peer = send ? p : ob;
            const int kind = refined[B] ? 1 : 0;
            auto &lst = L[4 * (size_t)peer + (send ? 0 : 2) + kind];
            for (int l = 0; l < 512; l++)
                if (mask[l]) lst.push_back((int32_t)(B * 512 + l));
        }
    }
    for (int p = 0; p < nranks; p++)
        for (int k = 0; k < 4; k++) {
            counts[4 * p + k] = (int64_t)L[4 * p + k].size();
            if (lists && lists[4 * p + k]) std::memcpy(lists[4 * p + k], L[4 * p + k].data(), 4 * L[4 * p + k].size());
        }
    return OCTO_OK;
}

int octo::exchange_plan_level(octo_fmm *h, Level &lv, cudaStream_t st)
{
    const int P = h->cfg.nranks;
    std::vector<int64_t> counts(4 * (size_t)P);
    int rc = octo_fmm_exchange_plan(h->cfg.theta, h->cfg.rank, P, lv.n, lv.ijk.data(), lv.refined.data(),
                                    lv.nb.data(), lv.owner.data(), counts.data(), nullptr);
    if (rc) return fail(h, rc, "exchange plan");
    std::vector<std::vector<int32_t>> L(4 * (size_t)P);
    std::vector<int32_t *> ptrs(4 * (size_t)P);
    for (size_t k = 0; k < L.size(); k++) {
        L[k].resize(counts[k]);
        ptrs[k] = L[k].data();
    }
    octo_fmm_exchange_plan(h->cfg.theta, h->cfg.rank, P, lv.n, lv.ijk.data(), lv.refined.data(), lv.nb.data(),
                           lv.owner.data(), counts.data(), ptrs.data());
    exchange_free_level(lv);
    for (int p = 0; p < P; p++) {
        if (p == h->cfg.rank) continue;
        if (!counts[4 * p] && !counts[4 * p + 1] && !counts[4 * p + 2] && !counts[4 * p + 3]) continue;
        PeerPlan pp;
        pp.peer = p;
        pp.send_leaf = L[4 * p + 0]; pp.send_ref = L[4 * p + 1];
        pp.recv_leaf = L[4 * p + 2]; pp.recv_ref = L[4 * p + 3];

        auto up = [&](int32_t **d, const std::vector<int32_t> &v) -> int {
            if (v.empty()) return OCTO_OK;
            CU(cudaMalloc(d, 4 * v.size()));
            CU(cudaMemcpyAsync(*d, v.data(), 4 * v.size(), cudaMemcpyHostToDevice, st));
            return OCTO_OK;
        };
        if ((rc = up(&pp.d_send_leaf, pp.send_leaf)) || (rc = up(&pp.d_send_ref, pp.send_ref)) ||
            (rc = up(&pp.d_recv_leaf, pp.recv_leaf)) || (rc = up(&pp.d_recv_ref, pp.recv_ref)))
            return rc;
        lv.peers.push_back(pp);
    }
    return OCTO_OK;
}

// ---------------------------------------------------------------------------
// Fused exchange of a set of levels: for every peer ONE send and ONE receive
// buffer holding all levels' ghost records; ONE pack kernel and ONE unpack
// kernel over a segment table (level, kind, index list, buffer) and ONE NCCL
// group with a send/recv pair per peer -- a handful of launches per step
// instead of a pack/unpack and a send/recv per level and peer.
// ---------------------------------------------------------------------------
struct XSeg {
    const int32_t *idx;   // node * 512 + cell
    double *buf;          // leaf: count values; refined: count x 16 (mass + 15 prepared)
    int64_t unit0;        // first work unit of the segment
    int level, is_ref, count, pad;
};

__global__ void xfer_kernel(const LevelDesc *__restrict__ levels, const XSeg *__restrict__ segs, int nseg,
                            int64_t nunits, int unpack, int fence = 0)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nunits; i += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {   // last segment with unit0 <= i
            const int mid = (lo + hi + 1) >> 1;
            if (segs[mid].unit0 <= i) lo = mid; else hi = mid - 1;
        }
        const XSeg &sg = segs[lo];
        const int64_t u = i - sg.unit0;
        const int64_t item = sg.is_ref ? u / NREC : u;
        const int comp = sg.is_ref ? (int)(u % NREC) : 0;
        const int32_t e = sg.idx[item];
        const LevelDesc &D = levels[sg.level];
        const int64_t node = e / 512;
        const int l = e % 512;
        const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
        const int q = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1);
        const int p = (lx >> 1) + 4 * (ly >> 1) + 16 * (lz >> 1);
        // leaf cells: the mass; refined cells: the 16 record components (mass included)
        double *src = !sg.is_ref ? const_cast<double *>(D.mass) + (node * 8 + q) * 64 + p
                                 : const_cast<double *>(D.pref) + prec(D.rslot[node], comp, q, p);
        if (unpack) *src = sg.buf[u];
        else sg.buf[u] = *src;
    }
    if (fence) __threadfence_system();   // puts: this thread's remote stores before the signal
}

// one-sided puts: publish epoch e to every receiving peer (release, system
// scope: the pack kernel's stores to that peer are visible before the flag)
__global__ void xsignal_kernel(unsigned long long *const *__restrict__ rflags, int n, unsigned long long e)
{
    const int i = threadIdx.x;
    if (i >= n) return;
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(rflags[i]), "l"(e) : "memory");
}

// one-sided puts: wait until every sending peer has published epoch e
// (acquire, system scope); a peer that never arrives sets err bit 4 after
// ~20 s instead of hanging the device
__global__ void xwait_kernel(const unsigned long long *__restrict__ flags, const int *__restrict__ senders, int n,
                             unsigned long long e, int *err)
{
    const int i = threadIdx.x;
    if (i >= n) return;
    const unsigned long long *f = flags + senders[i];
    const long long t0 = clock64();
    for (;;) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
        if (v >= e) break;
        if (clock64() - t0 > 40000000000LL) {
            atomicOr(err, 4);
            break;
        }
        __nanosleep(200);
    }
}

// ---------------------------------------------------------------------------
// One-sided NVLink puts (the B200 analogue of the paper's
// libfabric one-sided transfers).  Record of a rank published by
// ncclAllGather when the plan is built (structure changes only):
// [CUDA IPC handle of its arena][byte offset of each sender's segment].
// ---------------------------------------------------------------------------
constexpr int PUT_MAXR = 64;
struct PutRecord {
    cudaIpcMemHandle_t handle;
    int64_t off[PUT_MAXR];   // byte offset of sender s's parity-0 segment (parity 1 follows it)
    int64_t bytes[PUT_MAXR]; // bytes of sender s's segment (one parity)
};

static int put_allgather(octo_fmm *h, const PutRecord &mine, std::vector<PutRecord> &all, cudaStream_t st)
{
    const int P = h->cfg.nranks;
    if (h->cfg.flags & OCTO_EXTERNAL_BOOTSTRAP) {
        if (!h->boot_fn) return fail(h, OCTO_EINVAL, "OCTO_EXTERNAL_BOOTSTRAP handle without octo_fmm_set_bootstrap");
        all.assign(P, PutRecord{});
        if (h->boot_fn(h->boot_ctx, &mine, all.data(), (int64_t)sizeof(PutRecord)) != 0)
            return fail(h, OCTO_ENCCL, "bootstrap allgather (caller callback) failed");
        return OCTO_OK;
    }
    void *d = nullptr;
    CU(cudaMalloc(&d, sizeof(PutRecord) * P));
    CU(cudaMemcpyAsync((char *)d + sizeof(PutRecord) * h->cfg.rank, &mine, sizeof(PutRecord), cudaMemcpyHostToDevice, st));
    NC_(ncclAllGather((char *)d + sizeof(PutRecord) * h->cfg.rank, d, sizeof(PutRecord), ncclUint8,
                      (ncclComm_t)h->nccl_comm, st));
    all.resize(P);
    CU(cudaMemcpyAsync(all.data(), d, sizeof(PutRecord) * P, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    CU(cudaFree(d));
    return OCTO_OK;
}

static int put_teardown(octo_fmm *h, cudaStream_t st)
{
    XPlan &X = h->xplan;
    if (!X.puts || !X.arena) return OCTO_OK;
    CU(cudaStreamSynchronize(st));
    CU(cudaDeviceSynchronize());
    for (void *p : X.imported)
        if (p) cudaIpcCloseMemHandle(p);
    X.imported.clear();
    // every rank has closed its view of the others' arenas before any frees its own
    PutRecord none{};
    std::vector<PutRecord> all;
    int rc = put_allgather(h, none, all, st);
    if (rc) return rc;
    for (void *p : {(void *)X.arena, X.d_psend[0], X.d_psend[1], X.d_precv[0], X.d_precv[1], (void *)X.d_rflags,
                    (void *)X.d_wsend})
        if (p) cudaFree(p);
    X.arena = nullptr;
    return OCTO_OK;
}

static int put_build(octo_fmm *h, const std::vector<Level *> &lvs, const std::vector<int64_t> &rcount, uint64_t key,
                     cudaStream_t st)
{
    XPlan &X = h->xplan;
    const int P = h->cfg.nranks, me = h->cfg.rank;
    if (P > PUT_MAXR) return fail(h, OCTO_EINVAL, "one-sided exchange supports at most 64 ranks");
    // ---- my arena: flags, then per sender two copies of its records
    PutRecord mine{};
    int64_t off = 256 + 8 * (int64_t)P;
    off = (off + 255) / 256 * 256;
    for (int s = 0; s < P; s++) {
        mine.off[s] = off;
        mine.bytes[s] = 8 * rcount[s];
        off += 2 * ((8 * rcount[s] + 255) / 256 * 256);
    }
    CU(cudaMalloc(&X.arena, off));
    CU(cudaMemsetAsync(X.arena, 0, off, st));
    CU(cudaIpcGetMemHandle(&mine.handle, X.arena));
    std::vector<PutRecord> all;
    int rc = put_allgather(h, mine, all, st);
    if (rc) return rc;
    // ---- open the arenas of the peers this rank sends to
    X.imported.assign(P, nullptr);
    std::vector<unsigned long long *> rflags;
    std::vector<int> wsend;
    for (int p = 0; p < P; p++) {
        if (p == me) continue;
        // the double-buffered arena is safe only if every peer relation is
        // symmetric (a receive-only peer could run two epochs ahead and
        // overwrite a buffer still being unpacked): the neighbour relation is
        // symmetric, so sending to p <=> receiving from p; check it
        if ((X.peers[p].send_count != 0) != (X.peers[p].recv_count != 0) ||
            (X.peers[p].send_count != 0) != (all[p].bytes[me] != 0))
            return fail(h, OCTO_ESTRUCT, "ghost exchange is not symmetric between ranks " + std::to_string(me) +
                                             " and " + std::to_string(p) + " (send/receive sets differ)");
        if (X.peers[p].send_count) {
            void *base = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&base, all[p].handle, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess)
                return fail(h, OCTO_ECUDA, std::string("cudaIpcOpenMemHandle (peer arena; set OCTO_XCHG=nccl to use "
                                                       "NCCL send/recv instead): ") + cudaGetErrorString(e));
            X.imported[p] = base;
            if (all[p].bytes[me] != 8 * X.peers[p].send_count)
                return fail(h, OCTO_ESTRUCT, "ghost plan disagrees between ranks (send/receive sizes)");
            rflags.push_back((unsigned long long *)base + me);
        }
        if (X.peers[p].recv_count) wsend.push_back(p);
    }
    // ---- segment tables per parity: sends into the peers' arenas, receives from mine
    for (int par = 0; par < 2; par++) {
        std::vector<XSeg> ss, rs;
        int64_t su = 0, ru = 0;
        for (int p = 0; p < P; p++) {
            int64_t soff = 0, roff = 0;
            double *sbase = X.imported[p] ? (double *)((char *)X.imported[p] + all[p].off[me] +
                                                       par * ((all[p].bytes[me] + 255) / 256 * 256))
                                          : nullptr;
            double *rbase = (double *)((char *)X.arena + mine.off[p] + par * ((mine.bytes[p] + 255) / 256 * 256));
            for (Level *lv : lvs)
                for (auto &pp : lv->peers) {
                    if (pp.peer != p) continue;
                    struct { const std::vector<int32_t> *v; int32_t *d; int ref; bool send; } parts[4] = {
                        {&pp.send_leaf, pp.d_send_leaf, 0, true}, {&pp.send_ref, pp.d_send_ref, 1, true},
                        {&pp.recv_leaf, pp.d_recv_leaf, 0, false}, {&pp.recv_ref, pp.d_recv_ref, 1, false}};
                    for (auto &pt : parts) {
                        if (pt.v->empty()) continue;
                        XSeg sg{};
                        sg.idx = pt.d;
                        sg.level = lv->level;
                        sg.is_ref = pt.ref;
                        sg.count = (int)pt.v->size();
                        const int64_t n = (int64_t)sg.count * (pt.ref ? NREC : 1);
                        if (pt.send) {
                            sg.buf = sbase + soff;
                            sg.unit0 = su;
                            soff += n;
                            su += n;
                            ss.push_back(sg);
                        } else {
                            sg.buf = rbase + roff;
                            sg.unit0 = ru;
                            roff += n;
                            ru += n;
                            rs.push_back(sg);
                        }
                    }
                }
        }
        X.nsend = (int)ss.size();
        X.nrecv = (int)rs.size();
        X.send_units = su;
        X.recv_units = ru;
        if (X.nsend) {
            CU(cudaMalloc(&X.d_psend[par], sizeof(XSeg) * X.nsend));
            CU(cudaMemcpy(X.d_psend[par], ss.data(), sizeof(XSeg) * X.nsend, cudaMemcpyHostToDevice));
        }
        if (X.nrecv) {
            CU(cudaMalloc(&X.d_precv[par], sizeof(XSeg) * X.nrecv));
            CU(cudaMemcpy(X.d_precv[par], rs.data(), sizeof(XSeg) * X.nrecv, cudaMemcpyHostToDevice));
        }
    }
    X.nsig = (int)rflags.size();
    X.nwait = (int)wsend.size();
    if (X.nsig) {
        CU(cudaMalloc(&X.d_rflags, sizeof(void *) * X.nsig));
        CU(cudaMemcpy(X.d_rflags, rflags.data(), sizeof(void *) * X.nsig, cudaMemcpyHostToDevice));
    }
    if (X.nwait) {
        CU(cudaMalloc(&X.d_wsend, sizeof(int) * X.nwait));
        CU(cudaMemcpy(X.d_wsend, wsend.data(), sizeof(int) * X.nwait, cudaMemcpyHostToDevice));
    }
    CU(cudaStreamSynchronize(st));
    X.key = key;
    X.valid = true;
    return OCTO_OK;
}

static int xplan_build(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st)
{
    XPlan &X = h->xplan;
    // one plan over every loaded level (the caller passes them all), keyed by
    // the structure generation: per-level calls reuse it instead of rebuilding
    const uint64_t key = h->generation + 1;
    if (X.valid && X.key == key) return OCTO_OK;
    // free the old plan
    int rc0 = put_teardown(h, st);
    if (rc0) return rc0;
    for (void *p : {(void *)X.d_send_segs, (void *)X.d_recv_segs}) if (p) cudaFree(p);
    for (auto &pp : X.peers) {
        if (pp.sendbuf) cudaFree(pp.sendbuf);
        if (pp.recvbuf) cudaFree(pp.recvbuf);
    }
    X = XPlan();
    const int P = h->cfg.nranks;
    X.puts = h->xput != 0;
    std::vector<XSeg> ss, rs;
    std::vector<int64_t> scount(P, 0), rcount(P, 0);
    // sizes per peer
    for (Level *lv : lvs)
        for (auto &pp : lv->peers) {
            scount[pp.peer] += (int64_t)pp.send_leaf.size() + (int64_t)pp.send_ref.size() * NREC;
            rcount[pp.peer] += (int64_t)pp.recv_leaf.size() + (int64_t)pp.recv_ref.size() * NREC;
        }
    X.peers.resize(P);
    for (int p = 0; p < P; p++) {
        X.peers[p].send_count = scount[p];
        X.peers[p].recv_count = rcount[p];
        if (X.puts) continue;
        if (scount[p]) CU(cudaMalloc(&X.peers[p].sendbuf, 8 * scount[p]));
        if (rcount[p]) CU(cudaMalloc(&X.peers[p].recvbuf, 8 * rcount[p]));
    }
    if (X.puts) return put_build(h, lvs, rcount, key, st);
    // segments, per peer in level order (both sides use the same order)
    std::vector<int64_t> soff(P, 0), roff(P, 0);
    int64_t su = 0, ru = 0;
    for (int p = 0; p < P; p++)
        for (Level *lv : lvs)
            for (auto &pp : lv->peers) {
                if (pp.peer != p) continue;
                struct { const std::vector<int32_t> *v; int32_t *d; int ref; bool send; } parts[4] = {
                    {&pp.send_leaf, pp.d_send_leaf, 0, true}, {&pp.send_ref, pp.d_send_ref, 1, true},
                    {&pp.recv_leaf, pp.d_recv_leaf, 0, false}, {&pp.recv_ref, pp.d_recv_ref, 1, false}};
                for (auto &pt : parts) {
                    if (pt.v->empty()) continue;
                    XSeg sg{};
                    sg.idx = pt.d;
                    sg.level = lv->level;
                    sg.is_ref = pt.ref;
                    sg.count = (int)pt.v->size();
                    const int64_t n = (int64_t)sg.count * (pt.ref ? NREC : 1);
                    if (pt.send) {
                        sg.buf = X.peers[p].sendbuf + soff[p];
                        sg.unit0 = su;
                        soff[p] += n;
                        su += n;
                        ss.push_back(sg);
                    } else {
                        sg.buf = X.peers[p].recvbuf + roff[p];
                        sg.unit0 = ru;
                        roff[p] += n;
                        ru += n;
                        rs.push_back(sg);
                    }
                }
            }
    X.nsend = (int)ss.size();
    X.nrecv = (int)rs.size();
    X.send_units = su;
    X.recv_units = ru;
    if (X.nsend) {
        CU(cudaMalloc(&X.d_send_segs, sizeof(XSeg) * X.nsend));
        CU(cudaMemcpyAsync(X.d_send_segs, ss.data(), sizeof(XSeg) * X.nsend, cudaMemcpyHostToDevice, st));
    }
    if (X.nrecv) {
        CU(cudaMalloc(&X.d_recv_segs, sizeof(XSeg) * X.nrecv));
        CU(cudaMemcpyAsync(X.d_recv_segs, rs.data(), sizeof(XSeg) * X.nrecv, cudaMemcpyHostToDevice, st));
    }
    CU(cudaStreamSynchronize(st));   // host segment vectors must outlive the copies
    X.key = key;
    X.valid = true;
    return OCTO_OK;
}

void octo::exchange_destroy_plan(octo_fmm *h)
{
    XPlan &X = h->xplan;
    if (X.puts) {   // handle teardown: no collective here (peers may be gone); close and free
        cudaDeviceSynchronize();
        for (void *p : X.imported)
            if (p) cudaIpcCloseMemHandle(p);
        for (void *p : {(void *)X.arena, X.d_psend[0], X.d_psend[1], X.d_precv[0], X.d_precv[1],
                        (void *)X.d_rflags, (void *)X.d_wsend})
            if (p) cudaFree(p);
    }
    if (X.d_send_segs) cudaFree(X.d_send_segs);
    if (X.d_recv_segs) cudaFree(X.d_recv_segs);
    for (auto &pp : X.peers) {
        if (pp.sendbuf) cudaFree(pp.sendbuf);
        if (pp.recvbuf) cudaFree(pp.recvbuf);
    }
    X = XPlan();
}

int octo::exchange_pack(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st)
{
    int rc = xplan_build(h, lvs, st);
    if (rc) return rc;
    const XPlan &X = h->xplan;
    if (X.puts) {
        // pack straight into the peers' arenas (NVLink stores), then signal
        const unsigned long long e = ++h->xepoch;
        if (X.send_units) {
            xfer_kernel<<<148 * 4, 256, 0, st>>>(h->d_levels, (const XSeg *)X.d_psend[e & 1], X.nsend, X.send_units,
                                                 0, 1);
            h->launches++;
        }
        if (X.nsig) {
            xsignal_kernel<<<1, 32 * ((X.nsig + 31) / 32), 0, st>>>(X.d_rflags, X.nsig, e);
            h->launches++;
        }
        CU(cudaGetLastError());
        return OCTO_OK;
    }
    if (X.send_units) {
        xfer_kernel<<<148 * 4, 256, 0, st>>>(h->d_levels, (const XSeg *)X.d_send_segs, X.nsend, X.send_units, 0);
        h->launches++;
        CU(cudaGetLastError());
    }
    return OCTO_OK;
}

int octo::exchange_sendrecv_unpack(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st)
{
    (void)lvs;
    const XPlan &X = h->xplan;
    if (X.puts) {
        const unsigned long long e = h->xepoch;
        if (X.nwait) {
            xwait_kernel<<<1, 32 * ((X.nwait + 31) / 32), 0, st>>>((const unsigned long long *)X.arena, X.d_wsend,
                                                                   X.nwait, e, h->d_err);
            h->launches++;
        }
        if (X.recv_units) {
            xfer_kernel<<<148 * 4, 256, 0, st>>>(h->d_levels, (const XSeg *)X.d_precv[e & 1], X.nrecv, X.recv_units, 1);
            h->launches++;
        }
        CU(cudaGetLastError());
        return OCTO_OK;
    }
    ncclComm_t comm = (ncclComm_t)h->nccl_comm;
    NC_(ncclGroupStart());
    for (int p = 0; p < (int)X.peers.size(); p++) {
        if (X.peers[p].send_count) NC_(ncclSend(X.peers[p].sendbuf, (size_t)X.peers[p].send_count, ncclDouble, p, comm, st));
        if (X.peers[p].recv_count) NC_(ncclRecv(X.peers[p].recvbuf, (size_t)X.peers[p].recv_count, ncclDouble, p, comm, st));
    }
    NC_(ncclGroupEnd());
    if (X.recv_units) {
        xfer_kernel<<<148 * 4, 256, 0, st>>>(h->d_levels, (const XSeg *)X.d_recv_segs, X.nrecv, X.recv_units, 1);
        h->launches++;
        CU(cudaGetLastError());
    }
    return OCTO_OK;
}

int octo::exchange_levels(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st)
{
    int rc = exchange_pack(h, lvs, st);
    if (rc) return rc;
    return exchange_sendrecv_unpack(h, lvs, st);
}

int octo::exchange_level(octo_fmm *h, Level &lv, cudaStream_t st)
{
    std::vector<Level *> one{&lv};
    return exchange_levels(h, one, st);
}

extern "C" int octo_fmm_set_bootstrap(octo_fmm_t h, octo_allgather_fn fn, void *ctx)
{
    if (!h || !fn) return OCTO_EINVAL;
    if (!(h->cfg.flags & OCTO_EXTERNAL_BOOTSTRAP))
        return fail(h, OCTO_EINVAL, "octo_fmm_set_bootstrap needs a handle created with OCTO_EXTERNAL_BOOTSTRAP");
    h->boot_fn = fn;
    h->boot_ctx = ctx;
    return OCTO_OK;
}
