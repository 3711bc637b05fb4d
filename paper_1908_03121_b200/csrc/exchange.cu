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
                            int64_t nunits, int unpack)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nunits; i += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nseg - 1;
        while (lo < hi) {   // last segment with unit0 <= i
            const int mid = (lo + hi + 1) >> 1;
            if (segs[mid].unit0 <= i) lo = mid; else hi = mid - 1;
        }
        const XSeg &sg = segs[lo];
        const int64_t u = i - sg.unit0;
        const int64_t item = sg.is_ref ? u / (1 + NPREP) : u;
        const int comp = sg.is_ref ? (int)(u % (1 + NPREP)) : 0;
        const int32_t e = sg.idx[item];
        const LevelDesc &D = levels[sg.level];
        const int64_t node = e / 512;
        const int l = e % 512;
        const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
        const int q = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1);
        const int p = (lx >> 1) + 4 * (ly >> 1) + 16 * (lz >> 1);
        double *src = comp == 0 ? const_cast<double *>(D.mass) + (node * 8 + q) * 64 + p
                                : const_cast<double *>(D.pref) + (((int64_t)D.rslot[node] * NPREP + comp - 1) * 8 + q) * 64 + p;
        if (unpack) *src = sg.buf[u];
        else sg.buf[u] = *src;
    }
}

static int xplan_build(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st)
{
    XPlan &X = h->xplan;
    uint64_t key = h->generation * 1315423911ull;
    for (Level *lv : lvs) key = key * 31 + (uint64_t)lv->level + 1;
    if (X.valid && X.key == key) return OCTO_OK;
    // free the old plan
    for (void *p : {(void *)X.d_send_segs, (void *)X.d_recv_segs}) if (p) cudaFree(p);
    for (auto &pp : X.peers) {
        if (pp.sendbuf) cudaFree(pp.sendbuf);
        if (pp.recvbuf) cudaFree(pp.recvbuf);
    }
    X = XPlan();
    const int P = h->cfg.nranks;
    std::vector<XSeg> ss, rs;
    std::vector<int64_t> scount(P, 0), rcount(P, 0);
    // sizes per peer
    for (Level *lv : lvs)
        for (auto &pp : lv->peers) {
            scount[pp.peer] += (int64_t)pp.send_leaf.size() + (int64_t)pp.send_ref.size() * (1 + NPREP);
            rcount[pp.peer] += (int64_t)pp.recv_leaf.size() + (int64_t)pp.recv_ref.size() * (1 + NPREP);
        }
    X.peers.resize(P);
    for (int p = 0; p < P; p++) {
        X.peers[p].send_count = scount[p];
        X.peers[p].recv_count = rcount[p];
        if (scount[p]) CU(cudaMalloc(&X.peers[p].sendbuf, 8 * scount[p]));
        if (rcount[p]) CU(cudaMalloc(&X.peers[p].recvbuf, 8 * rcount[p]));
    }
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
                    const int64_t n = (int64_t)sg.count * (pt.ref ? 1 + NPREP : 1);
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
