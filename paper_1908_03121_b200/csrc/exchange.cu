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
    if (h->nccl_comm) ncclCommDestroy((ncclComm_t)h->nccl_comm);
    h->nccl_comm = nullptr;
}

void octo::exchange_free_level(Level &lv)
{
    for (auto &p : lv.peers) {
        void *ptrs[] = {p.d_send_leaf, p.d_send_ref, p.d_recv_leaf, p.d_recv_ref, p.d_sendbuf, p.d_recvbuf};
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

// ---------------------------------------------------------------------------
// device side: pack / unpack prepared records
// ---------------------------------------------------------------------------
// buffer layout per peer: [leaf masses][refined masses][refined 19 x n_ref]
__global__ void pack_kernel(const LevelDesc *__restrict__ levels, int lvl, const int32_t *__restrict__ leaf, int nl,
                            const int32_t *__restrict__ ref, int nrf, double *__restrict__ buf)
{
    const LevelDesc &D = levels[lvl];
    const int64_t tot = (int64_t)nl + (int64_t)nrf * (1 + NPREP);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t e;
        int comp;
        if (i < nl) { e = leaf[i]; comp = -1; }
        else {
            const int64_t j = i - nl;
            e = ref[j % nrf];
            comp = (int)(j / nrf) - 1;   // -1 = mass, 0..18 prepared
        }
        const int64_t node = e / 512;
        const int l = e % 512;
        const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
        const int q = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1);
        const int p = (lx >> 1) + 4 * (ly >> 1) + 16 * (lz >> 1);
        double v;
        if (comp < 0) v = D.mass[(node * 8 + q) * 64 + p];
        else v = D.pref[(((int64_t)D.rslot[node] * NPREP + comp) * 8 + q) * 64 + p];
        buf[i] = v;
    }
}

__global__ void unpack_kernel(const LevelDesc *__restrict__ levels, int lvl, const int32_t *__restrict__ leaf, int nl,
                              const int32_t *__restrict__ ref, int nrf, const double *__restrict__ buf)
{
    const LevelDesc &D = levels[lvl];
    double *mass = const_cast<double *>(D.mass);
    double *pref = const_cast<double *>(D.pref);
    const int64_t tot = (int64_t)nl + (int64_t)nrf * (1 + NPREP);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t e;
        int comp;
        if (i < nl) { e = leaf[i]; comp = -1; }
        else {
            const int64_t j = i - nl;
            e = ref[j % nrf];
            comp = (int)(j / nrf) - 1;
        }
        const int64_t node = e / 512;
        const int l = e % 512;
        const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
        const int q = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1);
        const int p = (lx >> 1) + 4 * (ly >> 1) + 16 * (lz >> 1);
        if (comp < 0) mass[(node * 8 + q) * 64 + p] = buf[i];
        else pref[(((int64_t)D.rslot[node] * NPREP + comp) * 8 + q) * 64 + p] = buf[i];
    }
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
        pp.send_count = (int64_t)pp.send_leaf.size() + (int64_t)pp.send_ref.size() * (1 + NPREP);
        pp.recv_count = (int64_t)pp.recv_leaf.size() + (int64_t)pp.recv_ref.size() * (1 + NPREP);
        auto up = [&](int32_t **d, const std::vector<int32_t> &v) -> int {
            if (v.empty()) return OCTO_OK;
            CU(cudaMalloc(d, 4 * v.size()));
            CU(cudaMemcpyAsync(*d, v.data(), 4 * v.size(), cudaMemcpyHostToDevice, st));
            return OCTO_OK;
        };
        if ((rc = up(&pp.d_send_leaf, pp.send_leaf)) || (rc = up(&pp.d_send_ref, pp.send_ref)) ||
            (rc = up(&pp.d_recv_leaf, pp.recv_leaf)) || (rc = up(&pp.d_recv_ref, pp.recv_ref)))
            return rc;
        if (pp.send_count) CU(cudaMalloc(&pp.d_sendbuf, 8 * pp.send_count));
        if (pp.recv_count) CU(cudaMalloc(&pp.d_recvbuf, 8 * pp.recv_count));
        lv.peers.push_back(pp);
    }
    return OCTO_OK;
}

// Ghost exchange of a set of levels: pack every (level, peer) buffer, ONE
// NCCL group of all sends and receives, unpack (levels are independent, so
// batching them costs one group latency instead of one per level).  Split in
// two so compute_interactions can overlap the group with interior work.
int octo::exchange_pack(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st)
{
    for (Level *lv : lvs)
        for (auto &p : lv->peers)
            if (p.send_count) {
                pack_kernel<<<148 * 4, 256, 0, st>>>(h->d_levels, lv->level, p.d_send_leaf, (int)p.send_leaf.size(),
                                                     p.d_send_ref, (int)p.send_ref.size(), p.d_sendbuf);
                h->launches++;
            }
    CU(cudaGetLastError());
    return OCTO_OK;
}

int octo::exchange_sendrecv_unpack(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st)
{
    ncclComm_t comm = (ncclComm_t)h->nccl_comm;
    NC_(ncclGroupStart());
    for (Level *lv : lvs)
        for (auto &p : lv->peers) {
            if (p.send_count) NC_(ncclSend(p.d_sendbuf, (size_t)p.send_count, ncclDouble, p.peer, comm, st));
            if (p.recv_count) NC_(ncclRecv(p.d_recvbuf, (size_t)p.recv_count, ncclDouble, p.peer, comm, st));
        }
    NC_(ncclGroupEnd());
    for (Level *lv : lvs)
        for (auto &p : lv->peers)
            if (p.recv_count) {
                unpack_kernel<<<148 * 4, 256, 0, st>>>(h->d_levels, lv->level, p.d_recv_leaf, (int)p.recv_leaf.size(),
                                                       p.d_recv_ref, (int)p.recv_ref.size(), p.d_recvbuf);
                h->launches++;
            }
    CU(cudaGetLastError());
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
