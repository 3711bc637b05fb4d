// internal.hpp -- handle / level state shared by octo_fmm.cu and exchange.cu.
#pragma once
#include "octo_fmm.h"
#include "layout.cuh"

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace octo {

constexpr int MAX_LEVELS = 32;

struct PeerPlan {
    int peer = -1;
    // send: (node, cell) of owned cells, receive: (node, cell) of ghost cells,
    // split into mass-only cells (leaf nodes) and refined cells (+19 values)
    std::vector<int32_t> send_leaf, send_ref, recv_leaf, recv_ref;   // packed node*512 + cell
    int32_t *d_send_leaf = nullptr, *d_send_ref = nullptr, *d_recv_leaf = nullptr, *d_recv_ref = nullptr;
};

// fused exchange of a set of levels (exchange.cu): one buffer pair per peer
struct XPeer {
    double *sendbuf = nullptr, *recvbuf = nullptr;
    int64_t send_count = 0, recv_count = 0;   // doubles
};
struct XPlan {
    bool valid = false;
    uint64_t key = 0;
    std::vector<XPeer> peers;
    void *d_send_segs = nullptr, *d_recv_segs = nullptr;
    int nsend = 0, nrecv = 0;
    int64_t send_units = 0, recv_units = 0;
    // one-sided puts: this rank's receive arena = [flags: one
    // uint64 epoch per sender][per sender: 2 x its records (double buffer)],
    // exported by CUDA IPC; the pack kernel stores straight into the peers'
    // arenas (segment tables per buffer parity), then signals their flags
    bool puts = false;
    double *arena = nullptr;
    std::vector<void *> imported;              // per peer: opened IPC base of its arena (or null)
    void *d_psend[2] = {nullptr, nullptr}, *d_precv[2] = {nullptr, nullptr};
    unsigned long long **d_rflags = nullptr;   // remote flag word of each peer this rank sends to
    int *d_wsend = nullptr;                    // senders this rank waits for
    int nsig = 0, nwait = 0;
};

struct Level {
    bool loaded = false, data_ready = false;
    int32_t level = -1;
    int64_t n = 0, nr = 0, n_owned = 0;
    double hc = 0.0, origin[3] = {0, 0, 0};
    std::vector<int32_t> ijk, nb, owner, rnode, oslot;
    std::vector<uint8_t> refined;
    std::vector<int2> work_ref, work_leaf, work_mixed;   // interior nodes first, then boundary
    std::vector<float> cost_ref, cost_leaf, cost_mixed;  // per work item (cost estimate, for LPT order)
    int nint[3] = {0, 0, 0};                              // interior counts of the three lists
    int64_t counts[3] = {0, 0, 0};
    int64_t h2d_bytes = 0;
    // ingest deferred to the next compute call (batched prep kernel)
    bool prep_pending = false;
    const double *src_mono = nullptr, *src_com = nullptr, *src_mom = nullptr;
    // device
    int32_t *d_ijk = nullptr, *d_nb = nullptr, *d_rslot = nullptr, *d_oslot = nullptr, *d_rnode = nullptr;
    uint8_t *d_kind = nullptr, *d_use = nullptr;
    double *d_mass = nullptr, *d_pref = nullptr, *d_L = nullptr, *d_Lc = nullptr;
    void *d_tmaps = nullptr;   // 7 CUtensorMap over d_pref (mixed kernel's halo boxes), nr > 0 only
    double *d_in_mono = nullptr, *d_in_com = nullptr, *d_in_mom = nullptr;
    int2 *d_work_ref = nullptr, *d_work_leaf = nullptr, *d_work_mixed = nullptr;
    int16_t *d_msort = nullptr;
    // output slots: owned refined nodes first, then owned leaf nodes (node
    // order within each), so the compact getter is plain 2-D copies;
    // ordslot[j] = slot of the j-th owned node in node order (node-order getters)
    std::vector<int32_t> ordslot;
    // runs [a, b) of owned nodes (node index) and of owned refined slots: the
    // only input rows a rank ingests, so host inputs copy just these
    std::vector<std::pair<int64_t, int64_t>> own_runs, own_rruns;
    int32_t *d_ordslot = nullptr;
    double *d_gbuf = nullptr;   // staging of get_expansions to host memory
    int64_t c_nref = 0, c_nleaf = 0;
    // multi-rank ghost exchange
    std::vector<PeerPlan> peers;
    // last descriptor uploaded to h->d_levels[level] (host copy: the source of
    // the asynchronous upload must stay alive, and an unchanged one is skipped)
    LevelDesc desc{};
    bool desc_valid = false;
};

struct WorkArr {
    int2 *ptr = nullptr;
    int n = 0, nint = 0;   // interior items first
};

}  // namespace octo

struct octo_fmm {
    octo_fmm_config cfg{};
    std::string last_error;
    int64_t launches = 0;
    int reach = 2;        // parent reach of the stencil: 2 (theta >= 1/3) or 3 (0.25 <= theta < 1/3)
    int p2p8 = 1;         // P2P: 1 = p2p8_kernel (8 targets per thread, K shared by a child row), 0 = p2p_kernel
    int mix_tma = 0;      // mixed kernel: 1 = halo boxes staged by TMA (cp.async.bulk.tensor + mbarrier)
    int m2l_unroll = -1;  // pairs per far-loop iteration of the reach-2 M2L kernel; -1: measured best (2)
    double *d_p2pk = nullptr;   // reach 3: K(d) table for |d| <= 7 (global memory)
    std::vector<int> elist, ecount, efar, rows, dlist, mstart, mitem;
    std::vector<uint32_t> emask;
    int64_t slot_count[27][2] = {};
    int *d_elist = nullptr, *d_ecount = nullptr, *d_efar = nullptr, *d_rows = nullptr;
    uint32_t *d_emask = nullptr;
    int *d_dlist = nullptr, *d_mstart = nullptr, *d_mitem = nullptr;
    octo::LevelDesc *d_levels = nullptr;
    int *d_err = nullptr;
    std::vector<octo::Level> levels;
    uint64_t generation = 0, all_gen = ~0ull;
    octo::WorkArr all_work[3];
    void *nccl_comm = nullptr;   // ncclComm_t
    // OCTO_EXTERNAL_BOOTSTRAP: the caller's allgather sets up the one-sided exchange
    octo_allgather_fn boot_fn = nullptr;
    void *boot_ctx = nullptr;
    int xput = 1;                // ghost exchange: 1 one-sided NVLink puts (CUDA IPC), 0 NCCL send/recv
    unsigned long long xepoch = 0;   // exchanges issued (the epoch the put flags carry)
    octo::XPlan xplan;
    // OCTO_TIMING: event quadruples per compute call (pending until queried)
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::array<cudaEvent_t, 6>> ev_pending;
    int64_t ncompute = 0;                 // compute calls since the last kernel_times query
    // multi-rank: ghost exchange on its own stream, overlapped with interior work
    cudaStream_t comm_stream = nullptr;
    // M2L on a higher-priority stream, the leaf kernels beside it on the caller's stream
    int concurrency = 0;    // leaf kernels beside M2L on the caller's stream (0 off, 1 on)
    // 1: exchange first (~0.1 ms with the whole GPU), then every node in one round;
    // 0: interior nodes overlapped with the exchange, boundary nodes after it (the
    // NCCL kernels then wait for SM slots behind long M2L CTAs: 0.6-1 ms measured)
    int xmode = 1;
    int lpt_mask = -1;      // LPT order per kernel (1 M2L, 2 P2P, 4 mixed), else Morton order; -1: 5
    cudaStream_t m2l_stream = nullptr;
    cudaStream_t root_stream = nullptr;   // the root kernel runs beside the level kernels
    cudaEvent_t ev_rfork = nullptr, ev_rjoin = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_packed = nullptr, ev_recv = nullptr;
    std::vector<std::array<cudaEvent_t, 2>> xev_pending;   // OCTO_TIMING: exchange events per call

};

namespace octo {
int fail(octo_fmm *h, int code, const std::string &msg);
int device_init(octo_fmm *h);
int exchange_init(octo_fmm *h);
void exchange_destroy(octo_fmm *h);
void exchange_free_level(Level &lv);
int exchange_plan_level(octo_fmm *h, Level &lv, cudaStream_t st);
int exchange_level(octo_fmm *h, Level &lv, cudaStream_t st);
int exchange_levels(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st);
int exchange_pack(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st);
void exchange_destroy_plan(octo_fmm *h);
int exchange_sendrecv_unpack(octo_fmm *h, const std::vector<Level *> &lvs, cudaStream_t st);
int parent_reach(double theta);
}  // namespace octo
