// octo_fmm.cu -- C-ABI implementation (include/octo_fmm.h) of the B200-native
// stencil FMM same-level step.  Host code: validation, structure caching,
// stencil tables, work lists, launches, ghost exchange (exchange.cu).
//
// Paper passages: P:L475-481 (same-level step), P:L485 (1074 stencil),
// P:L505-521 (interaction cases / kernels), P:L511-513 (sub-grid + 26
// neighbours as halo).  Readings: DESIGN.md.
#include "octo_fmm.h"
#include "kernels.cuh"
#include "internal.hpp"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace octo;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
extern "C" const char *octo_fmm_strerror(int code)
{
    switch (code) {
    case OCTO_OK: return "ok";
    case OCTO_EINVAL: return "invalid argument";
    case OCTO_ESTRUCT: return "structural error (neighbour table / 2:1 grading)";
    case OCTO_EMASS: return "non-positive cell mass";
    case OCTO_ECUDA: return "CUDA error";
    case OCTO_ENCCL: return "NCCL error";
    case OCTO_ENOMEM: return "out of device memory";
    default: return "unknown error";
    }
}

int octo::fail(octo_fmm *h, int code, const std::string &msg)
{
    if (h) h->last_error = std::string(octo_fmm_strerror(code)) + ": " + msg;
    return code;
}

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            if (e_ == cudaErrorMemoryAllocation) return fail(h, OCTO_ENOMEM, #call);           \
            return fail(h, OCTO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
        }                                                                                      \
    } while (0)

// failures of octo_fmm_create (no handle yet) are kept per thread
static thread_local std::string g_create_error;
extern "C" const char *octo_fmm_last_error(octo_fmm_t h) { return h ? h->last_error.c_str() : g_create_error.c_str(); }
extern "C" int64_t octo_fmm_launch_count(octo_fmm_t h) { return h ? h->launches : -1; }

// ---------------------------------------------------------------------------
// stencil (C1 reading): partner j of target i is taken at this
// level iff its parent is "parent-near": |floor(j/2) - floor(i/2)|^2 < R^2,
// R^2 = (1/theta)^2; far iff |j - i|^2 >= R^2, else near.  Equivalently, for
// target parity c the partners are the children q of the parent offsets P
// with |P|^2 < R^2, d = 2P + q - c != 0.  Built per (c, q) as P lists.
// ---------------------------------------------------------------------------
static void build_stencil(octo_fmm *h)
{
    const double r = 1.0 / h->cfg.theta;
    const double R2 = r * r;   // same rounding as the reading states: (1/theta)^2 computed once
    const int pmax = (int)std::floor(std::sqrt(R2)) + 1;
    h->elist.assign(64 * MAXE, 0);
    h->ecount.assign(64, 0);
    std::memset(h->slot_count, 0, sizeof(h->slot_count));
    h->efar.assign(64, 0);
    for (int c = 0; c < 8; c++) {
        const int cb[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
        for (int q = 0; q < 8; q++) {
            const int qb[3] = {q & 1, (q >> 1) & 1, (q >> 2) & 1};
            int n = 0;
            for (int pass = 0; pass < 2; pass++) {   // far entries first, then near
                for (int pz = -pmax; pz <= pmax; pz++)
                    for (int py = -pmax; py <= pmax; py++)
                        for (int px = -pmax; px <= pmax; px++) {
                            const long p2 = (long)px * px + (long)py * py + (long)pz * pz;
                            if (!((double)p2 < R2)) continue;
                            const int d[3] = {2 * px + qb[0] - cb[0], 2 * py + qb[1] - cb[1], 2 * pz + qb[2] - cb[2]};
                            const long d2 = (long)d[0] * d[0] + (long)d[1] * d[1] + (long)d[2] * d[2];
                            if (d2 == 0) continue;
                            const int nearf = ((double)d2 >= R2) ? 0 : 1;
                            if (nearf != pass) continue;
                            h->elist[(c * 8 + q) * MAXE + n] =
                                (px & 0xff) | ((py & 0xff) << 8) | ((pz & 0xff) << 16) | (nearf << 24);
                            n++;
                        }
                if (pass == 0) h->efar[c * 8 + q] = n;
            }
            h->ecount[c * 8 + q] = n;
        }
    }
    // neighbour-slot masks: for warp half `hf` of parity c (target parents
    // x 0..3, y 0..3, z 2hf..2hf+1) and entry e of list (c, q), the set of
    // neighbour slots its 32 partners fall into (kernels skip entries whose
    // slots hold no partner of the wanted kind with one AND).
    h->emask.assign(3 * 64 * MAXE * 2, 0u);
    for (int so = 0; so < 3; so++)
        for (int c = 0; c < 8; c++)
            for (int q = 0; q < 8; q++)
                for (int e = 0; e < h->ecount[c * 8 + q]; e++) {
                    const int v = h->elist[(c * 8 + q) * MAXE + e];
                    const int P[3] = {(int8_t)(v & 0xff), (int8_t)((v >> 8) & 0xff), (int8_t)((v >> 16) & 0xff)};
                    for (int hf = 0; hf < 2; hf++) {
                        uint32_t m = 0;
                        for (int lane = 0; lane < 32; lane++) {
                            // same lane -> target-parent map as orient_target (kernels.cuh)
                            const int a = lane & 3, b = (lane >> 2) & 3, sp = 2 * hf + (lane >> 4);
                            const int t[3] = {so == 0 ? sp : a, so == 1 ? sp : (so == 0 ? a : b), so == 2 ? sp : b};
                            int o[3];
                            for (int ax = 0; ax < 3; ax++) {
                                const int cell = 2 * (t[ax] + P[ax]) + ((q >> ax) & 1);
                                o[ax] = (cell >= 8) - (cell < 0);
                            }
                            m |= 1u << ((o[0] + 1) + 3 * (o[1] + 1) + 9 * (o[2] + 1));
                        }
                        h->emask[(((so * 64) + c * 8 + q) * MAXE + e) * 2 + hf] = m;
                    }
                }
    // additive window offsets of every entry per warp orientation (the M2L
    // kernel's index is base + offset; strides as in m2l_dense_kernel: the
    // split axis `so` gets the plane stride SW, the others 1 and SV)
    h->reach = octo::parent_reach(h->cfg.theta);
    h->dlist.assign(3 * 64 * MAXE, 0);
    for (int so = 0; so < 3; so++) {
        const int W = h->reach == 3 ? Win<3>::SW : Win<2>::SW, V = h->reach == 3 ? Win<3>::SV : Win<2>::SV;
        const int sx = so == 0 ? W : 1, sy = so == 1 ? W : (so == 0 ? 1 : V), sz = so == 2 ? W : V;
        for (int cq = 0; cq < 64; cq++)
            for (int e = 0; e < h->ecount[cq]; e++) {
                const int v = h->elist[cq * MAXE + e];
                const int px = (int8_t)(v & 0xff), py = (int8_t)((v >> 8) & 0xff), pz = (int8_t)((v >> 16) & 0xff);
                h->dlist[(so * 64 + cq) * MAXE + e] = px * sx + py * sy + pz * sz;
            }
    }
    // mixed kernel lists: for every cell l of a node and neighbour slot s, the
    // stencil partners (child parity q | parent index << 3) that land in slot
    // s, in (q, entry) order; mstart[l][28] prefix offsets into mitem
    h->mstart.assign(512 * 28, 0);
    h->mitem.clear();
    {
        std::vector<std::vector<int>> per(27);
        for (int l = 0; l < NC; l++) {
            for (auto &v : per) v.clear();
            const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
            const int c = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1);
            for (int q = 0; q < 8; q++)
                for (int e = 0; e < h->ecount[c * 8 + q]; e++) {
                    const int v = h->elist[(c * 8 + q) * MAXE + e];
                    const int px = (int8_t)(v & 0xff), py = (int8_t)((v >> 8) & 0xff), pz = (int8_t)((v >> 16) & 0xff);
                    const int gx = 2 * ((lx >> 1) + px) + (q & 1), gy = 2 * ((ly >> 1) + py) + ((q >> 1) & 1),
                              gz = 2 * ((lz >> 1) + pz) + (q >> 2);
                    const int ox = (gx >= 8) - (gx < 0), oy = (gy >= 8) - (gy < 0), oz = (gz >= 8) - (gz < 0);
                    const int pidx = ((gx - 8 * ox) >> 1) + 4 * ((gy - 8 * oy) >> 1) + 16 * ((gz - 8 * oz) >> 1);
                    per[(ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)].push_back(q | (pidx << 3));
                }
            for (int s = 0; s < 27; s++) {
                h->mstart[l * 28 + s] = (int)h->mitem.size();
                h->mitem.insert(h->mitem.end(), per[s].begin(), per[s].end());
            }
            h->mstart[l * 28 + 27] = (int)h->mitem.size();
        }
    }
    // P2P rows of the parent stencil: (Py, Pz) with the half-width xr of the
    // contiguous Px range {Px : Px^2 + Py^2 + Pz^2 < R^2}
    h->rows.clear();
    for (int pz = -pmax; pz <= pmax; pz++)
        for (int py = -pmax; py <= pmax; py++) {
            int xr = -1;
            for (int px = 0; px <= pmax; px++)
                if ((double)((long)px * px + (long)py * py + (long)pz * pz) < R2) xr = px;
            if (xr >= 0) h->rows.push_back((py & 0xff) | ((pz & 0xff) << 8) | (xr << 16));
        }
    // per-neighbour-slot counts for interaction accounting: for every target
    // cell of a node and every stencil partner, which neighbour slot it lands in
    for (int l = 0; l < NC; l++) {
        const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
        const int c = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1);
        for (int q = 0; q < 8; q++)
            for (int e = 0; e < h->ecount[c * 8 + q]; e++) {
                const int v = h->elist[(c * 8 + q) * MAXE + e];
                const int px = (int8_t)(v & 0xff), py = (int8_t)((v >> 8) & 0xff), pz = (int8_t)((v >> 16) & 0xff);
                const int nearf = (v >> 24) & 1;
                const int gx = lx + 2 * px + (q & 1) - (lx & 1);
                const int gy = ly + 2 * py + ((q >> 1) & 1) - (ly & 1);
                const int gz = lz + 2 * pz + ((q >> 2) & 1) - (lz & 1);
                const int ox = (gx >= 8) - (gx < 0), oy = (gy >= 8) - (gy < 0), oz = (gz >= 8) - (gz < 0);
                h->slot_count[(ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)][nearf]++;
            }
    }
}

extern "C" int octo_fmm_node_costs(double theta, int64_t n, const uint8_t *refined, const int32_t *nb,
                                   int64_t *counts)
{
    if (!(theta >= 0.25 && theta <= 1.0) || octo::parent_reach(theta) > 3 || n < 0) return OCTO_EINVAL;
    if (n > 0 && (!refined || !nb || !counts)) return OCTO_EINVAL;
    octo_fmm tmp;   // host tables only (no device state)
    tmp.cfg.theta = theta;
    build_stencil(&tmp);
    for (int64_t q = 0; q < n; q++) {
        int64_t *c = counts + 3 * q;
        c[0] = c[1] = c[2] = 0;
        for (int s = 0; s < 27; s++) {
            const int32_t r = nb[q * 27 + s];
            if (r < 0 || r >= n) continue;
            const int64_t nf = tmp.slot_count[s][0], nn = tmp.slot_count[s][1];
            if (refined[q]) c[1] += nf + (refined[r] ? 0 : nn);
            else if (refined[r]) c[2] += nf + nn;
            else c[0] += nf + nn;
        }
    }
    return OCTO_OK;
}

// K(d) = (-1/|d|, -d/|d|^3) for d in [-kb, kb]^3 (d = 0: zeros)
static void p2p_table(std::vector<double> &t, int kb)
{
    const int kd = 2 * kb + 1;
    t.assign(4 * kd * kd * kd, 0.0);
    for (int dz = -kb; dz <= kb; dz++)
        for (int dy = -kb; dy <= kb; dy++)
            for (int dx = -kb; dx <= kb; dx++) {
                const int k = (dx + kb) + kd * ((dy + kb) + kd * (dz + kb));
                const double d2 = (double)(dx * dx + dy * dy + dz * dz);
                if (d2 == 0.0) continue;
                const double r = std::sqrt(d2);
                const double r3 = r * d2;
                t[4 * k + 0] = -1.0 / r;
                t[4 * k + 1] = -(double)dx / r3;
                t[4 * k + 2] = -(double)dy / r3;
                t[4 * k + 3] = -(double)dz / r3;
            }
}

// ---------------------------------------------------------------------------
// create / destroy
// ---------------------------------------------------------------------------
extern "C" int octo_fmm_create(const octo_fmm_config *cfg, octo_fmm_t *out)
{
    octo_fmm *h = nullptr;
    if (!cfg || !out) return OCTO_EINVAL;
    *out = nullptr;
    // theta in [0.25, 1]: parent reach <= 3, stencil cell reach <= 7 < 8
    if (cfg->abi_version != OCTO_FMM_ABI_VERSION || cfg->n != 8 || !(cfg->theta >= 0.25 && cfg->theta <= 1.0) ||
        octo::parent_reach(cfg->theta) > 3 ||
        !(cfg->G > 0.0) || cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks)
        return OCTO_EINVAL;
    h = new octo_fmm();
    h->cfg = *cfg;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || cfg->device < 0 || cfg->device >= ndev) {
        delete h;
        return OCTO_ECUDA;
    }
    if (cudaSetDevice(cfg->device) != cudaSuccess) { delete h; return OCTO_ECUDA; }
    build_stencil(h);
    int rc = octo::device_init(h);
    if (rc != OCTO_OK) {
        g_create_error = h->last_error;
        delete h;
        return rc;
    }
    if (cfg->nranks > 1) {
        rc = octo::exchange_init(h);
        if (rc != OCTO_OK) {
            g_create_error = h->last_error;
            octo_fmm_destroy(h);
            return rc;
        }
    }
    *out = h;
    return OCTO_OK;
}

template <int R>
static int set_kernel_attrs(octo_fmm *h)
{
    const int m2l = (int)sizeof(M2LDSmem<R>), p2p = (int)sizeof(P2PSmem<R>);
    // R = 2: 3 CTAs x 72 KB per SM needs the whole shared-memory carveout
    auto m2l_attr = [&](auto k) -> int {
        CU(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, m2l));
        CU(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        return OCTO_OK;
    };
    int rc;
    if ((rc = m2l_attr(m2l_dense_kernel<true, 1, R>)) || (rc = m2l_attr(m2l_dense_kernel<false, 1, R>))) return rc;
    if constexpr (R == 2) {   // unrolled far loops: reach 2 only (the tuned path)
        if ((rc = m2l_attr(m2l_dense_kernel<true, 2, R>)) || (rc = m2l_attr(m2l_dense_kernel<true, 3, R>))) return rc;
#ifdef M2L_U4
        if ((rc = m2l_attr(m2l_dense_kernel<true, 4, R>))) return rc;
#endif
    }
    CU(cudaFuncSetAttribute(p2p_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, p2p));
    CU(cudaFuncSetAttribute(p2p8_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, p2p));
    // the mixed kernel's unstaged partners are read through L1: ask for just the
    // shared memory its resident CTAs need and leave the rest of the 256 KB to L1
    const int carve0 = std::min(100, (int)((100 * (MIX_MINB * (sizeof(MixSmem<false>) + 1024)) + 228 * 1024 - 1) / (228 * 1024)));
    const int carve1 = std::min(100, (int)((100 * (MIX_MINB_TMA * (sizeof(MixSmem<true>) + 1024)) + 228 * 1024 - 1) / (228 * 1024)));
    for (auto k : {m2l_mixed_kernel<true, R, false>, m2l_mixed_kernel<false, R, false>}) {
        CU(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MixSmem<false>)));
        CU(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve0));
    }
    for (auto k : {m2l_mixed_kernel<true, R, true>, m2l_mixed_kernel<false, R, true>}) {
        CU(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(MixSmem<true>)));
        CU(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve1));
    }
    return OCTO_OK;
}

int octo::device_init(octo_fmm *h)
{
    std::vector<double> t;
    p2p_table(t, KBOX2);
    CU(cudaMemcpyToSymbol(c_p2p, t.data(), t.size() * sizeof(double)));
    if (h->reach == 3) {   // |d| <= 7: the global K(d) table of the reach-3 P2P kernel
        p2p_table(t, KBOX);
        CU(cudaMalloc(&h->d_p2pk, t.size() * sizeof(double)));
        CU(cudaMemcpy(h->d_p2pk, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    CU(cudaMalloc(&h->d_elist, h->elist.size() * sizeof(int)));
    CU(cudaMalloc(&h->d_ecount, h->ecount.size() * sizeof(int)));
    CU(cudaMemcpy(h->d_elist, h->elist.data(), h->elist.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_ecount, h->ecount.data(), h->ecount.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&h->d_efar, h->efar.size() * sizeof(int)));
    CU(cudaMemcpy(h->d_efar, h->efar.data(), h->efar.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&h->d_emask, h->emask.size() * sizeof(uint32_t)));
    CU(cudaMemcpy(h->d_emask, h->emask.data(), h->emask.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&h->d_dlist, h->dlist.size() * sizeof(int)));
    CU(cudaMemcpy(h->d_dlist, h->dlist.data(), h->dlist.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&h->d_mstart, h->mstart.size() * sizeof(int)));
    CU(cudaMemcpy(h->d_mstart, h->mstart.data(), h->mstart.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&h->d_mitem, h->mitem.size() * sizeof(int)));
    CU(cudaMemcpy(h->d_mitem, h->mitem.data(), h->mitem.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&h->d_rows, h->rows.size() * sizeof(int)));
    CU(cudaMemcpy(h->d_rows, h->rows.data(), h->rows.size() * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&h->d_levels, sizeof(LevelDesc) * MAX_LEVELS));
    CU(cudaMemset(h->d_levels, 0, sizeof(LevelDesc) * MAX_LEVELS));
    CU(cudaMalloc(&h->d_err, sizeof(int)));
    CU(cudaMemset(h->d_err, 0, sizeof(int)));
    if (const char *v = std::getenv("OCTO_M2L_UNROLL")) h->m2l_unroll = std::atoi(v);   // tuning knob (1..3)
    if (const char *v = std::getenv("OCTO_MIX_TMA")) h->mix_tma = std::atoi(v) != 0;   // TMA halo staging (mixed)
    if (const char *v = std::getenv("OCTO_P2P8")) h->p2p8 = std::atoi(v) != 0;         // 8 targets per P2P thread
    if (h->m2l_unroll < 0) h->m2l_unroll = 2;
    int rc = h->reach == 3 ? set_kernel_attrs<3>(h) : set_kernel_attrs<2>(h);
    if (rc) return rc;
    if (const char *v = std::getenv("OCTO_CONCURRENCY")) h->concurrency = std::atoi(v);   // tuning knob (0, 1)
    if (const char *v = std::getenv("OCTO_LPT")) h->lpt_mask = std::atoi(v);   // tuning knob (0..7)
    // M2L in Morton order keeps neighbour reads L2-local (best on one GPU); with a
    // few hundred M2L CTAs per rank, longest-first order shortens the tail instead
    if (h->lpt_mask < 0) h->lpt_mask = 5;   // LPT for M2L and mixed; P2P (uniform cost per node) in Morton order
    if (const char *v = std::getenv("OCTO_XMODE")) h->xmode = std::atoi(v);   // tuning knob (0, 1)
    if (const char *v = std::getenv("OCTO_XCHG")) h->xput = std::string(v) != "nccl";   // exchange transport
    CU(cudaFuncSetAttribute(root_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RootSmem)));
    CU(cudaFuncSetAttribute(root_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RootSmem)));
    return OCTO_OK;
}

// TMA descriptors of a level's prepared records (the mixed kernel's halo
// boxes): pref viewed as a 5-D tensor of doubles {x-pair 8, y 4, z 4, q 8,
// pair-of-record 8 * nr} (strides 64 B, 256 B, 1 KB, 8 KB: layout.cuh prec),
// one box shape per neighbour-offset class: shape bits (x, y, z) set where
// the offset is non-zero (extent R there, 4 elsewhere).
static int make_tmaps(octo_fmm *h, Level &lv, cudaStream_t st)
{
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail(h, OCTO_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const int R = h->reach == 3 ? 3 : 2;   // the kernels' reach (reach 1 runs the reach-2 kernels)
    CUtensorMap maps[7];
    const cuuint64_t dims[5] = {8, 4, 4, 8, (cuuint64_t)(8 * lv.nr)};
    const cuuint64_t strides[4] = {64, 256, 1024, 8192};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    for (int sh = 1; sh <= 7; sh++) {
        const cuuint32_t box[5] = {(cuuint32_t)(2 * ((sh & 1) ? R : 4)), (cuuint32_t)((sh & 2) ? R : 4),
                                   (cuuint32_t)((sh & 4) ? R : 4), 8, 8};
        CUresult r = encode(&maps[sh - 1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, lv.d_pref, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(h, OCTO_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    }
    CU(cudaMalloc(&lv.d_tmaps, sizeof(maps)));
    CU(cudaMemcpyAsync(lv.d_tmaps, maps, sizeof(maps), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));   // maps is a stack buffer
    return OCTO_OK;
}

static void free_level(Level &lv)
{
    void *ptrs[] = {lv.d_ijk, lv.d_nb, lv.d_kind, lv.d_rslot, lv.d_oslot, lv.d_use, lv.d_rnode, lv.d_mass, lv.d_pref,
                    lv.d_tmaps,
                    lv.d_L, lv.d_Lc, lv.d_in_mono, lv.d_in_com, lv.d_in_mom, lv.d_work_ref, lv.d_work_leaf,
                    lv.d_work_mixed, lv.d_msort, lv.d_ordslot, lv.d_gbuf};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    octo::exchange_free_level(lv);
    lv = Level();
}

extern "C" int octo_fmm_destroy(octo_fmm_t h)
{
    if (!h) return OCTO_EINVAL;
    cudaSetDevice(h->cfg.device);
    for (auto &lv : h->levels) free_level(lv);
    if (h->d_elist) cudaFree(h->d_elist);
    if (h->d_ecount) cudaFree(h->d_ecount);
    if (h->d_efar) cudaFree(h->d_efar);
    if (h->d_rows) cudaFree(h->d_rows);
    if (h->d_emask) cudaFree(h->d_emask);
    if (h->d_dlist) cudaFree(h->d_dlist);
    if (h->d_mstart) cudaFree(h->d_mstart);
    if (h->d_mitem) cudaFree(h->d_mitem);
    if (h->d_levels) cudaFree(h->d_levels);
    if (h->d_err) cudaFree(h->d_err);
    if (h->d_p2pk) cudaFree(h->d_p2pk);
    for (auto &a : h->all_work)
        if (a.ptr) cudaFree(a.ptr);
    for (auto &ev : h->ev_pending)
        for (auto e : ev) h->ev_pool.push_back(e);
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->m2l_stream) cudaStreamDestroy(h->m2l_stream);
    if (h->root_stream) cudaStreamDestroy(h->root_stream);
    if (h->ev_rfork) cudaEventDestroy(h->ev_rfork);
    if (h->ev_rjoin) cudaEventDestroy(h->ev_rjoin);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    for (auto &xe : h->xev_pending)
        for (auto e : xe) cudaEventDestroy(e);
    cudaEvent_t evs[] = {h->ev_packed, h->ev_recv};
    for (auto e : evs)
        if (e) cudaEventDestroy(e);

    octo::exchange_destroy(h);
    delete h;
    return OCTO_OK;
}

// ---------------------------------------------------------------------------
// load_level
// ---------------------------------------------------------------------------
template <class T>
static bool same_vec(const std::vector<T> &a, const T *b, size_t n)
{
    return a.size() == n && (n == 0 || std::memcmp(a.data(), b, n * sizeof(T)) == 0);
}

// Warp orientation of a node's M2L/mixed work (kernels.cuh orient_target):
// split the parity classes along the axis that crosses most of the
// interface to the other node kind (refined neighbours for the mixed kernel,
// leaf neighbours for the refined kernel's near list), weighting face
// neighbours 16, edges 4, corners 1; z when there is none.
static int orientation(const int32_t *nb27, const uint8_t *refined, bool want_refined)
{
    double w[3] = {0, 0, 0};
    for (int s = 0; s < 27; s++) {
        if (s == 13 || nb27[s] < 0) continue;
        if ((refined[nb27[s]] != 0) != want_refined) continue;
        const int o[3] = {s % 3 - 1, (s / 3) % 3 - 1, s / 9 - 1};
        const int nz = (o[0] != 0) + (o[1] != 0) + (o[2] != 0);
        const double wt = nz == 1 ? 16.0 : (nz == 2 ? 4.0 : 1.0);
        for (int a = 0; a < 3; a++)
            if (o[a]) w[a] += wt;
    }
    int best = 2;
    for (int a = 0; a < 3; a++)
        if (w[a] > w[best]) best = a;
    return best;
}

static int set_structure(octo_fmm *h, Level &lv, int32_t level, int64_t n, const int32_t *ijk, const uint8_t *refined,
                         const int32_t *nb, const int32_t *owner, cudaStream_t st)
{
    const int rank = h->cfg.rank;
    // ---- validation (host)
    const int64_t lim = (int64_t)1 << level;
    for (int64_t q = 0; q < n; q++) {
        for (int a = 0; a < 3; a++)
            if (ijk[3 * q + a] < 0 || ijk[3 * q + a] >= lim) return fail(h, OCTO_EINVAL, "node_ijk out of the level's domain");
        if (refined[q] > 1) return fail(h, OCTO_EINVAL, "refined flag must be 0 or 1");
        if (owner && (owner[q] < 0 || owner[q] >= h->cfg.nranks)) return fail(h, OCTO_EINVAL, "owner out of range");
        if (nb[q * 27 + 13] != q) return fail(h, OCTO_ESTRUCT, "neighbors[q][13] must be q");
        for (int s = 0; s < 27; s++) {
            const int32_t r = nb[q * 27 + s];
            const int ox = s % 3 - 1, oy = (s / 3) % 3 - 1, oz = s / 9 - 1;
            if (r < -1 || r >= n) return fail(h, OCTO_ESTRUCT, "neighbour index out of range");
            if (r >= 0) {
                if (nb[(int64_t)r * 27 + (26 - s)] != q) return fail(h, OCTO_ESTRUCT, "asymmetric neighbour table");
                if (ijk[3 * r] != ijk[3 * q] + ox || ijk[3 * r + 1] != ijk[3 * q + 1] + oy || ijk[3 * r + 2] != ijk[3 * q + 2] + oz)
                    return fail(h, OCTO_ESTRUCT, "neighbour coordinates do not match the slot");
            } else if (refined[q]) {
                const int64_t x = ijk[3 * q] + ox, y = ijk[3 * q + 1] + oy, z = ijk[3 * q + 2] + oz;
                const bool inside = x >= 0 && x < lim && y >= 0 && y < lim && z >= 0 && z < lim;
                const bool mine = !owner || owner[q] == rank;
                if (inside && mine) return fail(h, OCTO_ESTRUCT, "refined node with an absent in-domain neighbour (2:1 grading)");
            }
        }
    }
    // ---- host structure
    free_level(lv);
    lv.level = level;
    lv.n = n;
    lv.ijk.assign(ijk, ijk + 3 * n);
    lv.refined.assign(refined, refined + n);
    lv.nb.assign(nb, nb + 27 * n);
    if (owner) lv.owner.assign(owner, owner + n); else lv.owner.assign(n, rank);
    std::vector<uint8_t> kind(n), use(n);
    std::vector<int32_t> rslot(n, -1), oslot(n, -1), rnode;
    int64_t n_own_ref = 0;
    for (int64_t q = 0; q < n; q++) {
        kind[q] = refined[q] ? 2 : 1;
        if (refined[q]) { rslot[q] = (int32_t)rnode.size(); rnode.push_back((int32_t)q); }
        use[q] = (lv.owner[q] == rank);
        if (use[q] && refined[q]) n_own_ref++;
    }
    // output slots: owned refined nodes first, then owned leaf nodes
    std::vector<int32_t> ordslot;
    int64_t ir = 0, il = n_own_ref;
    for (int64_t q = 0; q < n; q++)
        if (use[q]) {
            oslot[q] = (int32_t)(refined[q] ? ir++ : il++);
            ordslot.push_back(oslot[q]);
        }
    lv.n_owned = il;
    lv.c_nref = n_own_ref;
    lv.c_nleaf = il - n_own_ref;
    lv.nr = (int64_t)rnode.size();
    lv.rnode = rnode;
    lv.oslot = oslot;
    lv.ordslot = ordslot;
    auto runs = [](const std::vector<int64_t> &v) {
        std::vector<std::pair<int64_t, int64_t>> r;
        for (int64_t x : v) {
            if (!r.empty() && r.back().second == x) r.back().second = x + 1;
            else r.push_back({x, x + 1});
        }
        return r;
    };
    {
        std::vector<int64_t> on, orr;
        for (int64_t q = 0; q < n; q++)
            if (use[q]) {
                on.push_back(q);
                if (refined[q]) orr.push_back(rslot[q]);
            }
        lv.own_runs = runs(on);
        lv.own_rruns = runs(orr);
    }
    // ---- work lists + interaction counts (per-slot table, build_stencil)
    std::vector<int2> wr, wl, wm, wrb, wlb, wmb;   // interior / boundary (a ghost neighbour)
    std::vector<float> cr, cl, crb, clb;           // per-item cost (interaction count)
    lv.counts[0] = lv.counts[1] = lv.counts[2] = 0;
    for (int64_t q = 0; q < n; q++) {
        if (!use[q]) continue;
        bool any_ref = false;
        int64_t c_ref = 0, c_p2p = 0;
        for (int s = 0; s < 27; s++) {
            const int32_t r = nb[q * 27 + s];
            if (r < 0) continue;
            const int64_t nf = h->slot_count[s][0], nn = h->slot_count[s][1];
            if (refined[q]) c_ref += nf + (refined[r] ? 0 : nn);
            else if (refined[r]) { lv.counts[2] += nf + nn; any_ref = true; }
            else c_p2p += nf + nn;
        }
        lv.counts[1] += c_ref;
        lv.counts[0] += c_p2p;
        if (level == 0) continue;   // the root has its own kernel (no parent criterion)
        bool bnd = false;
        for (int s = 0; s < 27; s++) {
            const int32_t r = nb[q * 27 + s];
            if (r >= 0 && lv.owner[r] != rank) bnd = true;
        }
        const int2 it = make_int2(level, (int)q);
        if (!refined[q] && any_ref) kind[q] |= 4;   // P2P adds onto the mixed result
        if (refined[q]) {
            (bnd ? wrb : wr).push_back(make_int2(level | (orientation(nb + q * 27, refined, false) << 8), (int)q));
            (bnd ? crb : cr).push_back((float)c_ref);
        } else {
            (bnd ? wlb : wl).push_back(it);
            (bnd ? clb : cl).push_back((float)c_p2p);
            if (any_ref) (bnd ? wmb : wm).push_back(it);
        }
    }
    if (level == 0 && lv.n_owned > 0) {
        // C2: refined root -> far pairs (|d|^2 >= R^2) by M2L; leaf root -> all pairs by P2P
        lv.counts[0] = lv.counts[1] = lv.counts[2] = 0;
        const double r = 1.0 / h->cfg.theta, R2 = r * r;
        for (int i = 0; i < NC; i++)
            for (int j = 0; j < NC; j++) {
                const int dx = (j & 7) - (i & 7), dy = ((j >> 3) & 7) - ((i >> 3) & 7), dz = (j >> 6) - (i >> 6);
                const int d2 = dx * dx + dy * dy + dz * dz;
                if (d2 == 0) continue;
                if (!refined[0]) lv.counts[0]++;
                else if ((double)d2 >= R2) lv.counts[1]++;
            }
    }
    // mixed nodes: their cells sorted by mixed work (sum of the refined slots'
    // list lengths), descending, so the lanes of a warp get similar trip counts;
    // one work item per CTA (node, quarter) with the CTA's cost = the sum over
    // its warps of the heaviest lane (every quarter runs: the mixed kernel
    // writes all rows of the node, which P2P then adds onto)
    std::vector<int16_t> msort((size_t)n * NC, 0);
    std::vector<int2> wmc, wmbc;
    std::vector<float> cm, cmb;
    for (int b = 0; b < 2; b++)
        for (const int2 &it : (b ? wmb : wm)) {
            const int64_t q = it.y;
            std::vector<std::pair<int, int>> len(NC);
            for (int l = 0; l < NC; l++) {
                int tot = 0;
                for (int s = 0; s < 27; s++) {
                    const int32_t r = nb[q * 27 + s];
                    if (r >= 0 && refined[r]) tot += h->mstart[l * 28 + s + 1] - h->mstart[l * 28 + s];
                }
                len[l] = {-tot, l};
            }
            std::stable_sort(len.begin(), len.end());
            for (int l = 0; l < NC; l++) msort[(size_t)q * NC + l] = (int16_t)len[l].second;
            for (int sub = 0; sub < MIX_CTAS_PER_NODE; sub++) {
                float c = 0.f;
                for (int w = 0; w < MIX_THREADS / 32; w++) c += (float)-len[sub * MIX_THREADS + 32 * w].first;
                (b ? wmbc : wmc).push_back(make_int2(it.x | (sub << 8), it.y));
                (b ? cmb : cm).push_back(c);
            }
        }
    // longest-processing-time-first order inside the interior and boundary groups
    auto lpt = [&](std::vector<int2> &w, std::vector<float> &c, int bit) {
        if (!(h->lpt_mask & bit)) return;
        std::vector<int> o(w.size());
        for (size_t i = 0; i < o.size(); i++) o[i] = (int)i;
        std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return c[a] > c[b]; });
        std::vector<int2> w2(w.size());
        std::vector<float> c2(w.size());
        for (size_t i = 0; i < o.size(); i++) { w2[i] = w[o[i]]; c2[i] = c[o[i]]; }
        w.swap(w2); c.swap(c2);
    };
    lpt(wr, cr, 1); lpt(wrb, crb, 1); lpt(wl, cl, 2); lpt(wlb, clb, 2); lpt(wmc, cm, 4); lpt(wmbc, cmb, 4);
    wm.swap(wmc); wmb.swap(wmbc);
    lv.nint[0] = (int)wr.size(); lv.nint[1] = (int)wl.size(); lv.nint[2] = (int)wm.size();
    wr.insert(wr.end(), wrb.begin(), wrb.end());
    wl.insert(wl.end(), wlb.begin(), wlb.end());
    wm.insert(wm.end(), wmb.begin(), wmb.end());
    cr.insert(cr.end(), crb.begin(), crb.end());
    cl.insert(cl.end(), clb.begin(), clb.end());
    cm.insert(cm.end(), cmb.begin(), cmb.end());
    lv.work_ref = wr; lv.work_leaf = wl; lv.work_mixed = wm;
    lv.cost_ref = cr; lv.cost_leaf = cl; lv.cost_mixed = cm;
    // ---- device structure
    auto up = [&](void **d, const void *src, size_t bytes) -> int {
        if (bytes == 0) { *d = nullptr; return OCTO_OK; }
        CU(cudaMalloc(d, bytes));
        CU(cudaMemcpyAsync(*d, src, bytes, cudaMemcpyHostToDevice, st));
        return OCTO_OK;
    };
    int rc;
    if ((rc = up((void **)&lv.d_ijk, ijk, 12 * n))) return rc;
    if ((rc = up((void **)&lv.d_nb, nb, 108 * n))) return rc;
    if ((rc = up((void **)&lv.d_kind, kind.data(), n))) return rc;
    if ((rc = up((void **)&lv.d_use, use.data(), n))) return rc;
    if ((rc = up((void **)&lv.d_rslot, rslot.data(), 4 * n))) return rc;
    if ((rc = up((void **)&lv.d_oslot, oslot.data(), 4 * n))) return rc;
    if ((rc = up((void **)&lv.d_ordslot, ordslot.data(), 4 * ordslot.size()))) return rc;
    if ((rc = up((void **)&lv.d_rnode, rnode.data(), 4 * rnode.size()))) return rc;
    if ((rc = up((void **)&lv.d_work_ref, wr.data(), sizeof(int2) * wr.size()))) return rc;
    if ((rc = up((void **)&lv.d_work_leaf, wl.data(), sizeof(int2) * wl.size()))) return rc;
    if ((rc = up((void **)&lv.d_work_mixed, wm.data(), sizeof(int2) * wm.size()))) return rc;
    if ((rc = up((void **)&lv.d_msort, msort.data(), sizeof(int16_t) * msort.size()))) return rc;
    CU(cudaMalloc(&lv.d_mass, sizeof(double) * NC * (n > 0 ? n : 1)));
    CU(cudaMemsetAsync(lv.d_mass, 0, sizeof(double) * NC * (n > 0 ? n : 1), st));
    if (lv.nr) {
        CU(cudaMalloc(&lv.d_pref, sizeof(double) * NC * NREC * lv.nr));
        CU(cudaMemsetAsync(lv.d_pref, 0, sizeof(double) * NC * NREC * lv.nr, st));
        if ((rc = make_tmaps(h, lv, st))) return rc;
    }
    // Taylor rows 0..3 for every owned slot, rows 4..19 for the owned refined
    // slots only (a leaf node keeps L0, L1 and Lc: 7 rows, not 23)
    const int64_t no = lv.n_owned > 0 ? lv.n_owned : 1;
    const size_t lrows = (size_t)4 * no + (size_t)16 * lv.c_nref;
    CU(cudaMalloc(&lv.d_L, sizeof(double) * NC * lrows));
    CU(cudaMalloc(&lv.d_Lc, sizeof(double) * NC * 3 * no));
    CU(cudaMemsetAsync(lv.d_L, 0, sizeof(double) * NC * lrows, st));
    CU(cudaMemsetAsync(lv.d_Lc, 0, sizeof(double) * NC * 3 * no, st));
    lv.loaded = true;
    h->generation++;
    if (h->cfg.nranks > 1) {
        rc = octo::exchange_plan_level(h, lv, st);
        if (rc) return rc;
    }
    return OCTO_OK;
}

static LevelDesc make_desc(const octo_fmm *h, const Level &lv, double hc, const double *origin)
{
    LevelDesc d{};
    d.ijk = lv.d_ijk; d.nb = lv.d_nb; d.kind = lv.d_kind; d.rslot = lv.d_rslot; d.oslot = lv.d_oslot;
    d.mass = lv.d_mass; d.pref = lv.d_pref; d.L = lv.d_L; d.Lc = lv.d_Lc; d.msort = lv.d_msort; d.tmaps = lv.d_tmaps;
    d.Lhi = lv.d_L + 4 * lv.n_owned * NC;
    d.n_owned = lv.n_owned; d.n_oref = lv.c_nref; d.h = hc; d.ox = origin[0]; d.oy = origin[1]; d.oz = origin[2]; d.G = h->cfg.G;
    return d;
}

extern "C" int octo_fmm_load_level(octo_fmm_t h, int32_t level, double h_cell, const double origin[3], int64_t n_nodes,
                                   const int32_t *node_ijk, const uint8_t *refined, const int32_t *neighbors,
                                   const int32_t *owner, const double *mono, const double *com, const double *mom,
                                   int32_t mem, void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    if (level < 0 || level >= MAX_LEVELS) return fail(h, OCTO_EINVAL, "level out of range");
    if (level == 0 && n_nodes != 1) return fail(h, OCTO_EINVAL, "the root level holds exactly one node");
    if (!(h_cell > 0.0) || !origin || n_nodes < 0 || (n_nodes > 0 && (!node_ijk || !refined || !neighbors || !mono)))
        return fail(h, OCTO_EINVAL, "null or invalid argument");
    if (mem != OCTO_HOST && mem != OCTO_DEVICE) return fail(h, OCTO_EINVAL, "mem must be OCTO_HOST or OCTO_DEVICE");
    CU(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    if ((int)h->levels.size() <= level) h->levels.resize(level + 1);
    Level &lv = h->levels[level];
    int rc;
    const bool same = lv.loaded && lv.n == n_nodes && same_vec(lv.ijk, node_ijk, 3 * n_nodes) &&
                      same_vec(lv.refined, refined, n_nodes) && same_vec(lv.nb, neighbors, 27 * n_nodes) &&
                      (owner ? same_vec(lv.owner, owner, n_nodes)
                             : std::all_of(lv.owner.begin(), lv.owner.end(), [&](int32_t o) { return o == h->cfg.rank; }));
    if (!same) {
        if ((rc = set_structure(h, lv, level, n_nodes, node_ijk, refined, neighbors, owner, st))) return rc;
    }
    const int64_t n = n_nodes, nr = lv.nr;
    if (nr > 0 && (!com || !mom)) return fail(h, OCTO_EINVAL, "com/mom required for refined nodes");
    // ---- data
    const double *dmono = mono, *dcom = com, *dmom = mom;
    if (mem == OCTO_HOST) {
        // values (m > 0, mom[0] == mono) are validated by the ingest kernel and
        // reported by the next synchronising call, as for device inputs
        // only the owned rows are ingested (ghost rows come from the exchange),
        // so only they cross PCIe: one copy per run of owned nodes / refined slots
        if (!lv.d_in_mono) CU(cudaMalloc(&lv.d_in_mono, sizeof(double) * NC * (n > 0 ? n : 1)));
        lv.h2d_bytes = 0;
        for (auto &r : lv.own_runs) {
            const size_t off = (size_t)r.first * NC, len = (size_t)(r.second - r.first) * NC;
            CU(cudaMemcpyAsync(lv.d_in_mono + off, mono + off, sizeof(double) * len, cudaMemcpyHostToDevice, st));
            lv.h2d_bytes += sizeof(double) * len;
        }
        if (nr) {
            if (!lv.d_in_com) CU(cudaMalloc(&lv.d_in_com, sizeof(double) * NC * 3 * nr));
            if (!lv.d_in_mom) CU(cudaMalloc(&lv.d_in_mom, sizeof(double) * NC * 20 * nr));
            const size_t pitch = sizeof(double) * NC * nr;
            // mom rows 1..3 (the dipole about the centre of mass) are ignored by
            // contract (identically 0): row 0 (checked against mono) and rows 4..19 cross PCIe
            const size_t row = (size_t)NC * nr;   // elements per mom row
            for (auto &r : lv.own_rruns) {
                const size_t off = (size_t)r.first * NC, w = sizeof(double) * (r.second - r.first) * NC;
                CU(cudaMemcpy2DAsync(lv.d_in_com + off, pitch, com + off, pitch, w, 3, cudaMemcpyHostToDevice, st));
                CU(cudaMemcpyAsync(lv.d_in_mom + off, mom + off, w, cudaMemcpyHostToDevice, st));
                CU(cudaMemcpy2DAsync(lv.d_in_mom + 4 * row + off, pitch, mom + 4 * row + off, pitch, w, 16,
                                     cudaMemcpyHostToDevice, st));
                lv.h2d_bytes += 20 * w;
            }
        }
        dmono = lv.d_in_mono; dcom = lv.d_in_com; dmom = lv.d_in_mom;
    } else {
        lv.h2d_bytes = 0;
    }
    // ingest is batched: one prep launch for every level loaded since the last
    // compute call (flush_prep, at the start of compute_interactions)
    lv.src_mono = dmono; lv.src_com = dcom; lv.src_mom = dmom;
    lv.prep_pending = true;
    CU(cudaGetLastError());
    lv.hc = h_cell;
    lv.origin[0] = origin[0]; lv.origin[1] = origin[1]; lv.origin[2] = origin[2];
    // the device descriptor changes only with the structure (buffers) or the
    // geometry: re-loading a level's data every step (the bench, a time
    // loop) then costs no host->device copy beyond the data itself
    const LevelDesc d = make_desc(h, lv, h_cell, origin);
    if (!lv.desc_valid || std::memcmp(&d, &lv.desc, sizeof(LevelDesc)) != 0) {
        lv.desc = d;
        CU(cudaMemcpyAsync(h->d_levels + level, &lv.desc, sizeof(LevelDesc), cudaMemcpyHostToDevice, st));
        lv.desc_valid = true;
    }
    lv.data_ready = true;
    return OCTO_OK;
}

// ---------------------------------------------------------------------------
// compute
// ---------------------------------------------------------------------------
// Kernel launch through cudaLaunchKernelEx (one launch path for every level
// kernel).  Programmatic dependent launch (overlapping a kernel's tail with
// the next kernel) was measured slower here: co-resident leaf-kernel CTAs
// take SM slots from the M2L kernel (6.65 vs 6.14 ms per configs[3] step).
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*k)(KArgs...), dim3 g, dim3 b, size_t sm, cudaStream_t st, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Kernel schedule of one compute call, stream-ordered on the caller's stream:
// M2L (refined targets), mixed (leaf targets <- refined partners, writes),
// P2P (leaf targets <- leaf partners, adds onto the mixed rows), so every
// cell's sum has a fixed order.  (Running the leaf kernels on a side stream
// concurrently with M2L was measured: no gain -- all three are FP64-pipe
// bound -- and it blurs the per-kernel timing.)
// One round of the three kernels.  With concurrency on, M2L runs on a
// higher-priority stream beside the leaf kernels (mixed, then P2P) on the
// caller's stream: `first` forks the M2L stream from the caller's stream,
// `dep` (if set) is waited for by both streams, `last` joins them again.
static int launch_work(octo_fmm *h, const int2 *w_ref, int n_ref, const int2 *w_leaf, int n_leaf, const int2 *w_mix,
                       int n_mix, cudaStream_t st, bool first = true, bool last = true, cudaEvent_t dep = nullptr)
{
    const bool am = (h->cfg.flags & OCTO_AM_CORRECTION) != 0;
    const bool timing = (h->cfg.flags & OCTO_TIMING) != 0;
    std::array<cudaEvent_t, 6> ev{};
    if (timing) {
        for (int k = 0; k < 6; k++) {
            if (h->ev_pool.empty()) {
                cudaEvent_t e;
                CU(cudaEventCreate(&e));
                h->ev_pool.push_back(e);
            }
            ev[k] = h->ev_pool.back();
            h->ev_pool.pop_back();
        }
    }
    // M2L on a higher-priority stream when leaf work runs beside it: its CTAs
    // are dispatched first and the leaf kernels fill the SMs its tail leaves
    // idle (the split multi-rank step runs each kernel twice, so tails add up)
    const bool conc = h->concurrency > 0;
    cudaStream_t sm2l = st;
    if (conc) {
        if (!h->m2l_stream) {
            int lo = 0, hi = 0;
            CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CU(cudaStreamCreateWithPriority(&h->m2l_stream, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
            CU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        }
        sm2l = h->m2l_stream;
        if (first) {
            CU(cudaEventRecord(h->ev_fork, st));
            CU(cudaStreamWaitEvent(sm2l, h->ev_fork, 0));
        }
        if (dep) CU(cudaStreamWaitEvent(sm2l, dep, 0));
    }
    if (dep) CU(cudaStreamWaitEvent(st, dep, 0));
    const bool tk = timing;
    // ---- M2L + Lc, refined targets
    if (timing) CU(cudaEventRecord(ev[0], sm2l));
    if (n_ref > 0) {
        const dim3 g(n_ref * M2LD_CTAS_PER_NODE), b(M2LD_THREADS);
        const int *dl = h->d_dlist;
        const LevelDesc *L = h->d_levels;
        if (h->reach == 3) {
            const size_t sm = sizeof(M2LDSmem<3>);
            if (am) CU(launch_k(m2l_dense_kernel<true, 1, 3>, g, b, sm, sm2l, L, w_ref, dl, h->d_ecount, h->d_efar, h->d_emask));
            else CU(launch_k(m2l_dense_kernel<false, 1, 3>, g, b, sm, sm2l, L, w_ref, dl, h->d_ecount, h->d_efar, h->d_emask));
        } else {
            const size_t sm = sizeof(M2LDSmem<2>);
            auto k = m2l_dense_kernel<false, 1, 2>;
            if (am && h->m2l_unroll == 2) k = m2l_dense_kernel<true, 2, 2>;
#ifdef M2L_U4
            else if (am && h->m2l_unroll >= 4) k = m2l_dense_kernel<true, 4, 2>;
#endif
            else if (am && h->m2l_unroll >= 3) k = m2l_dense_kernel<true, 3, 2>;
            else if (am) k = m2l_dense_kernel<true, 1, 2>;
            CU(launch_k(k, g, b, sm, sm2l, L, w_ref, dl, h->d_ecount, h->d_efar, h->d_emask));
        }
        h->launches++;
    }
    if (tk) CU(cudaEventRecord(ev[1], sm2l));
    cudaStream_t sd = st;
    // ---- mixed then P2P, leaf targets
    if (tk) CU(cudaEventRecord(ev[2], sd));
    if (n_mix > 0) {
        auto mk = h->reach == 3 ? (am ? m2l_mixed_kernel<true, 3, false> : m2l_mixed_kernel<false, 3, false>)
                                : (am ? m2l_mixed_kernel<true, 2, false> : m2l_mixed_kernel<false, 2, false>);
        size_t msm = sizeof(MixSmem<false>);
        if (h->mix_tma) {   // TMA-staged halo boxes (measured slower than the L1 gather: DESIGN.md)
            mk = h->reach == 3 ? (am ? m2l_mixed_kernel<true, 3, true> : m2l_mixed_kernel<false, 3, true>)
                               : (am ? m2l_mixed_kernel<true, 2, true> : m2l_mixed_kernel<false, 2, true>);
            msm = sizeof(MixSmem<true>);
        }
        CU(launch_k(mk, dim3(n_mix), dim3(MIX_THREADS), msm, sd, h->d_levels, w_mix, h->d_mstart, h->d_mitem));
        h->launches++;
    }
    if (tk) CU(cudaEventRecord(ev[3], sd));
    if (tk) CU(cudaEventRecord(ev[4], sd));
    if (n_leaf > 0) {
        const int nrw = (int)h->rows.size(), nb = (n_leaf + 1) / 2;
        if (h->reach == 3)
            CU(launch_k(h->p2p8 ? p2p8_kernel<3> : p2p_kernel<3>, dim3(nb), dim3(P2P_THREADS), sizeof(P2PSmem<3>), sd,
                        h->d_levels, w_leaf, n_leaf, h->d_rows, nrw, (const double4 *)h->d_p2pk));
        else
            CU(launch_k(h->p2p8 ? p2p8_kernel<2> : p2p_kernel<2>, dim3(nb), dim3(P2P_THREADS), sizeof(P2PSmem<2>), sd,
                        h->d_levels, w_leaf, n_leaf, h->d_rows, nrw, (const double4 *)nullptr));
        h->launches++;
    }
    if (timing) CU(cudaEventRecord(ev[5], sd));
    if (conc && last) {
        CU(cudaEventRecord(h->ev_join, sm2l));
        CU(cudaStreamWaitEvent(sd, h->ev_join, 0));
    }
    if (timing) h->ev_pending.push_back(ev);
    CU(cudaGetLastError());
    return OCTO_OK;
}

static int build_all_work(octo_fmm *h, cudaStream_t st)
{
    if (h->all_gen == h->generation) return OCTO_OK;
    // all levels in one launch per kernel: interior items of every level, then
    // boundary items, each group in longest-processing-time-first order
    std::vector<std::pair<float, int2>> gv[3], gb[3];
    for (auto &lv : h->levels) {
        if (!lv.loaded) continue;
        const std::vector<int2> *src[3] = {&lv.work_ref, &lv.work_leaf, &lv.work_mixed};
        const std::vector<float> *cst[3] = {&lv.cost_ref, &lv.cost_leaf, &lv.cost_mixed};
        for (int k = 0; k < 3; k++)
            for (size_t i = 0; i < src[k]->size(); i++)
                ((int)i < lv.nint[k] ? gv[k] : gb[k]).push_back({(*cst[k])[i], (*src[k])[i]});
    }
    std::vector<int2> v[3], b[3];
    for (int k = 0; k < 3; k++) {
        auto cmp = [](const std::pair<float, int2> &x, const std::pair<float, int2> &y) { return x.first > y.first; };
        const int bit = k == 0 ? 1 : k == 1 ? 2 : 4;
        if (h->lpt_mask & bit) {
            std::stable_sort(gv[k].begin(), gv[k].end(), cmp);
            std::stable_sort(gb[k].begin(), gb[k].end(), cmp);
        }
        for (auto &e : gv[k]) v[k].push_back(e.second);
        for (auto &e : gb[k]) b[k].push_back(e.second);
    }
    for (int k = 0; k < 3; k++) {
        auto &a = h->all_work[k];
        if (a.ptr) cudaFree(a.ptr);
        a.ptr = nullptr;
        a.nint = (int)v[k].size();
        v[k].insert(v[k].end(), b[k].begin(), b[k].end());
        a.n = (int)v[k].size();
        if (a.n) {
            CU(cudaMalloc(&a.ptr, sizeof(int2) * a.n));
            CU(cudaMemcpyAsync(a.ptr, v[k].data(), sizeof(int2) * a.n, cudaMemcpyHostToDevice, st));
        }
    }
    h->all_gen = h->generation;
    return OCTO_OK;
}

static int flush_prep(octo_fmm *h, cudaStream_t st)
{
    PrepBatch b{};
    int k = 0;
    int64_t maxcells = 0;
    auto launch = [&]() -> int {
        if (k == 0) return OCTO_OK;
        const unsigned gx = (unsigned)std::min<int64_t>((maxcells + 255) / 256, 148 * 8);
        prep_batch_kernel<<<dim3(gx, k), 256, 0, st>>>(b, h->d_err);
        h->launches++;
        CU(cudaGetLastError());
        k = 0;
        maxcells = 0;
        return OCTO_OK;
    };
    int rc;
    for (auto &lv : h->levels) {
        if (!lv.loaded || !lv.prep_pending) continue;
        lv.prep_pending = false;
        if (lv.n == 0) continue;
        PrepDesc &d = b.d[k++];
        d.mono = lv.src_mono; d.com = lv.src_com; d.mom = lv.src_mom;
        d.mass = lv.d_mass; d.pref = lv.d_pref; d.rnode = lv.d_rnode; d.use = lv.d_use;
        d.n = lv.n; d.nr = lv.nr;
        maxcells = std::max<int64_t>(maxcells, std::max(lv.n, lv.nr) * NC);
        if (k == PREP_MAX && (rc = launch())) return rc;
    }
    return launch();
}

// The root (one sub-grid, 16 CTAs, latency-bound) runs on a side stream
// beside the level kernels instead of ahead of them; *joined tells the
// caller to make its stream wait for h->ev_rjoin at the end.
static int launch_root(octo_fmm *h, cudaStream_t st, bool *joined = nullptr)
{
    const Level &lv = h->levels[0];
    if (lv.n_owned == 0) return OCTO_OK;
    if (joined) {
        if (!h->root_stream) {
            CU(cudaStreamCreateWithFlags(&h->root_stream, cudaStreamNonBlocking));
            CU(cudaEventCreateWithFlags(&h->ev_rfork, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&h->ev_rjoin, cudaEventDisableTiming));
        }
        CU(cudaEventRecord(h->ev_rfork, st));
        CU(cudaStreamWaitEvent(h->root_stream, h->ev_rfork, 0));
        st = h->root_stream;
        *joined = true;
    }
    const double r = 1.0 / h->cfg.theta, R2 = r * r;
    if (h->cfg.flags & OCTO_AM_CORRECTION)
        root_kernel<true><<<NC / 32, ROOT_THREADS, sizeof(RootSmem), st>>>(h->d_levels, R2);
    else
        root_kernel<false><<<NC / 32, ROOT_THREADS, sizeof(RootSmem), st>>>(h->d_levels, R2);
    h->launches++;
    CU(cudaGetLastError());
    if (joined) CU(cudaEventRecord(h->ev_rjoin, st));
    return OCTO_OK;
}

// Work of one compute call: interior nodes (no ghost neighbour) first, then
// boundary nodes.  With nranks > 1 the ghost exchange of the levels runs on
// the handle's communication stream, overlapped with the interior work; the
// boundary work waits for it.
static int compute_split(octo_fmm *h, std::vector<Level *> lvs, const int2 *w[3], const int n[3], const int nint[3],
                         bool root, cudaStream_t st)
{
    int rc;
    h->ncompute++;
    if ((rc = flush_prep(h, st))) return rc;
    // nranks > 1: every rank takes part in every exchange (collective-safe
    // even for a rank with no peer at this level) over ALL loaded levels, so
    // one plan serves per-level and all-level calls alike
    const bool xchg = h->cfg.nranks > 1;
    if (xchg) {
        lvs.clear();
        for (auto &l : h->levels)
            if (l.loaded) lvs.push_back(&l);
        if (!h->comm_stream) {
            // highest priority: the NCCL kernels get the first SMs that free up
            // while the interior work runs
            int lo = 0, hi = 0;
            CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CU(cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, hi));
            CU(cudaEventCreateWithFlags(&h->ev_packed, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&h->ev_recv, cudaEventDisableTiming));
        }
        if ((rc = octo::exchange_pack(h, lvs, st))) return rc;
        CU(cudaEventRecord(h->ev_packed, st));
        CU(cudaStreamWaitEvent(h->comm_stream, h->ev_packed, 0));
        std::array<cudaEvent_t, 2> xe{};
        if (h->cfg.flags & OCTO_TIMING) {
            for (int k = 0; k < 2; k++) {
                if (h->ev_pool.empty()) {
                    cudaEvent_t e;
                    CU(cudaEventCreate(&e));
                    h->ev_pool.push_back(e);
                }
                xe[k] = h->ev_pool.back();
                h->ev_pool.pop_back();
            }
            CU(cudaEventRecord(xe[0], h->comm_stream));
        }
        if ((rc = octo::exchange_sendrecv_unpack(h, lvs, h->comm_stream))) return rc;
        if (h->cfg.flags & OCTO_TIMING) {
            CU(cudaEventRecord(xe[1], h->comm_stream));
            h->xev_pending.push_back(xe);
        }
        CU(cudaEventRecord(h->ev_recv, h->comm_stream));
    }
    bool rjoin = false;
    const bool side = n[0] + n[1] + n[2] > 0;   // anything for the root to run beside
    if (root && (rc = launch_root(h, st, side ? &rjoin : nullptr))) return rc;
    if (!xchg) {
        rc = launch_work(h, w[0], n[0], w[1], n[1], w[2], n[2], st);
    } else if (h->xmode == 1) {
        // exchange first (only the root kernel beside it), then every node in one round
        CU(cudaStreamWaitEvent(st, h->ev_recv, 0));
        rc = launch_work(h, w[0], n[0], w[1], n[1], w[2], n[2], st);
    } else {
        rc = launch_work(h, w[0], nint[0], w[1], nint[1], w[2], nint[2], st, true, false);
        if (!rc)
            rc = launch_work(h, w[0] + nint[0], n[0] - nint[0], w[1] + nint[1], n[1] - nint[1], w[2] + nint[2],
                             n[2] - nint[2], st, false, true, h->ev_recv);
    }
    if (rc) return rc;
    if (rjoin) CU(cudaStreamWaitEvent(st, h->ev_rjoin, 0));
    return OCTO_OK;
}

extern "C" int octo_fmm_compute_interactions(octo_fmm_t h, int32_t level, void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    CU(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    int rc;
    if (level == OCTO_ALL_LEVELS) {
        std::vector<Level *> lvs;
        for (auto &lv : h->levels) {
            if (lv.loaded && !lv.data_ready) return fail(h, OCTO_EINVAL, "level has no data");
            if (lv.loaded) lvs.push_back(&lv);
        }
        if ((rc = build_all_work(h, st))) return rc;
        const int2 *w[3] = {h->all_work[0].ptr, h->all_work[1].ptr, h->all_work[2].ptr};
        const int n[3] = {h->all_work[0].n, h->all_work[1].n, h->all_work[2].n};
        const int ni[3] = {h->all_work[0].nint, h->all_work[1].nint, h->all_work[2].nint};
        const bool root = !h->levels.empty() && h->levels[0].loaded;
        return compute_split(h, lvs, w, n, ni, root, st);
    }
    if (level < 0 || level >= (int)h->levels.size() || !h->levels[level].loaded || !h->levels[level].data_ready)
        return fail(h, OCTO_EINVAL, "level not loaded");
    Level &lv = h->levels[level];
    const int2 *w[3] = {lv.d_work_ref, lv.d_work_leaf, lv.d_work_mixed};
    const int n[3] = {(int)lv.work_ref.size(), (int)lv.work_leaf.size(), (int)lv.work_mixed.size()};
    return compute_split(h, {&lv}, w, n, lv.nint, level == 0, st);
}

// node-order result rows: dst[k][j][l] = row k of slot ordslot[j], for the
// ncomp components of a slot-order array whose rows >= nlow exist only for
// the first n_hi slots (at hi[k - nlow][slot]); missing rows read as 0
__global__ void gather_rows_kernel(const double *__restrict__ src, const double *__restrict__ hi, int64_t n_owned,
                                   int64_t n_hi, int nlow, const int32_t *__restrict__ ordslot, int ncomp,
                                   double *__restrict__ dst)
{
    const int64_t rs = n_owned * NC, tot = (int64_t)ncomp * rs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / rs, r = i % rs;
        const int64_t slot = ordslot[r / NC], l = r % NC;
        double v = 0.0;
        if (k < nlow) v = src[k * rs + slot * NC + l];
        else if (slot < n_hi) v = hi[(k - nlow) * n_hi * NC + slot * NC + l];
        dst[i] = v;
    }
}

extern "C" int octo_fmm_get_expansions(octo_fmm_t h, int32_t level, double *taylor, double *ang_corr, int32_t mem,
                                       void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    if (level < 0 || level >= (int)h->levels.size() || !h->levels[level].loaded)
        return fail(h, OCTO_EINVAL, "level not loaded");
    if (mem != OCTO_HOST && mem != OCTO_DEVICE && mem != OCTO_HOST_ASYNC) return fail(h, OCTO_EINVAL, "bad mem");
    CU(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    Level &lv = h->levels[level];
    const int64_t no = lv.n_owned;
    if (no == 0) return mem == OCTO_HOST ? octo_fmm_sync(h, cuda_stream) : OCTO_OK;
    double *dt = taylor, *da = ang_corr;
    if (mem != OCTO_DEVICE) {   // gather into the staging buffer, then one copy each
        if (!lv.d_gbuf) CU(cudaMalloc(&lv.d_gbuf, sizeof(double) * NC * 23 * no));
        dt = lv.d_gbuf;
        da = lv.d_gbuf + 20 * no * NC;
    }
    if (taylor) {
        gather_rows_kernel<<<148 * 4, 256, 0, st>>>(lv.d_L, lv.d_L + 4 * no * NC, no, lv.c_nref, 4, lv.d_ordslot,
                                                    20, dt);
        h->launches++;
    }
    if (ang_corr) {
        gather_rows_kernel<<<148 * 4, 256, 0, st>>>(lv.d_Lc, nullptr, no, 0, 3, lv.d_ordslot, 3, da);
        h->launches++;
    }
    CU(cudaGetLastError());
    if (mem != OCTO_DEVICE) {
        if (taylor) CU(cudaMemcpyAsync(taylor, dt, sizeof(double) * NC * 20 * no, cudaMemcpyDeviceToHost, st));
        if (ang_corr) CU(cudaMemcpyAsync(ang_corr, da, sizeof(double) * NC * 3 * no, cudaMemcpyDeviceToHost, st));
        if (mem == OCTO_HOST) return octo_fmm_sync(h, cuda_stream);
    }
    return OCTO_OK;
}

extern "C" int octo_fmm_get_expansions_compact(octo_fmm_t h, int32_t level, double *refined_out, double *leaf_out,
                                               int64_t *n_ref, int64_t *n_leaf, int32_t mem, void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    if (level < 0 || level >= (int)h->levels.size() || !h->levels[level].loaded)
        return fail(h, OCTO_EINVAL, "level not loaded");
    if (mem != OCTO_HOST && mem != OCTO_DEVICE && mem != OCTO_HOST_ASYNC) return fail(h, OCTO_EINVAL, "bad mem");
    CU(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    Level &lv = h->levels[level];
    if (n_ref) *n_ref = lv.c_nref;
    if (n_leaf) *n_leaf = lv.c_nleaf;
    if (!refined_out && !leaf_out) return OCTO_OK;   // size query
    // the slot layout puts owned refined rows first: every block below is a
    // strided run of whole rows, moved by the copy engines (no kernel, so a
    // result copy never waits for SM slots behind other work)
    const cudaMemcpyKind kind = mem == OCTO_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const size_t sp = sizeof(double) * NC * lv.n_owned;
    auto copy = [&](double *dst, const double *src, int64_t rows, int comps) -> int {
        if (rows == 0 || comps == 0) return OCTO_OK;
        const size_t w = sizeof(double) * NC * rows;
        CU(cudaMemcpy2DAsync(dst, w, src, sp, w, comps, kind, st));
        return OCTO_OK;
    };
    int rc;
    const int64_t nr = lv.c_nref, nf = lv.c_nleaf;
    if (refined_out) {
        if ((rc = copy(refined_out, lv.d_L, nr, 4))) return rc;
        if (nr) CU(cudaMemcpyAsync(refined_out + 4 * nr * NC, lv.d_L + 4 * lv.n_owned * NC,
                                   sizeof(double) * NC * 16 * nr, kind, st));   // rows 4..19: one block
        if ((rc = copy(refined_out + 20 * nr * NC, lv.d_Lc, nr, 3))) return rc;
    }
    if (leaf_out) {
        if ((rc = copy(leaf_out, lv.d_L + nr * NC, nf, 4))) return rc;
        if ((rc = copy(leaf_out + 4 * nf * NC, lv.d_Lc + nr * NC, nf, 3))) return rc;
    }
    if (mem == OCTO_HOST) return octo_fmm_sync(h, cuda_stream);
    return OCTO_OK;
}

extern "C" int octo_fmm_expansions_ptr(octo_fmm_t h, int32_t level, const double **taylor, const double **ang_corr,
                                       int64_t *n_owned)
{
    if (!h) return OCTO_EINVAL;
    if (level < 0 || level >= (int)h->levels.size() || !h->levels[level].loaded)
        return fail(h, OCTO_EINVAL, "level not loaded");
    const Level &lv = h->levels[level];
    if (taylor) *taylor = lv.d_L;
    if (ang_corr) *ang_corr = lv.d_Lc;
    if (n_owned) *n_owned = lv.n_owned;
    return OCTO_OK;
}

extern "C" int octo_fmm_sync(octo_fmm_t h, void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    CU(cudaSetDevice(h->cfg.device));
    int rc = flush_prep(h, (cudaStream_t)cuda_stream);   // ingest (and validate) levels loaded since the last compute
    if (rc) return rc;
    CU(cudaStreamSynchronize((cudaStream_t)cuda_stream));
    int err = 0;
    CU(cudaMemcpy(&err, h->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
        CU(cudaMemset(h->d_err, 0, sizeof(int)));
        if (err & 4) return fail(h, OCTO_ENCCL, "ghost exchange: a peer's data did not arrive within 20 s");
        if (err & 1) return fail(h, OCTO_EMASS, "cell mass <= 0 (device-side check)");
        return fail(h, OCTO_EINVAL, "mom[0] != mono (device-side check)");
    }
    return OCTO_OK;
}

extern "C" int octo_fmm_stencil(octo_fmm_t h, int8_t *offsets, uint8_t *cls, int32_t *counts, int32_t capacity)
{
    if (!h || !counts) return OCTO_EINVAL;
    for (int c = 0; c < 8; c++) {
        const int cb[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
        int n = 0;
        for (int q = 0; q < 8; q++)
            for (int e = 0; e < h->ecount[c * 8 + q]; e++) {
                const int v = h->elist[(c * 8 + q) * MAXE + e];
                const int px = (int8_t)(v & 0xff), py = (int8_t)((v >> 8) & 0xff), pz = (int8_t)((v >> 16) & 0xff);
                if (offsets) {
                    if (n >= capacity) return fail(h, OCTO_EINVAL, "stencil capacity");
                    offsets[(c * capacity + n) * 3 + 0] = (int8_t)(2 * px + (q & 1) - cb[0]);
                    offsets[(c * capacity + n) * 3 + 1] = (int8_t)(2 * py + ((q >> 1) & 1) - cb[1]);
                    offsets[(c * capacity + n) * 3 + 2] = (int8_t)(2 * pz + ((q >> 2) & 1) - cb[2]);
                    if (cls) cls[c * capacity + n] = (uint8_t)(((v >> 24) & 1) ? 2 : 1);
                }
                n++;
            }
        counts[c] = n;
    }
    return OCTO_OK;
}

extern "C" int octo_fmm_kernel_times(octo_fmm_t h, double ms[4], int64_t *calls)
{
    if (!h || !ms) return OCTO_EINVAL;
    CU(cudaSetDevice(h->cfg.device));
    ms[0] = ms[1] = ms[2] = ms[3] = 0.0;
    for (auto &ev : h->ev_pending) {
        CU(cudaEventSynchronize(ev[5]));
        CU(cudaEventSynchronize(ev[1]));
        float t;
        CU(cudaEventElapsedTime(&t, ev[4], ev[5]));   // P2P
        ms[0] += t;
        CU(cudaEventElapsedTime(&t, ev[2], ev[3]));   // mixed
        ms[1] += t;
        CU(cudaEventElapsedTime(&t, ev[0], ev[1]));   // M2L
        ms[2] += t;
        for (int k = 0; k < 6; k++) h->ev_pool.push_back(ev[k]);
    }
    for (auto &xe : h->xev_pending) {   // ghost exchange (NCCL group + unpack, comm stream)
        float t = 0.f;
        CU(cudaEventSynchronize(xe[1]));
        CU(cudaEventElapsedTime(&t, xe[0], xe[1]));
        ms[3] += t;
        h->ev_pool.push_back(xe[0]);
        h->ev_pool.push_back(xe[1]);
    }
    if (calls) *calls = h->ncompute;
    h->ev_pending.clear();
    h->xev_pending.clear();
    h->ncompute = 0;
    return OCTO_OK;
}

extern "C" int octo_fmm_interaction_counts(octo_fmm_t h, int32_t level, int64_t counts[3])
{
    if (!h || !counts) return OCTO_EINVAL;
    counts[0] = counts[1] = counts[2] = 0;
    if (level == OCTO_ALL_LEVELS) {
        for (auto &lv : h->levels)
            if (lv.loaded)
                for (int k = 0; k < 3; k++) counts[k] += lv.counts[k];
        return OCTO_OK;
    }
    if (level < 0 || level >= (int)h->levels.size() || !h->levels[level].loaded) return OCTO_OK;
    for (int k = 0; k < 3; k++) counts[k] = h->levels[level].counts[k];
    return OCTO_OK;
}
