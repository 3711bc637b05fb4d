// downward.cu -- FMM step 3 on the device: L2L + field.
//
// "In the third FMM step, the gravitational influence of cells
// outside of the opening criteria is computed, and the octree is traversed
// top-down. The respective Taylor series expansion of the parent node is
// passed to the child nodes and accumulated."  Reading C8: every
// child cell adds its parent cell's expansion re-centred by the exact cubic
// Taylor shift to the child's expansion centre; the angular-momentum
// correction Lc is passed down unchanged.  Runs in place on the library's
// result buffers, level by level from the root down, so a parent's buffer
// already holds its own inherited part when its children read it.  Field
// (P:L468): Phi = L0, g = -(L1 + Lc) (G is already applied to L and Lc).
#include "internal.hpp"

#include <algorithm>
#include <cstring>

using namespace octo;

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            if (e_ == cudaErrorMemoryAllocation) return fail(h, OCTO_ENOMEM, #call);           \
            return fail(h, OCTO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
        }                                                                                      \
    } while (0)

// child cell c of child node (parent node pn, octant o): parent cell, shift
__global__ void __launch_bounds__(256) l2l_kernel(const LevelDesc *__restrict__ levels, int plev,
                                                  const int32_t *__restrict__ parent_of, int64_t n_child)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_child * NC) return;
    const LevelDesc &P = levels[plev];
    const LevelDesc &C = levels[plev + 1];
    const int64_t cn = i / NC;
    const int l = (int)(i % NC);
    const int pn = parent_of[cn];
    const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
    // child cell global coords -> parent cell local index in node pn
    const int gx = 8 * C.ijk[3 * cn] + lx, gy = 8 * C.ijk[3 * cn + 1] + ly, gz = 8 * C.ijk[3 * cn + 2] + lz;
    const int px = (gx >> 1) - 8 * P.ijk[3 * pn], py = (gy >> 1) - 8 * P.ijk[3 * pn + 1],
              pz = (gz >> 1) - 8 * P.ijk[3 * pn + 2];
    const int pq = (px & 1) + 2 * (py & 1) + 4 * (pz & 1), pp = (px >> 1) + 4 * (py >> 1) + 16 * (pz >> 1);
    const int pl = px + 8 * py + 64 * pz;
    const int64_t prs_ = P.rslot[pn];
    const double XP[3] = {P.pref[prec(prs_, 1, pq, pp)], P.pref[prec(prs_, 2, pq, pp)], P.pref[prec(prs_, 3, pq, pp)]};
    const int cq = (lx & 1) + 2 * (ly & 1) + 4 * (lz & 1), cp = (lx >> 1) + 4 * (ly >> 1) + 16 * (lz >> 1);
    double Y[3];
    if ((C.kind[cn] & 3) == 2) {
        const int64_t crs_ = C.rslot[cn];
        Y[0] = C.pref[prec(crs_, 1, cq, cp)]; Y[1] = C.pref[prec(crs_, 2, cq, cp)]; Y[2] = C.pref[prec(crs_, 3, cq, cp)];
    } else {
        Y[0] = C.ox + ((double)gx + 0.5) * C.h;
        Y[1] = C.oy + ((double)gy + 0.5) * C.h;
        Y[2] = C.oz + ((double)gz + 0.5) * C.h;
    }
    const double z0 = Y[0] - XP[0], z1 = Y[1] - XP[1], z2 = Y[2] - XP[2];
    const int64_t prs = P.n_owned * NC, crs = C.n_owned * NC, phs = P.n_oref * NC, chs = C.n_oref * NC;
    const double *Lp = P.L + (int64_t)P.oslot[pn] * NC + pl;
    const double *Hp = P.Lhi + (int64_t)P.oslot[pn] * NC + pl;   // the parent is refined
    double L[20];
#pragma unroll
    for (int k = 0; k < 4; k++) L[k] = Lp[k * prs];
#pragma unroll
    for (int k = 4; k < 20; k++) L[k] = Hp[(k - 4) * phs];
    // symmetric storage: 4 xx 5 xy 6 xz 7 yy 8 yz 9 zz ; 10 xxx 11 xxy 12 xxz 13 xyy 14 xyz 15 xzz 16 yyy 17 yyz 18 yzz 19 zzz
    const double zz[3] = {z0, z1, z2};
    // L3 . z (a 3x3 symmetric tensor T_ab = L_abc z_c)
    const double Txx = L[10] * z0 + L[11] * z1 + L[12] * z2;
    const double Txy = L[11] * z0 + L[13] * z1 + L[14] * z2;
    const double Txz = L[12] * z0 + L[14] * z1 + L[15] * z2;
    const double Tyy = L[13] * z0 + L[16] * z1 + L[17] * z2;
    const double Tyz = L[14] * z0 + L[17] * z1 + L[18] * z2;
    const double Tzz = L[15] * z0 + L[18] * z1 + L[19] * z2;
    // L2' = L2 + T
    const double M2[6] = {L[4] + Txx, L[5] + Txy, L[6] + Txz, L[7] + Tyy, L[8] + Tyz, L[9] + Tzz};
    // L1'_a = L1_a + L2_ab z_b + 1/2 T_ab z_b
    const double Hx = (L[4] + 0.5 * Txx) * z0 + (L[5] + 0.5 * Txy) * z1 + (L[6] + 0.5 * Txz) * z2;
    const double Hy = (L[5] + 0.5 * Txy) * z0 + (L[7] + 0.5 * Tyy) * z1 + (L[8] + 0.5 * Tyz) * z2;
    const double Hz = (L[6] + 0.5 * Txz) * z0 + (L[8] + 0.5 * Tyz) * z1 + (L[9] + 0.5 * Tzz) * z2;
    // L0' = L0 + L1.z + 1/2 z.L2.z + 1/6 L3:zzz
    const double zL2z = z0 * (L[4] * z0 + L[5] * z1 + L[6] * z2) + z1 * (L[5] * z0 + L[7] * z1 + L[8] * z2) +
                        z2 * (L[6] * z0 + L[8] * z1 + L[9] * z2);
    const double zTz = z0 * (Txx * z0 + Txy * z1 + Txz * z2) + z1 * (Txy * z0 + Tyy * z1 + Tyz * z2) +
                       z2 * (Txz * z0 + Tyz * z1 + Tzz * z2);
    const double d0 = L[0] + (L[1] * z0 + L[2] * z1 + L[3] * z2) + 0.5 * zL2z + zTz / 6.0;
    (void)zz;
    double *Lc = C.L + (int64_t)C.oslot[cn] * NC + l;
    Lc[0] += d0;
    Lc[crs] += L[1] + Hx;
    Lc[2 * crs] += L[2] + Hy;
    Lc[3 * crs] += L[3] + Hz;
    if ((C.kind[cn] & 3) == 2) {   // a refined child keeps the orders 2 and 3 for its own children
        double *Hc = C.Lhi + (int64_t)C.oslot[cn] * NC + l;
#pragma unroll
        for (int k = 0; k < 6; k++) Hc[k * chs] += M2[k];
#pragma unroll
        for (int k = 10; k < 20; k++) Hc[(k - 4) * chs] += L[k];
    }
    const double *Ap = P.Lc + (int64_t)P.oslot[pn] * NC + pl;
    double *Ac = C.Lc + (int64_t)C.oslot[cn] * NC + l;
#pragma unroll
    for (int k = 0; k < 3; k++) Ac[k * crs] += Ap[k * prs];
}

// owned cells in node order (ordslot: node-order index -> output slot)
__global__ void field_kernel(const LevelDesc *__restrict__ levels, int lev, const int32_t *__restrict__ ordslot,
                             double *__restrict__ phi, double *__restrict__ g)
{
    const LevelDesc &D = levels[lev];
    const int64_t n = D.n_owned * NC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = (int64_t)ordslot[i / NC] * NC + i % NC;
        phi[i] = D.L[s];
#pragma unroll
        for (int a = 0; a < 3; a++) g[a * n + i] = -(D.L[(1 + a) * n + s] + D.Lc[a * n + s]);
    }
}

extern "C" int octo_fmm_propagate(octo_fmm_t h, void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    if (h->cfg.nranks != 1) return fail(h, OCTO_EINVAL, "propagate: single-rank only in this version");
    CU(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int nl = (int)h->levels.size();
    if (nl == 0 || !h->levels[0].loaded) return fail(h, OCTO_EINVAL, "propagate: the root level is not loaded");
    for (int l = 0; l + 1 < nl; l++) {
        const Level &P = h->levels[l], &C = h->levels[l + 1];
        if (!C.loaded || C.n == 0) break;
        if (!P.loaded) return fail(h, OCTO_EINVAL, "propagate: a level between root and leaves is missing");
        // parent node of every child node (by coordinates)
        std::vector<int32_t> parent(C.n, -1);
        {
            std::vector<std::pair<uint64_t, int32_t>> keys(P.n);
            for (int64_t q = 0; q < P.n; q++)
                keys[q] = {((uint64_t)P.ijk[3 * q] << 42) | ((uint64_t)P.ijk[3 * q + 1] << 21) | (uint64_t)P.ijk[3 * q + 2],
                           (int32_t)q};
            std::sort(keys.begin(), keys.end());
            for (int64_t q = 0; q < C.n; q++) {
                const uint64_t k = ((uint64_t)(C.ijk[3 * q] >> 1) << 42) | ((uint64_t)(C.ijk[3 * q + 1] >> 1) << 21) |
                                   (uint64_t)(C.ijk[3 * q + 2] >> 1);
                auto it = std::lower_bound(keys.begin(), keys.end(), std::make_pair(k, (int32_t)-1));
                if (it == keys.end() || it->first != k || !P.refined[it->second])
                    return fail(h, OCTO_ESTRUCT, "propagate: child node without a refined parent");
                parent[q] = it->second;
            }
        }
        int32_t *d = nullptr;
        CU(cudaMallocAsync((void **)&d, 4 * C.n, st));
        CU(cudaMemcpyAsync(d, parent.data(), 4 * C.n, cudaMemcpyHostToDevice, st));
        const int64_t tot = C.n * NC;
        l2l_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(h->d_levels, l, d, C.n);
        h->launches++;
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(st));   // the host table must outlive the copy
        CU(cudaFreeAsync(d, st));
    }
    return OCTO_OK;
}

extern "C" int octo_fmm_get_field(octo_fmm_t h, int32_t level, double *phi, double *g, void *cuda_stream)
{
    if (!h || !phi || !g) return OCTO_EINVAL;
    if (level < 0 || level >= (int)h->levels.size() || !h->levels[level].loaded)
        return fail(h, OCTO_EINVAL, "level not loaded");
    CU(cudaSetDevice(h->cfg.device));
    if (h->levels[level].n_owned == 0) return OCTO_OK;
    field_kernel<<<148 * 4, 256, 0, (cudaStream_t)cuda_stream>>>(h->d_levels, level, h->levels[level].d_ordslot, phi, g);
    h->launches++;
    CU(cudaGetLastError());
    return OCTO_OK;
}
