// upward.cu -- FMM step 1 on the device: P2M and M2M.
//
// "First, it computes the multipole moments and the
// center-of-masses of the individual cells ... The fluid density of the cells
// of the highest level is the starting point. The multipole moments of every
// other cell are then calculated using the multipole moments of its child
// cells."  Leaf cell: m = rho h^3 at the geometric centre; refined cell: the
// exact shift of its 8 children's moments to their joint centre of mass
// (DESIGN.md "Readings" C3).  Inputs and outputs use the ABI layout of
// octo_fmm_load_level, so a level can be ingested straight from these buffers.
#include "internal.hpp"

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

__global__ void p2m_kernel(const double *__restrict__ rho, double vol, double *__restrict__ mono, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        mono[i] = rho[i] * vol;
}

// table per parent refined slot: children[8] (child node index per octant
// o = ox + 2 oy + 4 oz); child_rslot[n_child]; child_ijk[n_child][3]
__global__ void __launch_bounds__(256) m2m_kernel(int64_t nrp, const int32_t *__restrict__ prow,
                                                  const int32_t *__restrict__ children,
                                                  const int32_t *__restrict__ child_rslot,
                                                  const int32_t *__restrict__ child_ijk, int64_t ncr, double ch,
                                                  double ox, double oy, double oz,
                                                  const double *__restrict__ cmono, const double *__restrict__ ccom,
                                                  const double *__restrict__ cmom, double *__restrict__ pmono,
                                                  double *__restrict__ pcom, double *__restrict__ pmom)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrp * NC) return;
    const int64_t p = i / NC;
    const int l = (int)(i % NC);
    const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
    const int64_t cst = ncr * NC;
    // child cell q of parent cell l: node, local index, refined slot
    auto child = [&](int q, int64_t &cn, int &cl, int &rs, int &gx, int &gy, int &gz) {
        gx = 2 * lx + (q & 1); gy = 2 * ly + ((q >> 1) & 1); gz = 2 * lz + ((q >> 2) & 1);
        const int o = (gx >> 3) + 2 * (gy >> 3) + 4 * (gz >> 3);
        cn = children[p * 8 + o];
        cl = (gx & 7) + 8 * (gy & 7) + 64 * (gz & 7);
        rs = child_rslot[cn];
    };
    auto pos = [&](int64_t cn, int cl, int rs, int gx, int gy, int gz, double *x) {
        if (rs >= 0) {
            const int64_t b = (int64_t)rs * NC + cl;
            x[0] = ccom[b]; x[1] = ccom[cst + b]; x[2] = ccom[2 * cst + b];
        } else {
            x[0] = ox + ((double)(8 * child_ijk[3 * cn] + (gx & 7)) + 0.5) * ch;
            x[1] = oy + ((double)(8 * child_ijk[3 * cn + 1] + (gy & 7)) + 0.5) * ch;
            x[2] = oz + ((double)(8 * child_ijk[3 * cn + 2] + (gz & 7)) + 0.5) * ch;
        }
    };
    // pass 1: mass and centre of mass
    double m = 0.0, X[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < 8; q++) {
        int64_t cn; int cl, rs, gx, gy, gz;
        child(q, cn, cl, rs, gx, gy, gz);
        double x[3];
        pos(cn, cl, rs, gx, gy, gz, x);
        const double mq = cmono[cn * NC + cl];
        m += mq;
        for (int a = 0; a < 3; a++) X[a] = fma(mq, x[a], X[a]);
    }
    const double mi = 1.0 / m;
    for (int a = 0; a < 3; a++) X[a] *= mi;
    // pass 2: shifted moments (M2 xx xy xz yy yz zz; M3 xxx xxy xxz xyy xyz xzz yyy yyz yzz zzz)
    double M2[6] = {0, 0, 0, 0, 0, 0}, M3[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < 8; q++) {
        int64_t cn; int cl, rs, gx, gy, gz;
        child(q, cn, cl, rs, gx, gy, gz);
        double x[3];
        pos(cn, cl, rs, gx, gy, gz, x);
        const double mq = cmono[cn * NC + cl];
        const double y0 = x[0] - X[0], y1 = x[1] - X[1], y2 = x[2] - X[2];
        double s[6] = {0, 0, 0, 0, 0, 0}, t[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (rs >= 0) {
            const int64_t b = (int64_t)rs * NC + cl;
            for (int k = 0; k < 6; k++) s[k] = cmom[(4 + k) * cst + b];
            for (int k = 0; k < 10; k++) t[k] = cmom[(10 + k) * cst + b];
        }
        const double sxx = s[0], sxy = s[1], sxz = s[2], syy = s[3], syz = s[4], szz = s[5];
        M2[0] += sxx + mq * y0 * y0; M2[1] += sxy + mq * y0 * y1; M2[2] += sxz + mq * y0 * y2;
        M2[3] += syy + mq * y1 * y1; M2[4] += syz + mq * y1 * y2; M2[5] += szz + mq * y2 * y2;
        // M3_abc += T_abc + S_ab y_c + S_ac y_b + S_bc y_a + m y_a y_b y_c
        M3[0] += t[0] + 3.0 * sxx * y0 + mq * y0 * y0 * y0;                       // xxx
        M3[1] += t[1] + sxx * y1 + 2.0 * sxy * y0 + mq * y0 * y0 * y1;            // xxy
        M3[2] += t[2] + sxx * y2 + 2.0 * sxz * y0 + mq * y0 * y0 * y2;            // xxz
        M3[3] += t[3] + 2.0 * sxy * y1 + syy * y0 + mq * y0 * y1 * y1;            // xyy
        M3[4] += t[4] + sxy * y2 + sxz * y1 + syz * y0 + mq * y0 * y1 * y2;       // xyz
        M3[5] += t[5] + 2.0 * sxz * y2 + szz * y0 + mq * y0 * y2 * y2;            // xzz
        M3[6] += t[6] + 3.0 * syy * y1 + mq * y1 * y1 * y1;                       // yyy
        M3[7] += t[7] + syy * y2 + 2.0 * syz * y1 + mq * y1 * y1 * y2;            // yyz
        M3[8] += t[8] + 2.0 * syz * y2 + szz * y1 + mq * y1 * y2 * y2;            // yzz
        M3[9] += t[9] + 3.0 * szz * y2 + mq * y2 * y2 * y2;                       // zzz
    }
    const int64_t pst = nrp * NC, pb = p * NC + l;
    pmono[(int64_t)prow[p] * NC + l] = m;
#pragma unroll
    for (int a = 0; a < 3; a++) pcom[a * pst + pb] = X[a];
    pmom[pb] = m;
    pmom[pst + pb] = 0.0;
    pmom[2 * pst + pb] = 0.0;
    pmom[3 * pst + pb] = 0.0;
#pragma unroll
    for (int k = 0; k < 6; k++) pmom[(4 + k) * pst + pb] = M2[k];
#pragma unroll
    for (int k = 0; k < 10; k++) pmom[(10 + k) * pst + pb] = M3[k];
}

extern "C" int octo_fmm_p2m(octo_fmm_t h, int64_t n_cells, const double *rho, double h_cell, double *mono,
                            void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    if (n_cells < 0 || (n_cells > 0 && (!rho || !mono)) || !(h_cell > 0.0)) return fail(h, OCTO_EINVAL, "p2m args");
    CU(cudaSetDevice(h->cfg.device));
    if (n_cells == 0) return OCTO_OK;
    p2m_kernel<<<148 * 8, 256, 0, (cudaStream_t)cuda_stream>>>(rho, h_cell * h_cell * h_cell, mono, n_cells);
    h->launches++;
    CU(cudaGetLastError());
    return OCTO_OK;
}

extern "C" int octo_fmm_m2m(octo_fmm_t h, int64_t n_parent_refined, const int32_t *parent_rows,
                            const int32_t *children, int64_t n_child, const int32_t *child_ijk,
                            const uint8_t *child_refined, double child_h, const double origin[3],
                            const double *child_mono, const double *child_com, const double *child_mom,
                            double *parent_mono, double *parent_com, double *parent_mom, void *cuda_stream)
{
    if (!h) return OCTO_EINVAL;
    if (n_parent_refined < 0 || n_child < 0 || !(child_h > 0.0) || !origin) return fail(h, OCTO_EINVAL, "m2m args");
    if (n_parent_refined == 0) return OCTO_OK;
    if (!parent_rows || !children || !child_ijk || !child_refined || !child_mono || !parent_mono || !parent_com ||
        !parent_mom)
        return fail(h, OCTO_EINVAL, "m2m: null argument");
    CU(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)cuda_stream;
    std::vector<int32_t> rslot(n_child, -1);
    int64_t ncr = 0;
    for (int64_t q = 0; q < n_child; q++)
        if (child_refined[q]) rslot[q] = (int32_t)ncr++;
    if (ncr > 0 && (!child_com || !child_mom)) return fail(h, OCTO_EINVAL, "m2m: child com/mom required");
    for (int64_t p = 0; p < 8 * n_parent_refined; p++)
        if (children[p] < 0 || children[p] >= n_child) return fail(h, OCTO_ESTRUCT, "m2m: missing child node");
    // small host tables -> one device scratch allocation (stream-ordered)
    const size_t b_prow = 4 * n_parent_refined, b_ch = 32 * n_parent_refined, b_rs = 4 * n_child, b_ijk = 12 * n_child;
    const size_t bytes = b_prow + b_ch + b_rs + b_ijk;
    std::vector<char> host(bytes);
    std::memcpy(host.data(), parent_rows, b_prow);
    std::memcpy(host.data() + b_prow, children, b_ch);
    std::memcpy(host.data() + b_prow + b_ch, rslot.data(), b_rs);
    std::memcpy(host.data() + b_prow + b_ch + b_rs, child_ijk, b_ijk);
    char *d = nullptr;
    CU(cudaMallocAsync((void **)&d, bytes, st));
    CU(cudaMemcpyAsync(d, host.data(), bytes, cudaMemcpyHostToDevice, st));
    const int64_t tot = n_parent_refined * NC;
    m2m_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        n_parent_refined, (const int32_t *)d, (const int32_t *)(d + b_prow), (const int32_t *)(d + b_prow + b_ch),
        (const int32_t *)(d + b_prow + b_ch + b_rs), ncr, child_h, origin[0], origin[1], origin[2], child_mono,
        child_com, child_mom, parent_mono, parent_com, parent_mom);
    h->launches++;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st));   // the host staging vector must outlive the copy
    CU(cudaFreeAsync(d, st));
    return OCTO_OK;
}
