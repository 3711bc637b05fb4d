// layout.cuh -- constants and the per-level device descriptor shared by the
// kernels (kernels.cuh) and the host code (octo_fmm.cu, exchange.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace octo {

constexpr int NC = 512;        // cells per sub-grid
constexpr int NREC = 16;       // record components: 0 m, 1-3 X, 4-8 Q2', 9-15 Q3'

// Prepared refined record in HBM: component pairs (2j, 2j+1) adjacent, so a
// partner's record is 8 aligned 16-byte loads (the M2L window's layout):
// component k of the cell (child parity q, parent index p) of refined slot rs.
__host__ __device__ __forceinline__ int64_t prec(int64_t rs, int k, int q, int p)
{
    return ((((rs * (NREC / 2) + (k >> 1)) * 8 + q) * 64 + p) << 1) + (k & 1);
}
constexpr int MAXE = 256;      // max entries per (c,q) list: 93 for theta >= 1/3 (parent reach 2), 251 at 0.25 (reach 3)
constexpr int KBOX = 7;        // |d| <= 7: parent reach <= 3 (theta >= 0.25)
constexpr int KDIM = 2 * KBOX + 1;
constexpr int KBOX2 = 5;       // |d| <= 5 at parent reach 2 (theta >= 1/3): the __constant__ P2P table
constexpr int KDIM2 = 2 * KBOX2 + 1;

struct LevelDesc {
    const int32_t *ijk;     // [n][3]
    const int32_t *nb;      // [n][27]
    const uint8_t *kind;    // [n] 1 leaf, 2 refined, 0 = unknown/ghost-not-received
    const int32_t *rslot;   // [n] refined slot or -1
    const int32_t *oslot;   // [n] owned output slot or -1
    const double *mass;     // [n][8][64]   parity-deinterleaved masses
    const double *pref;     // [nr][8 pairs][8][64][2] prepared refined records (prec)
    const int16_t *msort;   // [n][512] cells of a mixed-work node sorted by mixed work (desc)
    const void *tmaps;      // 7 CUtensorMap (64-byte aligned, global memory) over pref, one per halo box
                            // shape (face / edge / corner orientations), or null (no refined node)
    double *L;              // rows 0..3 of every owned slot: [4][n_owned][512]
    double *Lhi;            // rows 4..19 of the owned refined slots (slots 0..n_oref-1): [16][n_oref][512]
    double *Lc;             // [3][n_owned][512]
    int64_t n_owned, n_oref;
    double h;
    double ox, oy, oz;
    double G;
};

}  // namespace octo
