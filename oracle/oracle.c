/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the hot path
 * computes: Octo-Tiger's FMM step 2 ("same-level" interactions) on octree
 * levels of 8^3-cell sub-grids, plus the surrounding pieces needed to pin it
 * (step 1 P2M/M2M, step 3 L2L, direct N^2 summation, conservation invariants,
 * exactly-once coverage).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares NO code, header,
 * table or constant generator with the CUDA path under
 * paper_1908_03121_b200/ and neither side includes the other.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no fast-math, no FMA
 * contraction, IEEE binary64 round-to-nearest).
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn; "S:Lnnn" =
 * SPEC.md line nnn; "C1".."C10" = SURVEY.md section 8(c) rows whose readings
 * are listed in DESIGN.md section "Readings".
 *
 * Conventions:
 *   - cell local index l = lx + 8*ly + 64*lz; global cell coords at level ℓ:
 *     g = 8*node_ijk + (lx,ly,lz); cell width h_ℓ; leaf-cell position is the
 *     geometric centre origin + (g + 1/2) h.
 *   - multipole coefficient order (20): 0 m; 1-3 dipole x,y,z (identically 0
 *     about the centre of mass); 4-9 xx,xy,xz,yy,yz,zz; 10-19 xxx,xxy,xxz,xyy,
 *     xyz,xzz,yyy,yyz,yzz,zzz.  Entries are FULL Cartesian moments
 *     M_k = sum_i m_i (x_i - X)^k (no factorials, no detracing).
 *   - Taylor coefficients L (20), same index order, entries of the symmetric
 *     tensors L^(n): Phi(X_A + z) = L0 + L_a z_a + 1/2 L_ab z_a z_b
 *     + 1/6 L_abc z_a z_b z_c (full index sums); angular-momentum correction
 *     Lc (3).  Green's function phi = -1/r (G applied by the caller).
 *
 * Parity: all functions below are pinned by tests in tests/test_oracle_*.py
 * except the flop-count convention (C10), which is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NCELL 512

/* ------------------------------------------------------------------------ */
/* symmetric-tensor index helpers (plain lookup tables)                      */
/* ------------------------------------------------------------------------ */
static int sym2(int a, int b)
{
    static const int t[3][3] = {{4, 5, 6}, {5, 7, 8}, {6, 8, 9}};
    return t[a][b];
}

static int sym3(int a, int b, int c)
{
    /* sort a <= b <= c */
    int s[3] = {a, b, c}, tmp;
    if (s[0] > s[1]) { tmp = s[0]; s[0] = s[1]; s[1] = tmp; }
    if (s[1] > s[2]) { tmp = s[1]; s[1] = s[2]; s[2] = tmp; }
    if (s[0] > s[1]) { tmp = s[0]; s[0] = s[1]; s[1] = tmp; }
    if (s[0] == 0 && s[1] == 0 && s[2] == 0) return 10;
    if (s[0] == 0 && s[1] == 0 && s[2] == 1) return 11;
    if (s[0] == 0 && s[1] == 0 && s[2] == 2) return 12;
    if (s[0] == 0 && s[1] == 1 && s[2] == 1) return 13;
    if (s[0] == 0 && s[1] == 1 && s[2] == 2) return 14;
    if (s[0] == 0 && s[1] == 2 && s[2] == 2) return 15;
    if (s[0] == 1 && s[1] == 1 && s[2] == 1) return 16;
    if (s[0] == 1 && s[1] == 1 && s[2] == 2) return 17;
    if (s[0] == 1 && s[1] == 2 && s[2] == 2) return 18;
    return 19; /* 2,2,2 */
}

static double kd(int a, int b) { return a == b ? 1.0 : 0.0; }

/* floor(a / 2) for signed integers */
static int64_t fdiv2(int64_t a) { return (a >= 0) ? a / 2 : -((-a + 1) / 2); }

/* ------------------------------------------------------------------------ */
/* C1: opening criterion                  */
/* ------------------------------------------------------------------------ */

/* R^2 = (1/theta)^2, computed once per theta (C1 precision reading). */
double oc_R2(double theta)
{
    double r = 1.0 / theta;
    return r * r;
}

/*
 * Interaction class of target cell i and partner cell j on the same level:
 *   0 = no same-level interaction, 1 = far, 2 = near.
 * Levels >= 1: the pair is parent-near iff |floor(j/2)-floor(i/2)|^2 < R^2
 * (strict); within parent-near it is far iff |j-i|^2 >= R^2 (non-strict),
 * else near.  Root level (is_root): no parent; far iff |d|^2 >= R^2, near
 * iff 0 < |d|^2 < R^2 (C2 reading).
 */
int oc_pair_class(double R2, int is_root, const int64_t *i, const int64_t *j)
{
    int64_t d2 = 0, p2 = 0;
    int a;
    for (a = 0; a < 3; a++) {
        int64_t d = j[a] - i[a];
        d2 += d * d;
    }
    if (d2 == 0) return 0;
    if (!is_root) {
        for (a = 0; a < 3; a++) {
            int64_t p = fdiv2(j[a]) - fdiv2(i[a]);
            p2 += p * p;
        }
        if (!((double)p2 < R2)) return 0;
    }
    return ((double)d2 >= R2) ? 1 : 2;
}

/*
 * Per-parity stencil, C1.  For parity c = (cx,cy,cz) in {0,1}^3 (index
 * cx + 2cy + 4cz), list every offset d in [-B,B]^3 (B = box half width) with
 * its class.  out[(c*cap + k)*4 + 0..3] = dx, dy, dz, cls.  Returns 0, or -1
 * if cap is too small.  counts[c] = number of entries for parity c.
 */
int oc_stencil(double theta, int is_root, int box, int32_t *out, int32_t *counts, int cap)
{
    double R2 = oc_R2(theta);
    int c;
    for (c = 0; c < 8; c++) {
        int64_t i[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
        int n = 0;
        int dx, dy, dz;
        for (dx = -box; dx <= box; dx++)
            for (dy = -box; dy <= box; dy++)
                for (dz = -box; dz <= box; dz++) {
                    int64_t j[3] = {i[0] + dx, i[1] + dy, i[2] + dz};
                    int cls = oc_pair_class(R2, is_root, i, j);
                    if (cls == 0) continue;
                    if (n >= cap) return -1;
                    out[(c * cap + n) * 4 + 0] = dx;
                    out[(c * cap + n) * 4 + 1] = dy;
                    out[(c * cap + n) * 4 + 2] = dz;
                    out[(c * cap + n) * 4 + 3] = cls;
                    n++;
                }
        counts[c] = n;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* C5: derivative tensors of phi = -1/r at R (closed forms, full 3^n)        */
/* ------------------------------------------------------------------------ */
void oc_dtensors(const double *R, double *D0, double *D1, double *D2, double *D3, double *D4)
{
    double r2 = R[0] * R[0] + R[1] * R[1] + R[2] * R[2];
    double r = sqrt(r2);
    double r3 = r * r2, r5 = r3 * r2, r7 = r5 * r2, r9 = r7 * r2;
    int a, b, c, d;
    *D0 = -1.0 / r;
    for (a = 0; a < 3; a++) D1[a] = R[a] / r3;
    for (a = 0; a < 3; a++)
        for (b = 0; b < 3; b++)
            D2[a * 3 + b] = kd(a, b) / r3 - 3.0 * R[a] * R[b] / r5;
    for (a = 0; a < 3; a++)
        for (b = 0; b < 3; b++)
            for (c = 0; c < 3; c++)
                D3[(a * 3 + b) * 3 + c] =
                    -3.0 * (kd(a, b) * R[c] + kd(a, c) * R[b] + kd(b, c) * R[a]) / r5
                    + 15.0 * R[a] * R[b] * R[c] / r7;
    for (a = 0; a < 3; a++)
        for (b = 0; b < 3; b++)
            for (c = 0; c < 3; c++)
                for (d = 0; d < 3; d++)
                    D4[((a * 3 + b) * 3 + c) * 3 + d] =
                        -3.0 * (kd(a, b) * kd(c, d) + kd(a, c) * kd(b, d) + kd(a, d) * kd(b, c)) / r5
                        + 15.0 * (kd(a, b) * R[c] * R[d] + kd(a, c) * R[b] * R[d]
                                  + kd(a, d) * R[b] * R[c] + kd(b, c) * R[a] * R[d]
                                  + kd(b, d) * R[a] * R[c] + kd(c, d) * R[a] * R[b]) / r7
                        - 105.0 * R[a] * R[b] * R[c] * R[d] / r9;
}

/*
 * Magnitude bounds of the same closed forms (C9 parity scale): every term of
 * every D entry in absolute value, e.g. |D2|_ab = delta_ab/r^3 + 3|R_a R_b|/r^5.
 */
void oc_dtensors_abs(const double *R, double *D0, double *D1, double *D2, double *D3, double *D4)
{
    double r2 = R[0] * R[0] + R[1] * R[1] + R[2] * R[2];
    double r = sqrt(r2);
    double r3 = r * r2, r5 = r3 * r2, r7 = r5 * r2, r9 = r7 * r2;
    double A[3] = {fabs(R[0]), fabs(R[1]), fabs(R[2])};
    int a, b, c, d;
    *D0 = 1.0 / r;
    for (a = 0; a < 3; a++) D1[a] = A[a] / r3;
    for (a = 0; a < 3; a++)
        for (b = 0; b < 3; b++)
            D2[a * 3 + b] = kd(a, b) / r3 + 3.0 * A[a] * A[b] / r5;
    for (a = 0; a < 3; a++)
        for (b = 0; b < 3; b++)
            for (c = 0; c < 3; c++)
                D3[(a * 3 + b) * 3 + c] =
                    3.0 * (kd(a, b) * A[c] + kd(a, c) * A[b] + kd(b, c) * A[a]) / r5
                    + 15.0 * A[a] * A[b] * A[c] / r7;
    for (a = 0; a < 3; a++)
        for (b = 0; b < 3; b++)
            for (c = 0; c < 3; c++)
                for (d = 0; d < 3; d++)
                    D4[((a * 3 + b) * 3 + c) * 3 + d] =
                        3.0 * (kd(a, b) * kd(c, d) + kd(a, c) * kd(b, d) + kd(a, d) * kd(b, c)) / r5
                        + 15.0 * (kd(a, b) * A[c] * A[d] + kd(a, c) * A[b] * A[d]
                                  + kd(a, d) * A[b] * A[c] + kd(b, c) * A[a] * A[d]
                                  + kd(b, d) * A[a] * A[c] + kd(c, d) * A[a] * A[b]) / r7
                        + 105.0 * A[a] * A[b] * A[c] * A[d] / r9;
}

/* ------------------------------------------------------------------------ */
/* C4: P2P pair kernel (leaf <- leaf), t[0..3] = increments of L0, L1        */
/* ------------------------------------------------------------------------ */
void oc_p2p(double mB, const double *R, double *t)
{
    double r2 = R[0] * R[0] + R[1] * R[1] + R[2] * R[2];
    double r = sqrt(r2);
    double r3 = r * r2;
    t[0] = -mB / r;
    t[1] = mB * R[0] / r3;
    t[2] = mB * R[1] / r3;
    t[3] = mB * R[2] / r3;
}

/*
 * C5: M2L pair kernel with the angular-momentum correction.
 * Source B (mass mB, moments MB about its centre of mass), target A
 * (mass mA, moments MA), R = X_A - X_B.  Truncation n + m <= 3:
 *   L0    += mB D0 + 1/2 M2B:D2 - 1/6 M3B:D3
 *   L_a   += mB D_a + 1/2 M2B_bc D_abc
 *   L_ab  += mB D_ab            (refined targets only)
 *   L_abc += mB D_abc           (refined targets only)
 *   Lc_a  += -1/6 (M3B_bcd - M3A_bcd mB/mA) D_abcd
 * t[0..19] = L increments (rows 4..19 zero for leaf targets), t[20..22] = Lc.
 */
static void m2l_impl(double mA, const double *MA, double mB, const double *MB, const double *R,
                     int target_refined, int absmode, double *t)
{
    double D0, D1[3], D2[9], D3[27], D4[81];
    double M2B[9], M3B[27], M3A[27];
    int a, b, c, d;
    if (absmode) oc_dtensors_abs(R, &D0, D1, D2, D3, D4);
    else oc_dtensors(R, &D0, D1, D2, D3, D4);
    for (a = 0; a < 3; a++)
        for (b = 0; b < 3; b++) {
            M2B[a * 3 + b] = absmode ? fabs(MB[sym2(a, b)]) : MB[sym2(a, b)];
            for (c = 0; c < 3; c++) {
                M3B[(a * 3 + b) * 3 + c] = absmode ? fabs(MB[sym3(a, b, c)]) : MB[sym3(a, b, c)];
                M3A[(a * 3 + b) * 3 + c] = absmode ? -fabs(MA[sym3(a, b, c)]) : MA[sym3(a, b, c)];
            }
        }
    if (absmode) mB = fabs(mB);
    for (a = 0; a < 23; a++) t[a] = 0.0;
    /* L0 */
    {
        double s2 = 0.0, s3 = 0.0;
        for (a = 0; a < 3; a++)
            for (b = 0; b < 3; b++) {
                s2 += M2B[a * 3 + b] * D2[a * 3 + b];
                for (c = 0; c < 3; c++) s3 += M3B[(a * 3 + b) * 3 + c] * D3[(a * 3 + b) * 3 + c];
            }
        t[0] = absmode ? mB * D0 + 0.5 * s2 + s3 / 6.0 : mB * D0 + 0.5 * s2 - s3 / 6.0;
    }
    /* L1 */
    for (a = 0; a < 3; a++) {
        double s = 0.0;
        for (b = 0; b < 3; b++)
            for (c = 0; c < 3; c++) s += M2B[b * 3 + c] * D3[(a * 3 + b) * 3 + c];
        t[1 + a] = mB * D1[a] + 0.5 * s;
    }
    if (target_refined) {
        for (a = 0; a < 3; a++)
            for (b = a; b < 3; b++) t[sym2(a, b)] = mB * D2[a * 3 + b];
        for (a = 0; a < 3; a++)
            for (b = a; b < 3; b++)
                for (c = b; c < 3; c++) t[sym3(a, b, c)] = mB * D3[(a * 3 + b) * 3 + c];
    }
    /* Lc: angular-momentum correction (C5 reading of P:L229-232, L465) */
    for (a = 0; a < 3; a++) {
        double s = 0.0;
        for (b = 0; b < 3; b++)
            for (c = 0; c < 3; c++)
                for (d = 0; d < 3; d++) {
                    int k = (b * 3 + c) * 3 + d;
                    s += (M3B[k] - M3A[k] * mB / mA) * D4[((a * 3 + b) * 3 + c) * 3 + d];
                }
        t[20 + a] = absmode ? s / 6.0 : -s / 6.0;
    }
}

void oc_m2l(double mA, const double *MA, double mB, const double *MB, const double *R,
            int target_refined, double *t)
{
    m2l_impl(mA, MA, mB, MB, R, target_refined, 0, t);
}

/* C9 parity scale: the M2L formula evaluated with every factor in absolute
 * value (a forward-error magnitude bound of each output component). */
void oc_m2l_abs(double mA, const double *MA, double mB, const double *MB, const double *R,
                int target_refined, double *t)
{
    m2l_impl(mA, MA, mB, MB, R, target_refined, 1, t);
}

/* ------------------------------------------------------------------------ */
/* node lookup: sorted (key, index) pairs + binary search                    */
/* ------------------------------------------------------------------------ */
typedef struct { uint64_t key; int64_t idx; } oc_kv;

static uint64_t node_key(int64_t i, int64_t j, int64_t k)
{
    return ((uint64_t)i << 42) | ((uint64_t)j << 21) | (uint64_t)k;
}

static int kv_cmp(const void *x, const void *y)
{
    uint64_t a = ((const oc_kv *)x)->key, b = ((const oc_kv *)y)->key;
    return (a < b) ? -1 : (a > b) ? 1 : 0;
}

static oc_kv *build_lookup(int64_t n, const int32_t *ijk)
{
    oc_kv *t = (oc_kv *)malloc(sizeof(oc_kv) * (size_t)(n > 0 ? n : 1));
    int64_t q;
    for (q = 0; q < n; q++) {
        t[q].key = node_key(ijk[3 * q], ijk[3 * q + 1], ijk[3 * q + 2]);
        t[q].idx = q;
    }
    qsort(t, (size_t)n, sizeof(oc_kv), kv_cmp);
    return t;
}

static int64_t find_node(const oc_kv *t, int64_t n, int64_t i, int64_t j, int64_t k)
{
    int64_t lo = 0, hi = n - 1;
    uint64_t key;
    if (i < 0 || j < 0 || k < 0) return -1;
    key = node_key(i, j, k);
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (t[mid].key == key) return t[mid].idx;
        if (t[mid].key < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

static int64_t fdiv8(int64_t a) { return (a >= 0) ? a / 8 : -((-a + 7) / 8); }

/* ------------------------------------------------------------------------ */
/* C3: P2M (leaf cell mass = rho h^3) and M2M (bottom-up)                    */
/* ------------------------------------------------------------------------ */
void oc_p2m(int64_t n, const double *rho, double h, double *m)
{
    int64_t q;
    double vol = h * h * h;
    for (q = 0; q < n; q++) m[q] = rho[q] * vol;
}

/* read a cell's (m, X, M[20]) from a level (leaf: X = centre, M = (m,0..)) */
static void cell_data(int64_t node, int cell, const int32_t *ijk, const uint8_t *refined,
                      const int64_t *rslot, const double *m, const double *X, const double *M,
                      double h, const double *origin, double *mo, double *Xo, double *Mo)
{
    int a;
    *mo = m[node * NCELL + cell];
    if (refined[node]) {
        int64_t s = rslot[node];
        for (a = 0; a < 3; a++) Xo[a] = X[(s * NCELL + cell) * 3 + a];
        for (a = 0; a < 20; a++) Mo[a] = M[(s * NCELL + cell) * 20 + a];
    } else {
        int loc[3] = {cell & 7, (cell >> 3) & 7, (cell >> 6) & 7};
        for (a = 0; a < 3; a++) Xo[a] = origin[a] + ((double)(8 * (int64_t)ijk[3 * node + a] + loc[a]) + 0.5) * h;
        for (a = 0; a < 20; a++) Mo[a] = 0.0;
        Mo[0] = *mo;
    }
}

/*
 * M2M for every refined node of a parent level from its child level.
 * Parent cell g has children 2g + q (q in {0,1}^3) on the child level.
 *   m = sum m_i,  X = sum m_i X_i / m,  y_i = X_i - X,
 *   M2_ab  = sum [M2_i,ab + m_i y_a y_b]
 *   M3_abc = sum [M3_i,abc + M2_i,ab y_c + M2_i,ac y_b + M2_i,bc y_a + m_i y_a y_b y_c]
 * (exact shift of point-mass moments; dipoles vanish about the COM).
 * Writes m_p rows of refined nodes, X_p[rslot][cell][3], M_p[rslot][cell][20].
 * Returns 0, or -1 if a child node is missing.
 */
int oc_m2m(int64_t n_p, const int32_t *ijk_p, const uint8_t *refined_p, const int64_t *rslot_p,
           int64_t n_c, const int32_t *ijk_c, const uint8_t *refined_c, const int64_t *rslot_c,
           const double *m_c, const double *X_c, const double *M_c, double h_c, const double *origin,
           double *m_p, double *X_p, double *M_p)
{
    oc_kv *lk = build_lookup(n_c, ijk_c);
    int64_t P;
    for (P = 0; P < n_p; P++) {
        int cell;
        if (!refined_p[P]) continue;
        for (cell = 0; cell < NCELL; cell++) {
            int64_t g[3] = {8 * (int64_t)ijk_p[3 * P] + (cell & 7), 8 * (int64_t)ijk_p[3 * P + 1] + ((cell >> 3) & 7),
                            8 * (int64_t)ijk_p[3 * P + 2] + ((cell >> 6) & 7)};
            double cm[8], cX[8][3], cM[8][20];
            double mt = 0.0, Xt[3] = {0, 0, 0}, Mf2[9], Mf3[27];
            int q, a, b, c;
            for (q = 0; q < 8; q++) {
                int64_t ch[3] = {2 * g[0] + (q & 1), 2 * g[1] + ((q >> 1) & 1), 2 * g[2] + ((q >> 2) & 1)};
                int64_t cn = find_node(lk, n_c, fdiv8(ch[0]), fdiv8(ch[1]), fdiv8(ch[2]));
                int lcell;
                if (cn < 0) { free(lk); return -1; }
                lcell = (int)((ch[0] - 8 * fdiv8(ch[0])) + 8 * (ch[1] - 8 * fdiv8(ch[1])) + 64 * (ch[2] - 8 * fdiv8(ch[2])));
                cell_data(cn, lcell, ijk_c, refined_c, rslot_c, m_c, X_c, M_c, h_c, origin, &cm[q], cX[q], cM[q]);
            }
            for (q = 0; q < 8; q++) mt += cm[q];
            for (a = 0; a < 3; a++) {
                for (q = 0; q < 8; q++) Xt[a] += cm[q] * cX[q][a];
                Xt[a] /= mt;
            }
            for (a = 0; a < 9; a++) Mf2[a] = 0.0;
            for (a = 0; a < 27; a++) Mf3[a] = 0.0;
            for (q = 0; q < 8; q++) {
                double y[3];
                for (a = 0; a < 3; a++) y[a] = cX[q][a] - Xt[a];
                for (a = 0; a < 3; a++)
                    for (b = 0; b < 3; b++) {
                        Mf2[a * 3 + b] += cM[q][sym2(a, b)] + cm[q] * y[a] * y[b];
                        for (c = 0; c < 3; c++)
                            Mf3[(a * 3 + b) * 3 + c] += cM[q][sym3(a, b, c)]
                                + cM[q][sym2(a, b)] * y[c] + cM[q][sym2(a, c)] * y[b] + cM[q][sym2(b, c)] * y[a]
                                + cm[q] * y[a] * y[b] * y[c];
                    }
            }
            {
                int64_t s = rslot_p[P];
                double *Mo = &M_p[(s * NCELL + cell) * 20];
                m_p[P * NCELL + cell] = mt;
                for (a = 0; a < 3; a++) X_p[(s * NCELL + cell) * 3 + a] = Xt[a];
                Mo[0] = mt;
                Mo[1] = Mo[2] = Mo[3] = 0.0;
                for (a = 0; a < 3; a++)
                    for (b = a; b < 3; b++) {
                        Mo[sym2(a, b)] = Mf2[a * 3 + b];
                        for (c = b; c < 3; c++) Mo[sym3(a, b, c)] = Mf3[(a * 3 + b) * 3 + c];
                    }
            }
        }
    }
    free(lk);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* C6 + C4/C5: same-level interactions for a list of target cells            */
/* ------------------------------------------------------------------------ */
/* accumulate the C9 magnitude scale of one pair contribution */
static void add_abs(int a_ref, int b_ref, int cls, double mA, const double *MA, double mB, const double *MB,
                    const double *R, const double *term, double *aab)
{
    double ta[23];
    int k;
    (void)cls;
    if (!a_ref && !b_ref) {
        for (k = 0; k < 23; k++) aab[k] += fabs(term[k]);   /* P2P: |term| is the bound */
        return;
    }
    for (k = 0; k < 23; k++) ta[k] = 0.0;
    m2l_impl(mA, MA, mB, MB, R, a_ref, 1, ta);
    for (k = 0; k < 23; k++) aab[k] += ta[k];
}

/*
 * For each target (node, cell) on a level, sum over EVERY candidate partner
 * cell j on the same level the pair contribution selected by the class
 * predicate (C1/C2) and the AMR case rule (C6):
 *   refined target: far -> M2L (any partner); near -> M2L iff partner leaf;
 *   leaf target:    far or near -> P2P if partner leaf, M2L (mixed) else.
 * Candidates: all cells of all nodes (prune = 0) or the box |d|_inf <=
 * 2 floor(R) + 1 (prune = 1), which contains every parent-near partner
 * (|p_a| <= floor(R) => |d_a| <= 2 floor(R) + 1); the test suite checks the
 * two agree.  Order: lexicographic d (dx, dy, dz), i.e. deterministic.
 * Outputs: L[t][20], Lc[t][3], absL[t][23] = per-component magnitude scale
 * (C9): sum over pairs of the pair formula evaluated with |.| of every factor.
 * Returns 0 or -1 (bad target).
 */
int oc_same_level(int is_root, double theta, double h, const double *origin,
                  int64_t n, const int32_t *ijk, const uint8_t *refined, const int64_t *rslot,
                  const double *m, const double *X, const double *M,
                  int64_t n_targets, const int64_t *tgt_node, const int32_t *tgt_cell, int prune,
                  double *L, double *Lc, double *absL)
{
    double R2 = oc_R2(theta);
    int B = 2 * (int)floor(sqrt(R2)) + 1;
    oc_kv *lk = build_lookup(n, ijk);
    int64_t t;
    if (is_root) B = 7;
    for (t = 0; t < n_targets; t++) {
        int64_t A = tgt_node[t];
        int ca = tgt_cell[t];
        double mA, XA[3], MA[20];
        int64_t gi[3];
        double acc[23], aab[23];
        int k;
        if (A < 0 || A >= n || ca < 0 || ca >= NCELL) { free(lk); return -1; }
        cell_data(A, ca, ijk, refined, rslot, m, X, M, h, origin, &mA, XA, MA);
        gi[0] = 8 * (int64_t)ijk[3 * A] + (ca & 7);
        gi[1] = 8 * (int64_t)ijk[3 * A + 1] + ((ca >> 3) & 7);
        gi[2] = 8 * (int64_t)ijk[3 * A + 2] + ((ca >> 6) & 7);
        for (k = 0; k < 23; k++) acc[k] = aab[k] = 0.0;

        if (prune) {
            int dx, dy, dz;
            for (dx = -B; dx <= B; dx++)
                for (dy = -B; dy <= B; dy++)
                    for (dz = -B; dz <= B; dz++) {
                        int64_t gj[3] = {gi[0] + dx, gi[1] + dy, gi[2] + dz};
                        int64_t Bn;
                        int cb, cls;
                        double mB, XB[3], MB[20], R[3], term[23];
                        cls = oc_pair_class(R2, is_root, gi, gj);
                        if (cls == 0) continue;
                        Bn = find_node(lk, n, fdiv8(gj[0]), fdiv8(gj[1]), fdiv8(gj[2]));
                        if (Bn < 0) continue; /* absent nodes contribute nothing */
                        cb = (int)((gj[0] - 8 * fdiv8(gj[0])) + 8 * (gj[1] - 8 * fdiv8(gj[1])) + 64 * (gj[2] - 8 * fdiv8(gj[2])));
                        cell_data(Bn, cb, ijk, refined, rslot, m, X, M, h, origin, &mB, XB, MB);
                        for (k = 0; k < 3; k++) R[k] = XA[k] - XB[k];
                        for (k = 0; k < 23; k++) term[k] = 0.0;
                        if (refined[A]) {
                            if (cls == 1 || !refined[Bn]) oc_m2l(mA, MA, mB, MB, R, 1, term);
                            else continue;
                        } else {
                            if (!refined[Bn]) oc_p2p(mB, R, term);
                            else oc_m2l(mA, MA, mB, MB, R, 0, term);
                        }
                        for (k = 0; k < 23; k++) acc[k] += term[k];
                        add_abs(refined[A], refined[Bn], cls, mA, MA, mB, MB, R, term, aab);
                    }
        } else {
            int64_t Bn;
            for (Bn = 0; Bn < n; Bn++) {
                int cb;
                for (cb = 0; cb < NCELL; cb++) {
                    int64_t gj[3] = {8 * (int64_t)ijk[3 * Bn] + (cb & 7), 8 * (int64_t)ijk[3 * Bn + 1] + ((cb >> 3) & 7),
                                     8 * (int64_t)ijk[3 * Bn + 2] + ((cb >> 6) & 7)};
                    int cls = oc_pair_class(R2, is_root, gi, gj);
                    double mB, XB[3], MB[20], R[3], term[23];
                    if (cls == 0) continue;
                    cell_data(Bn, cb, ijk, refined, rslot, m, X, M, h, origin, &mB, XB, MB);
                    for (k = 0; k < 3; k++) R[k] = XA[k] - XB[k];
                    for (k = 0; k < 23; k++) term[k] = 0.0;
                    if (refined[A]) {
                        if (cls == 1 || !refined[Bn]) oc_m2l(mA, MA, mB, MB, R, 1, term);
                        else continue;
                    } else {
                        if (!refined[Bn]) oc_p2p(mB, R, term);
                        else oc_m2l(mA, MA, mB, MB, R, 0, term);
                    }
                    for (k = 0; k < 23; k++) acc[k] += term[k];
                    add_abs(refined[A], refined[Bn], cls, mA, MA, mB, MB, R, term, aab);
                }
            }
        }
        for (k = 0; k < 20; k++) { L[t * 20 + k] = acc[k]; absL[t * 23 + k] = aab[k]; }
        for (k = 0; k < 3; k++) { Lc[t * 3 + k] = acc[20 + k]; absL[t * 23 + 20 + k] = aab[20 + k]; }
    }
    free(lk);
    return 0;
}

/*
 * Interaction counts per target by class (for C10 flop accounting and the
 * bench's algorithmic work): counts[t][3] = {P2P, M2L (refined target), mixed
 * (leaf target <- refined partner)}.  Same enumeration as oc_same_level.
 */
int oc_count_interactions(int is_root, double theta, int64_t n, const int32_t *ijk, const uint8_t *refined,
                          int64_t n_targets, const int64_t *tgt_node, const int32_t *tgt_cell, int64_t *counts)
{
    double R2 = oc_R2(theta);
    int B = is_root ? 7 : 2 * (int)floor(sqrt(R2)) + 1;
    oc_kv *lk = build_lookup(n, ijk);
    int64_t t;
    for (t = 0; t < n_targets; t++) {
        int64_t A = tgt_node[t];
        int ca = tgt_cell[t];
        int64_t gi[3] = {8 * (int64_t)ijk[3 * A] + (ca & 7), 8 * (int64_t)ijk[3 * A + 1] + ((ca >> 3) & 7),
                         8 * (int64_t)ijk[3 * A + 2] + ((ca >> 6) & 7)};
        int dx, dy, dz;
        counts[t * 3] = counts[t * 3 + 1] = counts[t * 3 + 2] = 0;
        for (dx = -B; dx <= B; dx++)
            for (dy = -B; dy <= B; dy++)
                for (dz = -B; dz <= B; dz++) {
                    int64_t gj[3] = {gi[0] + dx, gi[1] + dy, gi[2] + dz};
                    int cls = oc_pair_class(R2, is_root, gi, gj);
                    int64_t Bn;
                    if (cls == 0) continue;
                    Bn = find_node(lk, n, fdiv8(gj[0]), fdiv8(gj[1]), fdiv8(gj[2]));
                    if (Bn < 0) continue;
                    if (refined[A]) {
                        if (cls == 1 || !refined[Bn]) counts[t * 3 + 1]++;
                    } else {
                        if (!refined[Bn]) counts[t * 3 + 0]++; else counts[t * 3 + 2]++;
                    }
                }
    }
    free(lk);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* C8: step 3 (L2L) and direct N^2 summation                                 */
/* ------------------------------------------------------------------------ */
/*
 * L2L: every cell of every node of the child level receives its parent
 * cell's expansion re-centred by the exact cubic Taylor shift z = Y - X_P
 * (Y = child cell expansion centre, X_P = parent cell COM):
 *   L0'  += L0 + L_a z_a + 1/2 L_ab z_a z_b + 1/6 L_abc z_a z_b z_c
 *   L_a' += L_a + L_ab z_b + 1/2 L_abc z_b z_c
 *   L_ab'+= L_ab + L_abc z_c ;  L_abc' += L_abc ;  Lc' += Lc
 * Lp/Lcp: [n_p][512][20]/[3] (parent totals); Lch/Lcch updated in place.
 */
int oc_l2l(int64_t n_p, const int32_t *ijk_p, const int64_t *rslot_p, const double *X_p,
           const double *Lp, const double *Lcp,
           int64_t n_c, const int32_t *ijk_c, const uint8_t *refined_c, const int64_t *rslot_c,
           const double *X_c, double h_c, const double *origin, double *Lch, double *Lcch)
{
    oc_kv *lk = build_lookup(n_p, ijk_p);
    int64_t C;
    for (C = 0; C < n_c; C++) {
        int cell;
        int64_t P = find_node(lk, n_p, fdiv2(ijk_c[3 * C]), fdiv2(ijk_c[3 * C + 1]), fdiv2(ijk_c[3 * C + 2]));
        if (P < 0 || rslot_p[P] < 0) { free(lk); return -1; }
        for (cell = 0; cell < NCELL; cell++) {
            int64_t g[3] = {8 * (int64_t)ijk_c[3 * C] + (cell & 7), 8 * (int64_t)ijk_c[3 * C + 1] + ((cell >> 3) & 7),
                            8 * (int64_t)ijk_c[3 * C + 2] + ((cell >> 6) & 7)};
            int64_t pg[3] = {fdiv2(g[0]), fdiv2(g[1]), fdiv2(g[2])};
            int pcell = (int)((pg[0] - 8 * (int64_t)ijk_p[3 * P]) + 8 * (pg[1] - 8 * (int64_t)ijk_p[3 * P + 1])
                              + 64 * (pg[2] - 8 * (int64_t)ijk_p[3 * P + 2]));
            const double *L = &Lp[(P * NCELL + pcell) * 20];
            const double *XP = &X_p[(rslot_p[P] * NCELL + pcell) * 3];
            double Y[3], z[3], L1[3], L2[9], L3[27];
            double *o = &Lch[(C * NCELL + cell) * 20];
            int a, b, c;
            if (refined_c[C]) {
                for (a = 0; a < 3; a++) Y[a] = X_c[(rslot_c[C] * NCELL + cell) * 3 + a];
            } else {
                for (a = 0; a < 3; a++) Y[a] = origin[a] + ((double)g[a] + 0.5) * h_c;
            }
            for (a = 0; a < 3; a++) z[a] = Y[a] - XP[a];
            for (a = 0; a < 3; a++) {
                L1[a] = L[1 + a];
                for (b = 0; b < 3; b++) {
                    L2[a * 3 + b] = L[sym2(a, b)];
                    for (c = 0; c < 3; c++) L3[(a * 3 + b) * 3 + c] = L[sym3(a, b, c)];
                }
            }
            {
                double s = L[0];
                for (a = 0; a < 3; a++) {
                    s += L1[a] * z[a];
                    for (b = 0; b < 3; b++) {
                        s += 0.5 * L2[a * 3 + b] * z[a] * z[b];
                        for (c = 0; c < 3; c++) s += L3[(a * 3 + b) * 3 + c] * z[a] * z[b] * z[c] / 6.0;
                    }
                }
                o[0] += s;
            }
            for (a = 0; a < 3; a++) {
                double s = L1[a];
                for (b = 0; b < 3; b++) {
                    s += L2[a * 3 + b] * z[b];
                    for (c = 0; c < 3; c++) s += 0.5 * L3[(a * 3 + b) * 3 + c] * z[b] * z[c];
                }
                o[1 + a] += s;
            }
            for (a = 0; a < 3; a++)
                for (b = a; b < 3; b++) {
                    double s = L2[a * 3 + b];
                    for (c = 0; c < 3; c++) s += L3[(a * 3 + b) * 3 + c] * z[c];
                    o[sym2(a, b)] += s;
                    for (c = b; c < 3; c++) o[sym3(a, b, c)] += L3[(a * 3 + b) * 3 + c];
                }
            for (a = 0; a < 3; a++) Lcch[(C * NCELL + cell) * 3 + a] += Lcp[(P * NCELL + pcell) * 3 + a];
        }
    }
    free(lk);
    return 0;
}

/* direct N^2: Phi_i = -G sum_{j!=i} m_j / r_ij, g_i = -G sum m_j (x_i-x_j)/r_ij^3 */
void oc_direct(int64_t n, const double *x, const double *m, double G, double *phi, double *g)
{
    int64_t i, j;
    for (i = 0; i < n; i++) {
        double p = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (j = 0; j < n; j++) {
            double R0, R1, R2, r2, r, r3;
            if (j == i) continue;
            R0 = x[3 * i] - x[3 * j];
            R1 = x[3 * i + 1] - x[3 * j + 1];
            R2 = x[3 * i + 2] - x[3 * j + 2];
            r2 = R0 * R0 + R1 * R1 + R2 * R2;
            r = sqrt(r2);
            r3 = r * r2;
            p += -m[j] / r;
            a0 += -m[j] * R0 / r3;
            a1 += -m[j] * R1 / r3;
            a2 += -m[j] * R2 / r3;
        }
        phi[i] = G * p;
        g[3 * i] = G * a0;
        g[3 * i + 1] = G * a1;
        g[3 * i + 2] = G * a2;
    }
}

/* ------------------------------------------------------------------------ */
/* C7: level-local force / torque invariants                                 */
/* ------------------------------------------------------------------------ */
/*
 * For cells with (m, X, M[20]) and same-level outputs (L[20], Lc[3]):
 *   F_A = -[ m_A (L1 + Lc) + 1/2 M2_bc L3_abc ]
 *   tau_A = X_A x F_A - eps_abc ( M2_bd L2_cd + 1/2 M3_bde L3_cde )
 * Returns sums F[3], T[3] and the scales sum|F_A|, sum|tau_A| (Euclidean).
 */
void oc_level_invariants(int64_t n, const double *m, const double *X, const double *M,
                         const double *L, const double *Lc, double *F, double *T, double *scale)
{
    int64_t q;
    int a, b, c, d, e;
    F[0] = F[1] = F[2] = T[0] = T[1] = T[2] = 0.0;
    scale[0] = scale[1] = 0.0;
    for (q = 0; q < n; q++) {
        const double *Mq = &M[q * 20], *Lq = &L[q * 20];
        double M2[9], M3[27], L2[9], L3[27], f[3], tau[3], inner[3];
        for (a = 0; a < 3; a++)
            for (b = 0; b < 3; b++) {
                M2[a * 3 + b] = Mq[sym2(a, b)];
                L2[a * 3 + b] = Lq[sym2(a, b)];
                for (c = 0; c < 3; c++) {
                    M3[(a * 3 + b) * 3 + c] = Mq[sym3(a, b, c)];
                    L3[(a * 3 + b) * 3 + c] = Lq[sym3(a, b, c)];
                }
            }
        for (a = 0; a < 3; a++) {
            double s = m[q] * (Lq[1 + a] + Lc[q * 3 + a]);
            for (b = 0; b < 3; b++)
                for (c = 0; c < 3; c++) s += 0.5 * M2[b * 3 + c] * L3[(a * 3 + b) * 3 + c];
            f[a] = -s;
        }
        /* inner[a] = eps_abc W_bc, W_bc = M2_bd L2_cd + 1/2 M3_bde L3_cde */
        {
            double W[9];
            for (b = 0; b < 3; b++)
                for (c = 0; c < 3; c++) {
                    double s = 0.0;
                    for (d = 0; d < 3; d++) {
                        s += M2[b * 3 + d] * L2[c * 3 + d];
                        for (e = 0; e < 3; e++) s += 0.5 * M3[(b * 3 + d) * 3 + e] * L3[(c * 3 + d) * 3 + e];
                    }
                    W[b * 3 + c] = s;
                }
            inner[0] = W[1 * 3 + 2] - W[2 * 3 + 1];
            inner[1] = W[2 * 3 + 0] - W[0 * 3 + 2];
            inner[2] = W[0 * 3 + 1] - W[1 * 3 + 0];
        }
        {
            const double *x = &X[q * 3];
            tau[0] = x[1] * f[2] - x[2] * f[1] - inner[0];
            tau[1] = x[2] * f[0] - x[0] * f[2] - inner[1];
            tau[2] = x[0] * f[1] - x[1] * f[0] - inner[2];
        }
        for (a = 0; a < 3; a++) { F[a] += f[a]; T[a] += tau[a]; }
        scale[0] += sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
        scale[1] += sqrt(tau[0] * tau[0] + tau[1] * tau[1] + tau[2] * tau[2]);
    }
}

/* ------------------------------------------------------------------------ */
/* C2/C6: exactly-once coverage by brute force over all finest-cell pairs    */
/* ------------------------------------------------------------------------ */
/*
 * Leaf cells given by (level, global cell coords).  For every unordered pair
 * count the levels l <= min(la, lb) at which the pair is taken: ancestors
 * g >> (la - l); node at level l is refined iff l < la; class by
 * oc_pair_class (root rule at l = 0); taken unless near and both refined.
 * hist[k] += number of pairs taken exactly k times (k = 0..3, 3 = ">= 3").
 */
void oc_coverage(double theta, int64_t n, const int32_t *lev, const int64_t *g, int64_t *hist)
{
    double R2 = oc_R2(theta);
    int64_t a, b;
    hist[0] = hist[1] = hist[2] = hist[3] = 0;
    for (a = 0; a < n; a++)
        for (b = a + 1; b < n; b++) {
            int lmin = lev[a] < lev[b] ? lev[a] : lev[b];
            int l, cnt = 0;
            for (l = 0; l <= lmin; l++) {
                int64_t ga[3], gb[3];
                int k, cls;
                for (k = 0; k < 3; k++) {
                    ga[k] = g[3 * a + k] >> (lev[a] - l);
                    gb[k] = g[3 * b + k] >> (lev[b] - l);
                }
                cls = oc_pair_class(R2, l == 0, ga, gb);
                if (cls == 0) continue;
                if (cls == 2 && l < lev[a] && l < lev[b]) continue;
                cnt++;
            }
            hist[cnt > 3 ? 3 : cnt]++;
        }
}
