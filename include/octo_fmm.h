/*
 * octo_fmm.h -- C ABI of the B200-native stencil FMM same-level step.
 *
 * What it computes: Octo-Tiger's FMM step 2 ("same-level" interactions,
 * P:L475-481 of /root/reference/PAPER.md): for every cell of every sub-grid
 * (octree node of 8^3 cells) of one octree level, the Taylor-series
 * increments (20 coefficients, order 3) contributed by the cells selected by
 * the opening criterion (1074-element stencil at the paper's
 * parameters), through the three kernels of P:L505-521:
 *   multipole target <- multipole / monopole partner   (M2L, cases 1+2),
 *   monopole target  <- monopole partner               (P2P, case 3),
 *   monopole target  <- multipole partner              (mixed, case 4),
 * plus the angular-momentum correction that makes linear and angular
 * momentum conserve to machine precision.
 * Exact definitions, readings of what the paper leaves open, and the
 * conventions below: DESIGN.md ("Readings", "Conventions").
 *
 * Conventions
 *   - A level is a list of nodes (sub-grids) with integer coordinates
 *     node_ijk at that level; node (I,J,K) holds the cells with global
 *     coordinates 8I..8I+7 (etc.).  Local cell index l = lx + 8 ly + 64 lz.
 *     Cell width h_cell; leaf-cell expansion centre = geometric centre
 *     origin + (g + 1/2) h_cell.
 *   - neighbors[q][27]: node index (into this level's list) of the neighbour
 *     at offset (dx,dy,dz), slot (dx+1) + 3(dy+1) + 9(dz+1); slot 13 = q;
 *     -1 = absent (absent nodes contribute nothing).
 *   - Multipoles (20 coefficients): 0 m; 1-3 dipole (ignored, identically 0
 *     about the centre of mass); 4-9 xx,xy,xz,yy,yz,zz; 10-19 xxx,xxy,xxz,
 *     xyy,xyz,xzz,yyy,yyz,yzz,zzz; full Cartesian moments about the cell's
 *     centre of mass, M_k = sum_i m_i (x_i - X)^k.
 *   - Taylor coefficients (20), same index order, entries of the symmetric
 *     tensors L^(n) of Phi(X + z) = L0 + L_a z_a + 1/2 L_ab z_a z_b
 *     + 1/6 L_abc z_a z_b z_c, Green's function -G/r; ang_corr (3) is the
 *     angular-momentum correction Lc; acceleration g = -(L1 + Lc).
 *   - Refined ("multipole") nodes are listed in node order; the k-th refined
 *     node owns row k of the refined-only arrays (com, mom).
 *
 * Ownership and errors
 *   - The caller owns every argument buffer.  With OCTO_DEVICE, device
 *     buffers passed to load_level are read asynchronously, by the ingest
 *     kernel that the next compute_interactions launches on its stream (one
 *     batched launch for every level loaded since the previous compute), and
 *     must stay alive until that work has completed.  The library owns its internal
 *     device copies, tables, NCCL communicator and (nranks > 1) the CUDA-IPC
 *     receive arena of the exchange; destroy frees them.
 *   - No exceptions cross the ABI.  Functions return OCTO_OK (0) or a
 *     negative code; octo_fmm_last_error(h) returns a message for the last
 *     failure on the handle.  Structure is validated on the host in the
 *     call; the values (m > 0, mom[0] == mono) are validated by the ingest
 *     kernel and reported by the next synchronising call (get_expansions /
 *     get_expansions_compact with OCTO_HOST, or octo_fmm_sync).
 *   - There is no CPU fallback: every compute step runs in the library's
 *     sm_100a kernels; without a usable device the calls return OCTO_ECUDA.
 */
#ifndef OCTO_FMM_H
#define OCTO_FMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCTO_FMM_ABI_VERSION 1

enum {
    OCTO_OK = 0,
    OCTO_EINVAL = -1,   /* null argument, n != 8, theta out of range, level not loaded, bad layout */
    OCTO_ESTRUCT = -2,  /* asymmetric neighbour table, or a refined node with an absent in-domain neighbour (2:1 grading) */
    OCTO_EMASS = -3,    /* a cell with m <= 0 (the AM correction divides by m_A; S:L153 rejects negative density) */
    OCTO_ECUDA = -4,
    OCTO_ENCCL = -5,
    OCTO_ENOMEM = -6
};

/* Memory kinds of caller buffers.  OCTO_HOST_ASYNC (outputs of
 * get_expansions / get_expansions_compact only): a page-locked host
 * destination written by an asynchronous copy on cuda_stream; the call does
 * not synchronise, the results are valid once the caller has synchronised
 * the stream, and deferred errors are reported by the next octo_fmm_sync.
 * It lets a caller pipeline steps (e.g. two handles on two streams, one
 * step's device->host copy overlapping the next step's work). */
enum { OCTO_HOST = 0, OCTO_DEVICE = 1, OCTO_HOST_ASYNC = 2 };

#define OCTO_AM_CORRECTION 1u  /* flags: apply the angular-momentum correction (default on) */
#define OCTO_TIMING 2u          /* flags: record CUDA events around each kernel class of compute_interactions */
#define OCTO_EXTERNAL_BOOTSTRAP 4u /* flags (nranks > 1): create no NCCL communicator; the one-time exchange
                                      set-up (IPC handles and arena offsets of every rank) goes through the
                                      caller's allgather (octo_fmm_set_bootstrap), so several ranks may share
                                      one GPU and the caller's process group (e.g. torch gloo) does the
                                      bootstrap; the exchange transport is the one-sided puts */
#define OCTO_ALL_LEVELS (-1)   /* compute_interactions: every loaded level, one fused launch per kernel */

typedef struct octo_fmm_config {
    int32_t abi_version;      /* OCTO_FMM_ABI_VERSION */
    int32_t n;                /* sub-grid edge, must be 8 */
    double theta;             /* opening parameter, 0.25 <= theta <= 1: parent-level reach <= 3,
                                 so the stencil (cell reach <= 7) stays inside the 26 neighbours; reach 2
                                 (theta >= 1/3) stages an 8^3-parent window, reach 3 a 10^3 one;
                                 the paper's 1074-element stencil is theta in [1/3, 0.353) */
    double G;                 /* gravitational constant applied to the outputs (code units) */
    uint32_t flags;           /* OCTO_AM_CORRECTION */
    int32_t device;           /* CUDA device ordinal */
    int32_t rank;             /* this process's rank (one process per GPU) */
    int32_t nranks;           /* number of ranks; > 1 enables the ghost exchange: one-sided
                                 NVLink stores into the peers' CUDA-IPC receive arenas with
                                 release/acquire epoch flags (default; the environment
                                 variable OCTO_XCHG=nccl selects NCCL send/recv instead) */
    uint8_t nccl_unique_id[128]; /* ncclUniqueId bytes (ignored when nranks == 1) */
} octo_fmm_config;

typedef struct octo_fmm *octo_fmm_t;

/* Create a handle (the same-level step of one theta):
 * validates cfg, builds the per-parity stencil tables on the device, creates
 * the NCCL communicator when nranks > 1 and OCTO_EXTERNAL_BOOTSTRAP is not
 * set (it carries NCCL send/recv, or bootstraps the one-sided exchange's IPC
 * arenas).  Returns OCTO_EINVAL on a bad config (theta outside [0.25, 1],
 * n != 8, rank/nranks inconsistent), OCTO_ECUDA / OCTO_ENCCL / OCTO_ENOMEM
 * otherwise; *out is NULL on failure and octo_fmm_last_error(NULL) holds the
 * message. */
int octo_fmm_create(const octo_fmm_config *cfg, octo_fmm_t *out);

/* Caller-supplied allgather for OCTO_EXTERNAL_BOOTSTRAP handles: gathers
 * `bytes` bytes from every rank into recv[nranks][bytes] in rank order and
 * returns 0 (non-zero = failure, reported as OCTO_ENCCL).  It is called on
 * the calling thread, only from inside compute_interactions when the ghost
 * plan is (re)built (first call after a structure change), and by every rank
 * at the same point of the call sequence (compute_interactions is collective
 * when nranks > 1).  The library keeps fn and ctx until the handle is
 * destroyed; ctx is owned by the caller. */
typedef int (*octo_allgather_fn)(void *ctx, const void *send, void *recv, int64_t bytes);
int octo_fmm_set_bootstrap(octo_fmm_t h, octo_allgather_fn fn, void *ctx);

int octo_fmm_destroy(octo_fmm_t h);

/* Load (or reload) one octree level.
 *   level          level number (0 = root; the root uses the C2 rule)
 *   h_cell, origin cell width at this level and domain origin
 *   n_nodes        nodes in the list (owned + ghost nodes owned by other ranks)
 *   node_ijk       HOST [n_nodes][3] integer node coordinates at this level
 *   refined        HOST [n_nodes] 1 = refined (multipole) node, 0 = leaf (monopole)
 *   neighbors      HOST [n_nodes][27] (see Conventions)
 *   owner          HOST [n_nodes] owning rank, or NULL (all owned by this rank)
 *   mono           [n_nodes][512] cell masses of every node (m = rho h^3 for leaves)
 *   com            [3][n_refined][512] centres of mass of refined nodes' cells
 *   mom            [20][n_refined][512] moments of refined nodes' cells (mom[0] == mono)
 *                  Only the rows of OWNED nodes are read (and, with OCTO_HOST,
 *                  copied to the device); rows of ghost nodes may hold anything:
 *                  their cells arrive through the ghost exchange.
 *   mem            OCTO_HOST or OCTO_DEVICE for mono/com/mom
 * Rows of ghost nodes (owner != rank) are ignored and filled by the exchange.
 * Lifetime: with OCTO_HOST the host rows are copied by cudaMemcpyAsync on
 * cuda_stream, which returns before the copy has run when the buffers are
 * page-locked; the caller keeps them alive and unmodified until cuda_stream
 * has passed the next compute_interactions (or octo_fmm_sync).  With
 * OCTO_DEVICE the same holds for the device buffers (read by the ingest
 * kernel of the next compute_interactions).
 * The structure (node_ijk, refined, neighbors, owner) is cached: reloading a
 * level with identical structure only re-ingests the data. */
int octo_fmm_load_level(octo_fmm_t h, int32_t level, double h_cell, const double origin[3], int64_t n_nodes,
                        const int32_t *node_ijk, const uint8_t *refined, const int32_t *neighbors,
                        const int32_t *owner, const double *mono, const double *com, const double *mom, int32_t mem,
                        void *cuda_stream);

/* Run the same-level step of `level` (or OCTO_ALL_LEVELS) asynchronously on
 * cuda_stream (the four interaction cases of P:L505-521; SURVEY
 * 8(a) a4-a9): ingest of the levels loaded since the last call, ghost
 * exchange (nranks > 1), then the M2L+Lc, mixed and P2P kernels over the
 * owned nodes of every level in one launch each (the root level's kernel on
 * a side stream, joined before the call's work ends).  Levels are
 * independent.  With nranks > 1 the call is COLLECTIVE: every rank makes the
 * same sequence of calls (same `level` arguments), and each call refreshes
 * the ghost cells of every loaded level (one exchange plan over all loaded
 * levels, rebuilt only when a level's structure changes).  Errors:
 * OCTO_EINVAL (level not loaded / no data), OCTO_ESTRUCT (ghost plans that
 * disagree between ranks), OCTO_ECUDA, OCTO_ENCCL (exchange set-up failed;
 * a peer that never signals is reported by the next octo_fmm_sync). */
int octo_fmm_compute_interactions(octo_fmm_t h, int32_t level, void *cuda_stream);

/* Copy the results of `level` out:
 *   taylor   [20][n_owned][512]  (leaf nodes: rows 0..3, rows 4..19 are 0)
 *   ang_corr [3][n_owned][512]
 * n_owned = owned nodes in node order.  Overwrites the caller's buffers.
 * With OCTO_HOST the call synchronises cuda_stream; OCTO_HOST_ASYNC does not. */
int octo_fmm_get_expansions(octo_fmm_t h, int32_t level, double *taylor, double *ang_corr, int32_t mem,
                            void *cuda_stream);

/* The same results in a compact layout without the zero padding of leaf
 * rows 4..19 (about 2.5x fewer bytes to copy):
 *   refined_out [23][n_ref][512]  -- L 0..19 then Lc 0..2 of the owned refined nodes (node order)
 *   leaf_out    [7][n_leaf][512]  -- L 0..3 then Lc 0..2 of the owned leaf nodes (node order)
 * Either output may be NULL; both NULL queries *n_ref / *n_leaf only.  With
 * OCTO_HOST the call synchronises cuda_stream (and reports deferred errors);
 * with OCTO_HOST_ASYNC it does not.  The copies are 2-D DMA copies out of the
 * slot-ordered result buffers (no kernel), ordered on cuda_stream after the
 * compute; do not reuse the handle on another stream before they complete. */
int octo_fmm_get_expansions_compact(octo_fmm_t h, int32_t level, double *refined_out, double *leaf_out,
                                    int64_t *n_ref, int64_t *n_leaf, int32_t mem, void *cuda_stream);

/* Zero-copy access to the library's result buffers for `level` (device
 * pointers).  Node rows are in SLOT order: the n_ref owned refined nodes
 * first, then the owned leaf nodes, node order within each (the order of
 * the compact layout).  taylor = rows 0..3 of every slot [4][n_owned][512]
 * followed by rows 4..19 of the refined slots [16][n_ref][512];
 * ang_corr [3][n_owned][512].  Valid until the level is reloaded with a
 * different structure or the handle is destroyed. */
int octo_fmm_expansions_ptr(octo_fmm_t h, int32_t level, const double **taylor, const double **ang_corr,
                            int64_t *n_owned);

/* Synchronise cuda_stream and report deferred device-side validation errors. */
int octo_fmm_sync(octo_fmm_t h, void *cuda_stream);

/* Stencil introspection (tests): per parity c = cx + 2cy + 4cz, the offsets d
 * (int8 triples) and class (1 far, 2 near) of the level >= 1 stencil.
 * offsets may be NULL to query counts[8]; capacity is per parity. */
int octo_fmm_stencil(octo_fmm_t h, int8_t *offsets, uint8_t *cls, int32_t *counts, int32_t capacity);

/* Interaction counts of the last compute of `level` (0 if not loaded):
 * counts[3] = {P2P, M2L (refined targets), mixed (leaf targets <- refined)};
 * counted on the host from the structure when the level is loaded. */
int octo_fmm_interaction_counts(octo_fmm_t h, int32_t level, int64_t counts[3]);

/* With OCTO_TIMING: per-kernel-class device time (ms) accumulated over the
 * compute_interactions calls since the last query, from CUDA events recorded
 * on the launching stream around each kernel: ms[0] P2P, ms[1] mixed, ms[2]
 * M2L (refined targets), ms[3] ghost exchange (wait/transfer + unpack on the
 * handle's communication stream; 0 when nranks == 1); *calls = number of
 * compute calls summed.  Waits for the
 * recorded events; resets the accumulators. */
int octo_fmm_kernel_times(octo_fmm_t h, double ms[4], int64_t *calls);

/* Kernel launches issued by this handle since creation (bench evidence). */
int64_t octo_fmm_launch_count(octo_fmm_t h);

/* FMM step 1 on the device, producing load_level
 * inputs without a host round trip.  All array arguments are DEVICE pointers
 * in the load_level (ABI) layout unless marked HOST.
 *   p2m: mono[i] = rho[i] * h_cell^3 for n_cells cells (leaf cells).
 *   m2m: for every refined node of a parent level (n_parent_refined, in node
 *        order; parent_rows HOST [n_parent_refined] = their node indices in
 *        the parent list), the cells' mass, centre of mass and 20 moments from
 *        the 8 children on the child level (children HOST [n_parent_refined][8]:
 *        child node index per octant ox + 2 oy + 4 oz).  child_ijk / child_refined
 *        HOST [n_child]; child_com/child_mom rows follow the child level's
 *        refined order.  Writes parent_mono rows parent_rows[k], and rows k of
 *        parent_com [3][n_parent_refined][512], parent_mom [20][n_parent_refined][512]. */
int octo_fmm_p2m(octo_fmm_t h, int64_t n_cells, const double *rho, double h_cell, double *mono, void *cuda_stream);
int octo_fmm_m2m(octo_fmm_t h, int64_t n_parent_refined, const int32_t *parent_rows, const int32_t *children,
                 int64_t n_child, const int32_t *child_ijk, const uint8_t *child_refined, double child_h,
                 const double origin[3], const double *child_mono, const double *child_com, const double *child_mom,
                 double *parent_mono, double *parent_com, double *parent_mom, void *cuda_stream);

/* FMM step 3 on the device.  propagate: after
 * compute_interactions on every level from the root down, add each parent
 * cell's expansion, re-centred by the exact cubic Taylor shift, to its 8
 * children, level by level top-down, in place on the result buffers (Lc is
 * passed down unchanged; reading C8); single rank (nranks == 1).
 * get_field: Phi = L0 and g = -(L1 + Lc) of every owned cell of a level,
 * DEVICE buffers phi[n_owned][512], g[3][n_owned][512] (meaningful at leaf
 * nodes after propagate). */
int octo_fmm_propagate(octo_fmm_t h, void *cuda_stream);
int octo_fmm_get_field(octo_fmm_t h, int32_t level, double *phi, double *g, void *cuda_stream);

/* Multi-rank helpers.  nccl_unique_id: rank 0 creates the id that every rank
 * passes in octo_fmm_config.nccl_unique_id (one fresh id per handle: an id
 * bootstraps exactly one communicator).  exchange_plan: host-only (no
 * CUDA) per-peer ghost cell lists of `rank` for one level, as used by
 * load_level when nranks > 1: entries node * 512 + cell in canonical order
 * (Morton order of node_ijk, then cell); counts[peer*4 + k] for k = send
 * leaf / send refined / receive leaf / receive refined; lists may be NULL
 * (sizes only) or an array of nranks*4 caller buffers. */
int octo_fmm_nccl_unique_id(uint8_t *out128);
int octo_fmm_exchange_plan(double theta, int32_t rank, int32_t nranks, int64_t n_nodes, const int32_t *node_ijk,
                           const uint8_t *refined, const int32_t *neighbors, const int32_t *owner, int64_t *counts,
                           int32_t **lists);

/* Partition helper, host-only (no CUDA): the same-level interaction counts of
 * every node of a level (levels >= 1, C1/C6 readings), counts[node][3] =
 * {P2P, M2L (refined target), mixed (leaf target <- refined)}, as the kernels
 * will evaluate them -- the cost weights of a balanced space-filling-curve
 * partition.  neighbors as in load_level.  Returns
 * OCTO_EINVAL for a theta outside the supported range or null arguments. */
int octo_fmm_node_costs(double theta, int64_t n_nodes, const uint8_t *refined, const int32_t *neighbors,
                        int64_t *counts);

const char *octo_fmm_strerror(int code);
const char *octo_fmm_last_error(octo_fmm_t h);

#ifdef __cplusplus
}
#endif
#endif /* OCTO_FMM_H */
