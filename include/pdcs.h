/*
 * pdcs.h — C ABI of libpdcs.so, the B200-native (sm_100a, fp64) hot path of
 * PDCS (arxiv 2505.00311): restarted, reflected-Halpern PDHG with adaptive
 * steps, primal weights, Ruiz/Pock-Chambolle rescaling and projections onto
 * diagonally rescaled cones.
 *
 * Problem (§2 Eq. 1):
 *     min <c, x>  s.t.  G x - h in K_d^*,   l <= x_1 <= u,   x_2 in K_p
 * with x = (x_1 in R^{n1}, x_2 in R^{n2}), G in R^{m x n} (CSR, fp64).
 * Dual (Eq. 2-3):  y in K_d, lambda = c - G^T y.
 *
 * Conventions (every entry point):
 *   - Plain pointers and sizes only; no framework types.
 *   - Ownership: the caller owns every input array; the library deep-copies
 *     at create/set time into device memory it allocates (cudaMalloc on the
 *     context's device) and frees at pdcs_destroy.  Output arrays are
 *     caller-allocated with the documented sizes.
 *   - mem_kind says whether input pointers are host (PDCS_MEM_HOST) or device
 *     (PDCS_MEM_DEVICE) memory.  Output pointers follow the same mem_kind.
 *   - Errors: a pdcs_status code; the library never aborts.  The message of the
 *     last failure on a context is returned by pdcs_last_error(ctx).  On error
 *     the context stays valid unless documented otherwise.
 *   - Call order: pdcs_create -> pdcs_set_cones -> (pdcs_iterate | pdcs_kkt |
 *     pdcs_solve | pdcs_get_*)* -> pdcs_destroy.  Violations: PDCS_ERR_STATE.
 *   - A context is single-owner and not thread-safe.  All work is enqueued on
 *     the stream given at create (NULL = legacy default stream); functions
 *     that return host data synchronise that stream.
 *   - No CPU fallback: without a usable sm_100 device pdcs_create fails with
 *     PDCS_ERR_CUDA.
 */
#ifndef PDCS_H_
#define PDCS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pdcs_ctx pdcs_ctx;

typedef enum {
  PDCS_OK = 0,
  PDCS_ERR_ARG = 1,       /* null pointer / bad enum / bad size */
  PDCS_ERR_DIM = 2,       /* CSR shape inconsistent (row_ptr not monotone, col out of range) */
  PDCS_ERR_BOUNDS = 3,    /* l_i > u_i, or NaN bound */
  PDCS_ERR_NONFINITE = 4, /* non-finite matrix entry, c or h */
  PDCS_ERR_CONE = 5,      /* bad cone kind/dim, dims do not sum to n2 / m */
  PDCS_ERR_SHARD = 6,     /* a SOC/RSOC/exp row cone straddles this rank's row range (Zero / NonNeg runs may be cut) */
  PDCS_ERR_CUDA = 7,      /* CUDA runtime error (incl. no sm_100 device) */
  PDCS_ERR_NCCL = 8,      /* NCCL error */
  PDCS_ERR_NUMERICAL = 9, /* eta underflow, > ls_max_rejects line-search rejects */
  PDCS_ERR_STATE = 10     /* call order violated */
} pdcs_status;

/* Cone kinds.  In the primal list they are the blocks of K_p
 * over x[n1:n].  In the row list they are the CONSTRAINT cones C_b of
 * G x - h in C_b (the blocks of K_d^*), so the dual y_b lives in C_b^*:
 * ZERO rows are equalities (y free), NONNEG rows are >= (y >= 0), EXP rows
 * mean G x - h in K_exp (y in K_exp^*), DUAL_EXP rows G x - h in K_exp^*.
 * RSOC is {(a,b,z): a,b >= 0, ||z||^2 <= 2ab}.
 * Dims: SOC >= 2, RSOC >= 3, EXP = DUAL_EXP = 3, ZERO/NONNEG >= 1. */
typedef enum {
  PDCS_CONE_ZERO = 0,
  PDCS_CONE_NONNEG = 1,
  PDCS_CONE_SOC = 2,
  PDCS_CONE_RSOC = 3,
  PDCS_CONE_EXP = 4,
  PDCS_CONE_DUAL_EXP = 5
} pdcs_cone_kind;

typedef enum { PDCS_MEM_HOST = 0, PDCS_MEM_DEVICE = 1 } pdcs_mem_kind;

typedef enum {
  PDCS_OPTIMAL = 0,
  PDCS_ITERATION_LIMIT = 1,
  PDCS_TIME_LIMIT = 2,
  PDCS_NUMERICAL_ERROR = 3,
  PDCS_RUNNING = 4
} pdcs_solve_status;

/* Iterate selectors for pdcs_get_iterate / pdcs_kkt. */
typedef enum {
  PDCS_CURRENT = 0,   /* z^{t,k}: the current (Halpern) iterate */
  PDCS_PDHG_OUT = 1,  /* z^: the last accepted PDHG output (always feasible) */
  PDCS_ANCHOR = 2,    /* z^{t,0}: restart anchor */
  PDCS_BEST = 3,      /* best-ever evaluated candidate (returned by pdcs_solve) */
  PDCS_CANDIDATE = 4  /* last restart candidate */
} pdcs_which;

typedef enum { PDCS_SCALED = 0, PDCS_ORIGINAL = 1 } pdcs_space;

/* Solver parameters (defaults in brackets via
 * pdcs_default_params).  Layout is part of the ABI. */
typedef struct {
  double tol;             /* [1e-6] Eq. 9 termination threshold */
  int64_t max_iters;      /* [1e6] accepted inner iterations for pdcs_solve */
  double time_limit_s;    /* [0 = none] */
  int32_t ruiz_iters;     /* [10] Ruiz rounds */
  int32_t pock_chambolle; /* [1] one Pock-Chambolle pass, alpha = 1 */
  int32_t check_interval; /* [40] Eq. 9 / restart cadence */
  int32_t vanilla_pdhg;   /* [0] 1: plain PDHG, tau = sigma = 0.9/||G||_2, no
                             scaling/Halpern/restarts */
  double eta0;            /* [0 = 1/||K~||_inf] initial step (vanilla: the fixed step) */
  double omega0;          /* [0 = ||c~||_inf/||h~||_inf clipped to [1e-4,1e4]] */
  double beta_max;        /* [1] reflection parameter cap */
  int32_t refl_window;    /* [40] beta window (reading A9) */
  int32_t pad0;
  double restart_suff;    /* [0.2]  */
  double restart_nec;     /* [0.8]  */
  double restart_art;     /* [0.36] */
  double ls_shrink;       /* [0.5]  */
  double ls_grow;         /* [1.05] */
  int32_t ls_max_rejects; /* [60]   */
  int32_t verbose;        /* [0]    */
} pdcs_params;

/* Eq. 9 residuals on the ORIGINAL problem. */
typedef struct {
  double err_p, err_d, err_gap, pobj, dobj;
} pdcs_kkt_t;

typedef struct {
  int32_t status;         /* pdcs_solve_status */
  int32_t pad;
  pdcs_kkt_t kkt;         /* residuals of the returned (best) point */
  int64_t iters;          /* accepted inner iterations */
  int64_t trials;         /* PDHG trials incl. line-search rejects */
  int64_t restarts;
  int64_t spmv_K, spmv_KT; /* matrix passes over K~ / K~^T: one K sweep per trial (K x^ and
                             K x together), one K^T sweep per accepted step, and per Eq. 9
                             check K^T y^ (+ K xbar and K^T ybar for the average candidate) */
  double eta, omega, beta;
  double solve_seconds;
} pdcs_result_t;

/* Fill p with the defaults listed above. */
void pdcs_default_params(pdcs_params *p);

/* Create a context: validate and deep-copy the problem, build CSR(K) and
 * CSR(K^T) on the device, and (unless vanilla) apply Ruiz + Pock-Chambolle
 * rescaling on the device.
 *   m_global        rows of G over all ranks
 *   n, n1           columns of G; the first n1 are box variables
 *   row_begin/end   this rank's rows [row_begin, row_end) (0, m_global unsharded)
 *   row_ptr [rows+1] int64, 0-based local offsets; col_idx [nnz] int32 global
 *                    columns, strictly increasing within a row; vals [nnz]
 *   c [n], h [rows], l [n1], u [n1] (+-INFINITY allowed in l, u)
 *   p               parameters (NULL: defaults)
 *   device          CUDA device ordinal; cuda_stream a cudaStream_t or NULL
 *   nccl_unique_id  128-byte ncclUniqueId when world > 1, else NULL
 * Row-sharded contexts (world > 1, or world == 1 with an id) exchange only
 * all-reduces; every decision of Alg. 1 is taken from
 * all-reduced values, so all ranks take the same decisions and stop at the
 * same Eq. 9 check (the time limit is decided collectively).  Their iteration
 * is recorded into the CUDA graph with the NCCL calls inside
 * (PDCS_DIST_GRAPH=0: host-driven loop).
 * Errors: ARG, DIM, BOUNDS, NONFINITE, CUDA, NCCL.  *out is NULL on error;
 * the message is then available from pdcs_last_error(NULL). */
pdcs_status pdcs_create(pdcs_ctx **out, int64_t m_global, int64_t n, int64_t n1,
                        int64_t row_begin, int64_t row_end, const int64_t *row_ptr,
                        const int32_t *col_idx, const double *vals, const double *c,
                        const double *h, const double *l, const double *u,
                        const pdcs_params *p, int device, void *cuda_stream, int mem_kind,
                        const void *nccl_unique_id, int rank, int world);

/* Cone lists (host arrays always): npc primal blocks (kinds pk, dims pdim)
 * over x[n1:n] and nrc row blocks over the GLOBAL rows (kinds rk, dims rdim).
 * Scaling (Ruiz + PC) runs here because RSOC blocks need equal leading
 * divisors.  Errors: ARG, CONE, SHARD, STATE, CUDA. */
pdcs_status pdcs_set_cones(pdcs_ctx *ctx, const int32_t *pk, const int64_t *pdim, int64_t npc,
                           const int32_t *rk, const int64_t *rdim, int64_t nrc);

/* Run exactly n_inner ACCEPTED inner iterations of Alg. 1
 * including the Eq. 9 checks, restarts and primal-weight updates at the
 * check cadence; does not stop at tol.  out (may be NULL) receives counters.
 * Errors: STATE (also after a pdcs_solve that finished: OPTIMAL, ITERATION_ or
 * TIME_LIMIT until pdcs_set_tolerance; NUMERICAL_ERROR for good), NUMERICAL,
 * CUDA, NCCL. */
pdcs_status pdcs_iterate(pdcs_ctx *ctx, int64_t n_inner, pdcs_result_t *out);

/* Eq. 9 residuals of the selected iterate, ORIGINAL space. */
pdcs_status pdcs_kkt(pdcs_ctx *ctx, int which, pdcs_kkt_t *out);

/* Alg. 1 until max(err_p, err_d, err_gap) <= tol or a limit; returns the best
 * evaluated point's residuals (reading A15).  Continues from the current state.
 * On a context whose last solve finished (OPTIMAL, ITERATION_ or TIME_LIMIT)
 * it runs nothing and reports that result again (pdcs_set_tolerance continues
 * the trajectory).  Errors: STATE (after NUMERICAL_ERROR), CUDA, NCCL; a line-
 * search failure is reported as status NUMERICAL_ERROR with PDCS_OK. */
pdcs_status pdcs_solve(pdcs_ctx *ctx, pdcs_result_t *out);

/* Set the stopping tolerance (>= 0) and solve time limit (seconds, 0 = none)
 * for later pdcs_solve calls, and clear a finished status (OPTIMAL, ITERATION_
 * or TIME_LIMIT) so the next pdcs_solve continues from the current state: the
 * iterate, anchor, average, eta, omega and counters are kept.  Used to time
 * one trajectory to several tolerances (1e-3 and
 * 1e-6).  Errors: ARG (negative / NaN), STATE (before set_cones, or after
 * NUMERICAL_ERROR), CUDA. */
pdcs_status pdcs_set_tolerance(pdcs_ctx *ctx, double tol, double time_limit_s);

/* Copy an iterate out: x [n], y [local rows]; space SCALED or ORIGINAL
 * (x = x~/q, y = y~/r, reading A2).  Output memory per the create mem_kind. */
pdcs_status pdcs_get_iterate(pdcs_ctx *ctx, int which, int space, double *x, double *y);

/* Set the current iterate from ORIGINAL-space x [n], y [local rows] and start
 * a new epoch there (as a restart does): anchor z0 = PDHG
 * output = the point, its anchor KKT error evaluated, the inner counter k,
 * the average sums and weight W, beta (= beta_max) and the previous-check
 * error reset.  eta, omega and the total / trial / restart counters are kept. */
pdcs_status pdcs_set_iterate(pdcs_ctx *ctx, const double *x, const double *y);

/* Checkpoint / resume of the full Alg. 1 state in SCALED space.  These two
 * calls REPLACE SURVEY §8(b)'s pdcs_set_decision_trace: instead of forcing the
 * oracle's discrete decisions onto the GPU, the parity tests load the oracle's
 * exact state every few iterations and compare the decisions both sides then
 * take (checkpoint shadowing).  The state is:
 *   x, y (current z^{t,k}), x0, y0 (anchor z^{t,0}), xsum, ysum (sum eta z of
 *   the epoch) — n / local-rows doubles each, memory per the create mem_kind;
 *   sc[13] = eta, eta_init, omega, beta, W, r_start, e_anchor, e_prev, best_e,
 *            k, total, trials, restarts (host array).
 * pdcs_set_state recomputes the cached products K~x, K~^T y, K~x0, K~^T y0 on
 * the device.  Any pointer may be NULL on get.  Errors: STATE, ARG, CUDA. */
pdcs_status pdcs_get_state(pdcs_ctx *ctx, double *x, double *y, double *x0, double *y0,
                           double *xsum, double *ysum, double *sc);
pdcs_status pdcs_set_state(pdcs_ctx *ctx, const double *x, const double *y, const double *x0,
                           const double *y0, const double *xsum, const double *ysum,
                           const double *sc);

/* Row and column divisors r [local rows], q [n] (K~ = diag(1/r) G diag(1/q)). */
pdcs_status pdcs_get_scaling(pdcs_ctx *ctx, double *r, double *q);

/* Device-side timing of the kernels launched by the last pdcs_iterate call:
 * names/ms accumulated per kernel family (diagnostics; fills up to cap
 * entries, returns the count). */
int pdcs_kernel_times(pdcs_ctx *ctx, char (*names)[32], double *ms, int64_t *launches, int cap);
void pdcs_enable_timing(pdcs_ctx *ctx, int on);

/* Control-state snapshot (diagnostics / decision-trace comparison).  Fills up
 * to cap doubles: eta, omega, beta, k, total, trials, restarts, e_anchor, W,
 * eta_init, kkt_cur[5], kkt_avg[5], e_prev, best_e, use_avg, restart flag,
 * last line-search numerator and cross term, then setup diagnostics: tiled_K
 * (0/1), autotune ms (CSR, tiled) for K, the same three for K^T, host build
 * ms of the tiled K and K^T formats, wall ms of pdcs_create and of
 * pdcs_set_cones, and 1 if the box columns are stored in a locality order
 * (every x-side array crossing this ABI stays in the
 * caller's order), then the L2 column panels of K~ and K~^T (DESIGN.md
 * §7.7): number of panels kept (0 = CSR / tiled sweep) and the autotune ms of
 * the CSR and the panelled sweep, for K~ then K~^T, then the fused combine
 * of the tiled sweeps: kept (0/1) and its autotune ms, for
 * K~ then K~^T, then the CSR kernel's entries in flight per lane (8 or 4)
 * for K~ and K~^T.  Returns the number of values written (<= 49). */
int pdcs_get_scalars(pdcs_ctx *ctx, double *out, int cap);

/* Number of kernel launches issued by the last pdcs_iterate call. */
int64_t pdcs_launch_count(const pdcs_ctx *ctx);

const char *pdcs_last_error(const pdcs_ctx *ctx);
void pdcs_destroy(pdcs_ctx *ctx);

/* Host-only diagnostic: build the column-tiled format of the CSR (row_ptr
 * [rows+1], col [nnz], host memory) on host threads exactly as pdcs_create /
 * pdcs_set_cones do, and report out[0] = total build ms, out[1] = ms of the
 * threaded per-range phase, out[2] = staged nonzeros.  elem 2 = the K sweep's
 * (x^, x) pair gather, 1 = the K^T sweep's doubles.  Returns 3, or 0 on bad
 * arguments.  No device is touched. */
int pdcs_tiled_build_host(const int64_t *row_ptr, const int32_t *col, int64_t rows, int64_t nvec, int elem,
                          double *out);

/* Device diagnostic (needs a GPU): build the column-tiled layout both ways the
 * library can, all on the host, and deferred (host structure, shared-memory
 * bank balancing and sliced re-layout on the device; the solver's default,
 * PDCS_TILE_DEVICE=0 turns it off), and compare them entry by entry.
 * out[0] = mismatching entries (column ids, value permutation, row pointers,
 * block bases, segment descriptors); out[1] = all-host ms; out[2] = deferred
 * host ms; out[3] = device ms; out[4] = layout entries.  Returns 5, 0 on bad
 * arguments (or when the deferred build does not apply), -1 on a CUDA error. */
int pdcs_tiled_device_check(const int64_t *row_ptr, const int32_t *col, int64_t rows, int64_t nvec, int elem,
                            double *out);

/* Diagnostic: the device structure build of the column-tiled layout (the
 * solver's default: the entries of the CSR never pass through
 * the host) against the all-host build, entry by entry: column ids and value
 * permutation of staged and direct entries, row pointers, row order, block
 * bases, segment descriptors, work items, batches, chunks.  row_ptr[rows+1],
 * col[nnz] are HOST arrays (copied to the device here).  out[0] = mismatches;
 * out[1] = all-host ms; out[2] = device-build ms; out[3] = staged entries;
 * out[4] = layout entries.  Returns 5, 0 on bad arguments (or when the
 * sliced, balanced layout is switched off), -1 on a CUDA error. */
int pdcs_tiled_devbuild_check(const int64_t *row_ptr, const int32_t *col, int64_t rows, int64_t nvec, int elem,
                              double *out);

/* Host-only diagnostic, no GPU needed: build the column-tiled layout
 * of a CSR structure (row_ptr[rows+1], col[nnz], valid and
 * sorted; elem = 2 for the (x^, x) pair gather of K, 1 for the y gather of
 * K^T) and model the shared-memory gathers of its partial kernel.  Writes up to
 * cap doubles: nnz, staged nnz, quads, pad entries, staged segments, work
 * items, modeled ld.shared instructions, modeled shared-memory wavefronts,
 * host build ms, a lower bound on those wavefronts for the layout's row
 * grouping (per phase: max(active slots, entries of the most loaded bank
 * group)), and the number of structure errors (entries stored under a wrong
 * column, twice, or not at all; 0 for a correct layout).  Returns the number
 * written (0 on bad arguments). */
int pdcs_tiled_layout_stats(const int64_t *row_ptr, const int32_t *col, int64_t rows, int64_t nvec, int elem,
                            double *out, int cap);

/* ---- Standalone multi-cone projection (§4 "GPU
 * implementation", Table "Projection strategies", Figs. 3-4; Thm 1
 * PAPER.md:651-661 and Thm 4 PAPER.md:1272-1311 for the rescaled cones).
 *
 * A plan holds the block descriptors of one cone product K = K_1 x ... x K_nb,
 * block b of kind kinds[b] (PDCS_CONE_SOC dim >= 2, PDCS_CONE_RSOC dim >= 3,
 * PDCS_CONE_EXP / PDCS_CONE_DUAL_EXP dim 3) covering dims[b] consecutive
 * coordinates, in order, of a vector of length sum(dims).  team selects the
 * parallel strategy for the SOC/RSOC blocks: -1 the solver's size classes
 * (thread <= 32, warp <= 512, CTA <= 4096, 8-CTA cluster <= 131072, whole
 * grid beyond); 0..4 forces thread / warp / CTA / cluster / grid for every one
 * of them (the paper's thread-, block- and grid-wise strategies).  Exp blocks
 * are always one thread per cone.  kinds/dims are host arrays,
 * copied; the plan owns device memory on `device` until pdcs_proj_destroy.
 * Errors: PDCS_ERR_ARG (null lists, bad team/device), PDCS_ERR_CONE (bad
 * kind/dim), PDCS_ERR_CUDA (no sm_100 device).  The message is returned by
 * pdcs_last_error(NULL). */
typedef struct pdcs_proj pdcs_proj;
pdcs_status pdcs_proj_create(pdcs_proj **out, int device, const int32_t *kinds, const int64_t *dims,
                             int64_t nblocks, int team);
/* out = P_{diag(D) K}(v), blockwise (the rescaled cone D K = {D w : w in K}).
 * v, out: device arrays of sum(dims) doubles (may not alias); D: device array
 * of positive multipliers of the same length, or NULL for K itself (unit
 * scaling).  RSOC blocks need D[0] == D[1] (reading A21).  Enqueued on
 * `stream` (a cudaStream_t, NULL = legacy default); does not synchronise. */
pdcs_status pdcs_proj_run(pdcs_proj *plan, const double *D, const double *v, double *out, void *stream);
/* Blocks and grid size per team (thread, warp, CTA, cluster, grid) into
 * counts[5] / grids[5] (either may be NULL).  Returns 5. */
int pdcs_proj_info(const pdcs_proj *plan, int64_t *counts, int64_t *grids);
void pdcs_proj_destroy(pdcs_proj *plan);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 broadcasts it). */
pdcs_status pdcs_nccl_unique_id(void *out128);

/* ---- Device memory: a caller allocator for every later
 * context's device buffers (matrices, tiled formats, vectors, scratch).
 * alloc(bytes, user) returns device memory on the context's device or NULL
 * (the call then fails with PDCS_ERR_CUDA); free(ptr, user) releases it.
 * Process-wide; set it before pdcs_create and keep it until every context
 * using it is destroyed.  NULL, NULL restores the default: a library-owned
 * stream-ordered memory pool per device (cudaMallocFromPoolAsync, used
 * synchronously) that keeps freed memory for later contexts of the process
 * (PDCS_POOL=0: plain cudaMalloc / cudaFree).  Buffers are allocated at
 * create / set_cones time only, never per iteration.
 * Errors: ARG (one function NULL, the other not). */
/* Return the default pool's unused device memory (buffers of destroyed
 * contexts, setup scratch) to the driver; memory of live contexts stays.
 * Process-wide.  Returns the bytes released, -1 on a CUDA error.  The next
 * context then maps its memory afresh (slower setup). */
int64_t pdcs_trim_memory(void);

typedef void *(*pdcs_alloc_fn)(size_t bytes, void *user);
typedef void (*pdcs_free_fn)(void *ptr, void *user);
pdcs_status pdcs_set_allocator(pdcs_alloc_fn alloc, pdcs_free_fn free_fn, void *user);

/* ---- In-process loopback ranks (SURVEY §8(e) tests on one GPU).
 * A loopback group stands in for NCCL when `world` row-sharded contexts live
 * in ONE process on one device, each driven from its own host thread (NCCL
 * refuses two ranks on one device).  Every collective is a host rendezvous of
 * the group followed by a device reduction over the ranks' buffers in rank
 * order, so every rank receives identical bits (as with NCCL).  A rank whose
 * call fails aborts the group: its peers' pending calls fail with
 * PDCS_ERR_NCCL instead of waiting (PDCS_LOOPBACK_TIMEOUT_S, default 600 s,
 * bounds a rendezvous).  The group is owned by the caller and must outlive its
 * contexts.  Loopback contexts run the host-driven loop (no CUDA graph).
 * Errors: ARG (world outside 1..16). */
typedef struct pdcs_loopback pdcs_loopback;
pdcs_status pdcs_loopback_create(pdcs_loopback **out, int world);
void pdcs_loopback_destroy(pdcs_loopback *group);

/* pdcs_create for rank `rank` of a loopback group (world = the group's size);
 * every other argument as pdcs_create. */
pdcs_status pdcs_create_loopback(pdcs_ctx **out, int64_t m_global, int64_t n, int64_t n1,
                                 int64_t row_begin, int64_t row_end, const int64_t *row_ptr,
                                 const int32_t *col_idx, const double *vals, const double *c,
                                 const double *h, const double *l, const double *u,
                                 const pdcs_params *p, int device, void *cuda_stream, int mem_kind,
                                 pdcs_loopback *group, int rank);

#ifdef __cplusplus
}
#endif
#endif /* PDCS_H_ */
