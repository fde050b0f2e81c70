// internal.cuh — device data structures shared by the libpdcs kernels.
//
// Layout in HBM: structure-of-arrays fp64 vectors,
// CSR(K~) and CSR(K~^T) with int32 row pointers / column ids, one byte of
// element kind per row and per column, and a small control block (Ctl) that
// holds every scalar of Alg. 1 on the device so that decisions never need a
// host round trip.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace pdcs {

constexpr int kThreads = 256;          // CTA size of the streaming kernels
constexpr int kThreadsSmall = 64;
constexpr int kNClass = 5;             // cone block size classes: thread, warp, cta, cluster, grid
constexpr int kClusterCtas = 8;        // CTAs per thread-block cluster of the cluster class      // CTA size of the thread-per-cone kernel (spreads cones over all SMs)
constexpr int kCtaPerSm = 4;           // resident CTAs per SM targeted by grid sizing
constexpr double kRsqrt2 = 0.70710678118654752440;  // 1/sqrt(2), RSOC rotation

enum Cone : int32_t { C_ZERO = 0, C_NONNEG = 1, C_SOC = 2, C_RSOC = 3, C_EXP = 4, C_DEXP = 5 };

// Per-element kinds.  Columns: box types for x_1, zero/nonneg coordinates of
// K_p, or "inside a block cone".  Rows: free (Zero cone), nonneg, or block.
enum ElemKind : uint8_t {
  EK_FREE = 0,     // box (-inf, inf)  /  row: y free (Zero constraint cone)
  EK_NONNEG = 1,   // x2 coordinate in R_+ block / row: y >= 0
  EK_ZERO = 2,     // x2 coordinate in a Zero block: x = 0
  EK_BLOCK = 3,    // coordinate of an SOC/RSOC/EXP/DEXP block
  EK_LO0 = 4,      // box [0, inf)
  EK_LO = 5,       // box [l, inf)
  EK_UP = 6,       // box (-inf, u]
  EK_BOTH = 7      // box [l, u]
};

// Block cone descriptor (one per SOC/RSOC/EXP/DEXP block).
struct Block {
  int64_t off;     // first coordinate (column index for primal blocks, local row for dual)
  int32_t kind;    // Cone
  int32_t dim;
};

// One row-length class of a CSR SpMV plan: V lanes per row (V in 1,4,8,16,32)
// or V == 0 for one CTA per row.  rows == nullptr means the contiguous range
// [range_begin, range_begin + nrows).
struct SpmvClass {
  int32_t V;
  int32_t ncta;
  int64_t nrows;
  int64_t range_begin;
  const int32_t* rows;
};
constexpr int kMaxClasses = 6;
struct SpmvPlan {
  SpmvClass cls[kMaxClasses];
  int32_t ncls;
  int32_t total_cta;
};

struct DevCsr {
  int64_t m = 0, n = 0, nnz = 0;
  int32_t* ptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  SpmvPlan plan{};
  int csr_u = 8;          // entries in flight per lane of the CSR kernel (8 or 4, setup autotune)
};

// Solver control block, device resident (all scalars of Alg. 1).
struct Ctl {
  // step-size state (AdaptiveStepPDHG)
  double eta, eta_init, omega, beta, tau, sigma;
  double eta_used;           // step of the last accepted trial
  double ha, hb;             // Halpern coefficients (k+1)/(k+2), 1/(k+2)
  double hbeta;              // beta used by the last accepted step
  double Wsum;               // sum of eta over the epoch (average weight)
  double r_start;            // beta window start residual (reading A9)
  double last_num, last_cross, last_dxx, last_dyy;
  // restart state
  double e_anchor, e_prev, best_e;
  double kkt[2][5];          // Eq. 9 of the two candidates (err_p, err_d, err_gap, pobj, dobj)
  double best_kkt[5];
  double dist[2][2];         // ||x_c - x0||, ||y_c - y0|| per candidate
  double tol;
  int64_t k, total, trials, restarts, rejects;
  int32_t accepted, status, store_kty, need_check;
  int32_t restart, use_avg, best_flag, done;
  int32_t vanilla, ncand;
  int32_t stop_at_tol, pad2;
  double red3[3];            // trial sums (dxx, dyy, cross) when reduced outside k_decide
  double kred[20];           // Eq. 9 reductions (10 per candidate) before the decision
  // parameters
  double ls_shrink, ls_grow, beta_max, suff, nec, art;
  int32_t ls_max_rejects, refl_window, check_interval, pad;
  int64_t checks;            // Eq. 9 checks run by the iteration (matrix-pass accounting)
};

// Partial-sum slots: every reducing kernel writes NACC doubles per CTA.
constexpr int kAcc = 3;      // trial: (dxx) | (dyy, cross)
constexpr int kKAcc = 20;    // KKT: 10 per candidate (2 candidates)

}  // namespace pdcs
