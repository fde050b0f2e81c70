// kernels.cuh — the PDCS hot-path kernels (Alg. 1) except SpMV.
#pragma once
#include "cones.cuh"
#include "spmv.cuh"

namespace pdcs {

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ double box_proj(uint8_t k, double v, const double* lt, const double* ut,
                                           int64_t j) {
  switch (k) {
    case EK_FREE: return v;
    case EK_NONNEG:
    case EK_LO0: return fmax(v, 0.0);
    case EK_ZERO: return 0.0;
    case EK_LO: return fmax(v, lt[j]);
    case EK_UP: return fmin(v, ut[j]);
    case EK_BOTH: return fmin(fmax(v, lt[j]), ut[j]);
    default: return v;
  }
}

// Partial-sum writer for kernels that are not SpMVs.
template <int NA>
__device__ __forceinline__ void write_partials(Acc<NA>& a, double* part, int64_t slot) {
  cta_write_partials<NA>(a, part, slot);
}

// ---------------------------------------------------------------- vector sources
// Trial primal point v = x - tau (c~ - K~^T y)  (Eq. 5 first line)
struct SrcPrimalTrial {
  const double *x, *c, *kty, *D;
  double tau;
  int64_t off;
  __device__ double v(int64_t i) const { return x[off + i] - tau * (c[off + i] - kty[off + i]); }
  __device__ double D_(int64_t i) const { return D[off + i]; }
};
// Average point zbar = sum eta z / sum eta (Alg. 1 line 7)
struct SrcAverage {
  const double *sum, *D;
  double W;
  int64_t off;
  __device__ double v(int64_t i) const { return sum[off + i] / W; }
  __device__ double D_(int64_t i) const { return D[off + i]; }
};
// Stored pre-projection values (dual trial: the SpMV epilogue leaves v in yh)
struct SrcStored {
  const double *v_, *D;
  int64_t off;
  __device__ double v(int64_t i) const { return v_[off + i]; }
  __device__ double D_(int64_t i) const { return D ? D[off + i] : 1.0; }
};
template <class S>
struct SrcAdapt {       // adapts .D_ to the .D expected by soc_team
  const S& s;
  __device__ double v(int64_t i) const { return s.v(i); }
  __device__ double D(int64_t i) const { return s.D_(i); }
};

// ---------------------------------------------------------------- destinations
// 0: trial primal (xh <- val, acc0 += (val - x)^2)
// 1: trial dual   (yh <- val, acc1 += (val - y)^2, acc2 += (val - y)(Kxh - Kx))
// 2: plain store  (out <- val)
// 3: KKT residual (acc += max |src - val|, max |val|) into kacc[base + 0/2] or [5]
struct DstTrialPrimal {
  double *xh; const double* x; int64_t off; Acc<kAcc>* acc;
  __device__ void put(int64_t i, double val) {
    const double xo = x[off + i];
    xh[off + i] = val;
    const double d = val - xo;
    acc->v[0] += d * d;
  }
};
struct DstTrialDual {
  double *yh; const double *y, *kxd; int64_t off; Acc<kAcc>* acc;
  __device__ void put(int64_t i, double val) {
    const int64_t j = off + i;
    yh[j] = val;
    const double d = val - y[j];
    acc->v[1] += d * d;
    acc->v[2] += d * kxd[j];
  }
};
struct DstStore {
  double* out; int64_t off;
  __device__ void put(int64_t i, double val) { out[off + i] = val; }
};
struct DstKktRows {       // distance of res to C_b (unit scaling), Eq. 9 err_p
  const double* res; int64_t off; double* mviol; double* mproj;
  __device__ void put(int64_t i, double val) {
    *mviol = fmax(*mviol, fabs(res[off + i] - val));
    *mproj = fmax(*mproj, fabs(val));
  }
};
struct DstKktCols {       // distance of lambda_2 to K_p^*, Eq. 9 err_d
  const double* lam; int64_t off; double* mviol;
  __device__ void put(int64_t i, double val) { *mviol = fmax(*mviol, fabs(lam[off + i] - val)); }
};

// Project one block with a team.  exp_dual: EXP means K_exp^* (and DEXP K_exp).
// HAS_EXP = false for the multi-thread teams (exp blocks are always in the
// thread class): the exp root finder is then not compiled into their kernels,
// whose register allocation would otherwise be set by it.
// exp_phase (thread class only): 0 whole projection; 1 the quick cases of an
// exp block only, false when it needs the root case (nothing written); 2 the
// root case only.  Non-exp blocks ignore it.
template <bool HAS_EXP, class Team, class Src, class Dst>
__device__ __forceinline__ bool project_block(Team& tm, const Block& b, bool exp_dual, bool unit,
                                              const Src& src, Dst& dst, int exp_phase = 0,
                                              double* warm = nullptr) {
  if (!HAS_EXP || b.kind == C_SOC || b.kind == C_RSOC) {
    SrcAdapt<Src> s{src};
    soc_team(tm, (int64_t)b.dim, b.kind == C_RSOC, unit, s, dst, nullptr, warm);
  } else {  // 3-d exponential blocks: one thread
    if (tm.rank() == 0) {
      const double r0 = src.v(0), s0 = src.v(1), t0 = src.v(2);
      const double dr = unit ? 1.0 : src.D_(0), ds = unit ? 1.0 : src.D_(1), dt = unit ? 1.0 : src.D_(2);
      double o0, o1, o2;
      const bool dual = (b.kind == C_EXP) == exp_dual;
      if (dual) {
        if (!proj_dexp_d(r0, s0, t0, dr, ds, dt, o0, o1, o2, exp_phase)) return false;
      } else if (exp_phase == 1) {
        if (!proj_exp_quick(r0, s0, t0, dr, ds, dt, o0, o1, o2)) return false;
      } else if (exp_phase == 2) {
        proj_exp_case4(r0, s0, t0, dr, ds, dt, o0, o1, o2);
      } else {
        proj_exp_d(r0, s0, t0, dr, ds, dt, o0, o1, o2);
      }
      dst.put(0, o0); dst.put(1, o1); dst.put(2, o2);
    }
  }
  return true;
}

// ---------------------------------------------------------------- block-cone kernels
// Operation codes for the block kernels.
enum BlockOp : int32_t {
  BOP_TRIAL_PRIMAL = 0,   // x^ = P_{diag(q_B) K_B}(x - tau(c - K^T y))
  BOP_TRIAL_DUAL = 1,     // y^ = P_{diag(r_b) C_b^*}(v) in place
  BOP_AVG_PRIMAL = 2,     // xa = P(xsum/W)
  BOP_AVG_DUAL = 3,       // ya = P(ysum/W)
  BOP_KKT_ROWS = 4,       // dist(res, C_b), unit scaling
  BOP_KKT_COLS = 5,       // dist(lam_2, K_p^*), unit scaling
  BOP_PROJECT = 6         // standalone: out = P_{D K}(v) (pdcs_proj_run; D == nullptr: unit)
};

struct BlockArgs {
  const Block* blocks;
  int64_t nblocks;
  int32_t op;
  int32_t cand;           // KKT candidate index (0/1)
  // vectors
  const double *x, *c, *kty, *D;  // primal trial source
  double* xh;
  const double* y;                // dual trial
  double* yh;
  const double* kxd;              // K x^ - K x of block rows
  const double* sum;              // average source
  double* out;                    // average destination
  const double* scratch;          // KKT residuals / lambdas
  double* part;                   // trial partials (kAcc) or KKT partials (kKAcc)
  int64_t slot0;
  double* warm;                   // trial ops: each block's last SOC/RSOC multiplier (soc_team)
};

// OP is the kernel's template constant (BlockOp), so each kernel holds one path.
template <bool HAS_EXP, int OP, class Team>
__device__ __forceinline__ bool run_block(Team& tm, const BlockArgs& A, const Ctl* ctl, const Block& b,
                                          Acc<kAcc>& acc, double* kv, int exp_phase = 0, int64_t bidx = 0) {
  bool done = true;
  switch (OP) {
    case BOP_TRIAL_PRIMAL: {
      SrcPrimalTrial s{A.x, A.c, A.kty, A.D, ctl->tau, b.off};
      DstTrialPrimal d{A.xh, A.x, b.off, &acc};
      done = project_block<HAS_EXP>(tm, b, false, false, s, d, exp_phase, A.warm ? A.warm + bidx : nullptr);
      break;
    }
    case BOP_TRIAL_DUAL: {
      SrcStored s{A.yh, A.D, b.off};
      DstTrialDual d{A.yh, A.y, A.kxd, b.off, &acc};
      done = project_block<HAS_EXP>(tm, b, true, false, s, d, exp_phase, A.warm ? A.warm + bidx : nullptr);
      break;
    }
    case BOP_AVG_PRIMAL:
    case BOP_AVG_DUAL: {
      SrcAverage s{A.sum, A.D, ctl->Wsum, b.off};
      DstStore d{A.out, b.off};
      done = project_block<HAS_EXP>(tm, b, OP == BOP_AVG_DUAL, false, s, d, exp_phase);
      break;
    }
    case BOP_KKT_ROWS: {
      SrcStored s{A.scratch, nullptr, b.off};
      DstKktRows d{A.scratch, b.off, kv + 0, kv + 2};
      done = project_block<HAS_EXP>(tm, b, false, true, s, d, exp_phase);
      break;
    }
    case BOP_KKT_COLS: {
      SrcStored s{A.scratch, nullptr, b.off};
      DstKktCols d{A.scratch, b.off, kv + 5};
      done = project_block<HAS_EXP>(tm, b, true, true, s, d, exp_phase);
      break;
    }
    case BOP_PROJECT: {
      SrcStored s{A.scratch, A.D, b.off};
      DstStore d{A.out, b.off};
      done = project_block<HAS_EXP>(tm, b, false, A.D == nullptr, s, d, exp_phase);
      break;
    }
  }
  return done;
}

template <int OP>
__device__ __forceinline__ bool block_op_active(const BlockArgs& A, const Ctl* ctl) {
  if (OP == BOP_TRIAL_PRIMAL || OP == BOP_TRIAL_DUAL) return ctl->status == 4;  // running
  return true;
}

template <int OP>
__device__ __forceinline__ void finish_block_partials(const BlockArgs& A, Acc<kAcc>& acc, double* kv) {
  if (OP == BOP_TRIAL_PRIMAL || OP == BOP_TRIAL_DUAL) {
    cta_write_partials<kAcc>(acc, A.part, A.slot0 + blockIdx.x);
  } else if (OP == BOP_KKT_ROWS || OP == BOP_KKT_COLS) {
    // max-reduce kv[0..9] over the CTA; write into candidate half of the slot
    __shared__ double red[10][kThreads / 32];
    for (int i = 0; i < 10; ++i) {
      double s = kv[i];
      for (int o = 16; o >= 1; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
      if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = s;
    }
    __syncthreads();
    if (threadIdx.x < kKAcc) {
      const int i = threadIdx.x;
      double s = 0.0;
      const int cbase = 10 * A.cand;
      if (i >= cbase && i < cbase + 10)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = fmax(s, red[i - cbase][w]);
      A.part[(A.slot0 + blockIdx.x) * kKAcc + i] = s;
    }
  }
}

// One block per thread (exp / dual exp / SOC of dim <= 32).  Two passes per
// CTA step: every thread projects its block, an exp block only through its
// quick cases (membership, the r0, s0 <= 0 face); the exp blocks that need the
// root finder are then packed in thread order into a shared list and
// projected by the first threads of the CTA.  Lanes that finished early no
// longer idle beside a root finder in the same warp (round 1: 5.6 of 32 lanes
// active per instruction on mixed cfg 5).  Work per thread is fixed by the
// data, so the accumulators are summed in a fixed order.
template <int OP>
__global__ void __launch_bounds__(kThreads) k_blocks_thread(BlockArgs A, const Ctl* ctl) {
  if (!block_op_active<OP>(A, ctl)) return;
  Acc<kAcc> acc; acc.zero();
  double kv[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  ThreadTeam tm;
  __shared__ int32_t s_list[kThreads];
  __shared__ int32_t s_wcnt[kThreads / 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < A.nblocks; base += stride) {
    const int64_t bi = base + threadIdx.x;
    bool defer = false;
    if (bi < A.nblocks) {
      const Block b = A.blocks[bi];
      defer = !run_block<true, OP>(tm, A, ctl, b, acc, kv, 1, bi);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, defer);
    if (lane == 0) s_wcnt[warp] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      off += w < warp ? s_wcnt[w] : 0;
      tot += s_wcnt[w];
    }
    if (defer) s_list[off + __popc(bal & ((1u << lane) - 1u))] = threadIdx.x;
    __syncthreads();
    for (int k = threadIdx.x; k < tot; k += blockDim.x) {
      const Block b = A.blocks[base + s_list[k]];
      run_block<true, OP>(tm, A, ctl, b, acc, kv, 2, base + s_list[k]);
    }
    __syncthreads();
  }
  finish_block_partials<OP>(A, acc, kv);
}

// One block per warp (SOC/RSOC of dim 33..512).
template <int OP>
__global__ void __launch_bounds__(kThreads) k_blocks_warp(BlockArgs A, const Ctl* ctl) {
  if (!block_op_active<OP>(A, ctl)) return;
  Acc<kAcc> acc; acc.zero();
  double kv[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  WarpTeam tm{(int)(threadIdx.x & 31)};
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t bi = wid; bi < A.nblocks; bi += nw) {
    const Block b = A.blocks[bi];
    run_block<false, OP>(tm, A, ctl, b, acc, kv, 0, bi);
  }
  finish_block_partials<OP>(A, acc, kv);
}

// One block per CTA (SOC/RSOC of dim 513..4096).
template <int OP>
__global__ void __launch_bounds__(kThreads) k_blocks_cta(BlockArgs A, const Ctl* ctl) {
  if (!block_op_active<OP>(A, ctl)) return;
  __shared__ double sm[2 * (kThreads / 32) + 2];
  Acc<kAcc> acc; acc.zero();
  double kv[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  CtaTeam tm{sm};
  for (int64_t bi = blockIdx.x; bi < A.nblocks; bi += gridDim.x) {
    const Block b = A.blocks[bi];
    run_block<false, OP>(tm, A, ctl, b, acc, kv, 0, bi);
  }
  finish_block_partials<OP>(A, acc, kv);
}

// One block per thread-block cluster of kClusterCtas CTAs (SOC/RSOC of dim
// 4097..131072): per-pass reductions through distributed shared memory.
template <int OP>
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kThreads)
    k_blocks_cluster(BlockArgs A, const Ctl* ctl) {
  if (!block_op_active<OP>(A, ctl)) return;
  __shared__ double sm[2 * (kThreads / 32) + 2];
  Acc<kAcc> acc; acc.zero();
  double kv[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  ClusterTeam tm{sm};
  const int64_t cid = blockIdx.x / kClusterCtas, ncl = gridDim.x / kClusterCtas;
  for (int64_t bi = cid; bi < A.nblocks; bi += ncl) {
    const Block b = A.blocks[bi];
    run_block<false, OP>(tm, A, ctl, b, acc, kv, 0, bi);
  }
  finish_block_partials<OP>(A, acc, kv);
}

// All CTAs on one block at a time (giant SOC/RSOC; cooperative launch).
constexpr size_t kGridSmem = 2 * kGridCache * kThreads * sizeof(double);   // 32 KB
template <int OP>
#ifndef PDCS_GRID_MINB
#define PDCS_GRID_MINB 1
#endif
__global__ void __launch_bounds__(kThreads, PDCS_GRID_MINB) k_blocks_grid(BlockArgs A, const Ctl* ctl, double* gbuf) {
  if (!block_op_active<OP>(A, ctl)) return;
  __shared__ double sm[2 * (kThreads / 32) + 2];
  Acc<kAcc> acc; acc.zero();
  double kv[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  extern __shared__ double gcache[];        // kGridSmem bytes (launch_blocks_op)
  GridTeam tm{sm, gbuf, 0, gcache};
  for (int64_t bi = 0; bi < A.nblocks; ++bi) {
    const Block b = A.blocks[bi];
    run_block<false, OP>(tm, A, ctl, b, acc, kv, 0, bi);
  }
  finish_block_partials<OP>(A, acc, kv);
}

// Host side: launch the kernel of size class c (thread, warp, CTA, cluster,
// grid) for block operation op; each (class, op) pair is its own kernel.
template <int OP>
inline cudaError_t launch_blocks_op(int c, int g, BlockArgs B, const Ctl* ctl, double* gbuf, cudaStream_t st) {
  switch (c) {
    case 0: k_blocks_thread<OP><<<g, kThreadsSmall, 0, st>>>(B, ctl); return cudaGetLastError();
    case 1: k_blocks_warp<OP><<<g, kThreads, 0, st>>>(B, ctl); return cudaGetLastError();
    case 2: k_blocks_cta<OP><<<g, kThreads, 0, st>>>(B, ctl); return cudaGetLastError();
    case 3: k_blocks_cluster<OP><<<g, kThreads, 0, st>>>(B, ctl); return cudaGetLastError();
    default: {
      void* args[] = {(void*)&B, (void*)&ctl, (void*)&gbuf};
      return cudaLaunchCooperativeKernel((void*)k_blocks_grid<OP>, dim3(g), dim3(kThreads), args, kGridSmem, st);
    }
  }
}
inline cudaError_t launch_blocks(int c, int g, const BlockArgs& B, const Ctl* ctl, double* gbuf, cudaStream_t st) {
  switch (B.op) {
    case BOP_TRIAL_PRIMAL: return launch_blocks_op<BOP_TRIAL_PRIMAL>(c, g, B, ctl, gbuf, st);
    case BOP_TRIAL_DUAL: return launch_blocks_op<BOP_TRIAL_DUAL>(c, g, B, ctl, gbuf, st);
    case BOP_AVG_PRIMAL: return launch_blocks_op<BOP_AVG_PRIMAL>(c, g, B, ctl, gbuf, st);
    case BOP_AVG_DUAL: return launch_blocks_op<BOP_AVG_DUAL>(c, g, B, ctl, gbuf, st);
    case BOP_KKT_ROWS: return launch_blocks_op<BOP_KKT_ROWS>(c, g, B, ctl, gbuf, st);
    case BOP_KKT_COLS: return launch_blocks_op<BOP_KKT_COLS>(c, g, B, ctl, gbuf, st);
    default: return launch_blocks_op<BOP_PROJECT>(c, g, B, ctl, gbuf, st);
  }
}
// Co-resident CTAs per SM of the grid-team kernel (cooperative launch bound),
// the minimum over its instantiations.
inline cudaError_t grid_team_occupancy(int* nb) {
  int m = 1 << 20, v = 0;
  cudaError_t e;
#define PDCS_OCC(OPV) \
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_blocks_grid<OPV>, kThreads, kGridSmem)) != cudaSuccess) return e; \
  m = v < m ? v : m;
  PDCS_OCC(BOP_TRIAL_PRIMAL) PDCS_OCC(BOP_TRIAL_DUAL) PDCS_OCC(BOP_AVG_PRIMAL) PDCS_OCC(BOP_AVG_DUAL)
  PDCS_OCC(BOP_KKT_ROWS) PDCS_OCC(BOP_KKT_COLS) PDCS_OCC(BOP_PROJECT)
#undef PDCS_OCC
  *nb = m;
  return cudaSuccess;
}

}  // namespace pdcs
