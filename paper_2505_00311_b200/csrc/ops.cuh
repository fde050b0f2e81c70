// ops.cuh — elementwise / control kernels of Alg. 1 and the SpMV epilogues.
#pragma once
#include "kernels.cuh"

namespace pdcs {

constexpr double kInf = __builtin_huge_val();
enum { ST_OPTIMAL = 0, ST_ITER = 1, ST_TIME = 2, ST_NUMERICAL = 3, ST_RUNNING = 4 };

// ---------------------------------------------------------------- primal update (elementwise part)
// x^_j = P_{[l~,u~]}(x_j - tau (c~_j - (K~^T y)_j)) for box / zero / nonneg
// coordinates (Eq. 5); block coordinates are left to the block
// kernels.  Accumulates ||x^ - x||^2 for the line search.
__global__ void __launch_bounds__(kThreads) k_primal_elem(int64_t n, const uint8_t* __restrict__ ek,
                                                          const double* __restrict__ x,
                                                          const double* __restrict__ c,
                                                          const double* __restrict__ kty,
                                                          const double* __restrict__ lt,
                                                          const double* __restrict__ ut,
                                                          double* __restrict__ xh,
                                                          const Ctl* ctl, double* part, int64_t slot0) {
  if (ctl->status != ST_RUNNING) return;
  const double tau = ctl->tau;
  Acc<kAcc> acc; acc.zero();
  // 4 grid strides per step, every load of the 4 issued before the first use:
  // each thread visits the same coordinates in the same order as a plain
  // grid-stride loop (same accumulation order, same bits), with 4x the bytes
  // in flight (Fisher: 1e7 box coordinates per trial)
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < n; j0 += 4 * T) {
    uint8_t k[4];
    double xj[4], cj[4], kj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = j0 + u * T < n ? ek[j0 + u * T] : (uint8_t)EK_BLOCK;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + u * T;
      xj[u] = cj[u] = kj[u] = 0.0;
      if (k[u] != EK_BLOCK) { xj[u] = x[j]; cj[u] = c[j]; kj[u] = kty[j]; }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (k[u] == EK_BLOCK) continue;
      const int64_t j = j0 + u * T;
      const double v = xj[u] - tau * (cj[u] - kj[u]);
      const double p = box_proj(k[u], v, lt, ut, j);
      xh[j] = p;
      const double d = p - xj[u];
      acc.v[0] += d * d;
    }
  }
  cta_write_partials<kAcc>(acc, part, slot0 + blockIdx.x);
}

// Average candidate, elementwise part: out = P(sum / W) (Alg. 1 line 7 + reading A10).
__global__ void __launch_bounds__(kThreads) k_avg_elem(int64_t n, const uint8_t* __restrict__ ek,
                                                       const double* __restrict__ sum,
                                                       const double* __restrict__ lt,
                                                       const double* __restrict__ ut,
                                                       double* __restrict__ out, const Ctl* ctl) {
  const double W = ctl->Wsum;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t k = ek[j];
    if (k == EK_BLOCK) continue;
    out[j] = box_proj(k, sum[j] / W, lt, ut, j);
  }
}

// ---------------------------------------------------------------- line search / reflection
// AdaptiveStepPDHG accept test (reading A7) and
// AdaptiveReflectionParameter (reading A9), Halpern coefficients
// (PAPER.md:606).  One CTA; partial sums reduced in a fixed order.
// In graph mode (h_retry != 0) the decision also drives the graph's WHILE node
// (repeat the trial while rejected) and IF node (run the Eq. 9 check).
__device__ __forceinline__ void set_graph_flags(unsigned long long h_retry, unsigned long long h_check,
                                                unsigned int retry, unsigned int check) {
  if (h_retry) {
    cudaGraphSetConditional((cudaGraphConditionalHandle)h_retry, retry);
    cudaGraphSetConditional((cudaGraphConditionalHandle)h_check, check);
  }
}

// Sum of the trial partial slots in a fixed order by one CTA of kDecideThreads:
// each thread keeps 4 independent chains (slots t, t+T, t+2T, t+3T, then
// +4T ...) so 12 loads are in flight per thread instead of 3 (the serial
// chain had made k_decide ~11 us, latency-bound: profiles/r1_launches_*).
constexpr int kDecideThreads = 1024;
__device__ __forceinline__ void block_sum3(const double* __restrict__ part, int64_t nslots, double out[3]) {
  double s[4][3] = {};
  const int64_t T = blockDim.x;
  int64_t i = threadIdx.x;
  for (; i + 3 * T < nslots; i += 4 * T) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < 3; ++c) s[u][c] += part[(i + u * T) * kAcc + c];
  }
  for (; i < nslots; i += T)
#pragma unroll
    for (int c = 0; c < 3; ++c) s[0][c] += part[i * kAcc + c];
  __shared__ double red[3][kDecideThreads];
#pragma unroll
  for (int c = 0; c < 3; ++c) red[c][threadIdx.x] = (s[0][c] + s[1][c]) + (s[2][c] + s[3][c]);
  __syncthreads();
  for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) {
#pragma unroll
      for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + w];
    }
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] = red[c][0];
}

// Reduce the trial partial slots into ctl->red3 (row-sharded runs all-reduce
// red3[1..2] between this kernel and k_decide).
__global__ void __launch_bounds__(kDecideThreads) k_reduce_trial(const double* __restrict__ part, int64_t nslots,
                                                                 Ctl* ctl) {
  if (ctl->status != ST_RUNNING) return;
  double r[3];
  block_sum3(part, nslots, r);
  if (threadIdx.x == 0) { ctl->red3[0] = r[0]; ctl->red3[1] = r[1]; ctl->red3[2] = r[2]; }
}

// Thread 0 of k_decide: accept test, beta window, Halpern coefficients, flags.
__device__ __forceinline__ void decide_serial(Ctl& C, const double red[3], int prereduced,
                                           unsigned long long h_retry, unsigned long long h_check) {
  const double dxx = prereduced ? C.red3[0] : red[0];
  const double dyy = prereduced ? C.red3[1] : red[1];
  const double cross = prereduced ? C.red3[2] : red[2];
  C.last_dxx = dxx; C.last_dyy = dyy; C.last_cross = cross;
  const double num = C.omega * dxx + dyy / C.omega;
  C.last_num = num;
  C.trials++;
  bool acc;
  if (C.vanilla) {
    acc = true;
    C.eta_used = C.eta;
  } else {
    const double den = fabs(cross);
    const double etabar = den > 0.0 ? num / (2.0 * den) : kInf;
    if (C.eta <= etabar) {
      acc = true;
      C.eta_used = C.eta;
      C.eta = fmin(C.ls_grow * C.eta, etabar);
    } else {
      acc = false;
      C.eta *= C.ls_shrink;
      C.rejects++;
      if (C.eta < 1e-12 * C.eta_init || C.rejects > C.ls_max_rejects) C.status = ST_NUMERICAL;
    }
  }
  C.accepted = acc ? 1 : 0;
  C.need_check = 0;
  C.store_kty = 0;
  if (acc) {
    C.rejects = 0;
    if (C.vanilla) {
      C.ha = 1.0; C.hb = 0.0; C.hbeta = 0.0;
    } else {
      const double res = sqrt(num);
      const int64_t W = C.refl_window;
      if (C.k % W == 0) C.r_start = res;
      if (C.k % W == W - 1 && res > C.r_start) C.beta *= 0.5;
      C.ha = (double)(C.k + 1) / (double)(C.k + 2);
      C.hb = 1.0 / (double)(C.k + 2);
      C.hbeta = C.beta;
      C.Wsum += C.eta_used;
    }
    C.k++;
    C.total++;
    if (C.k % C.check_interval == 0) { C.need_check = 1; C.store_kty = 1; }
  }
  C.tau = C.eta / C.omega;
  C.sigma = C.eta * C.omega;
  set_graph_flags(h_retry, h_check, (!acc && C.status == ST_RUNNING) ? 1u : 0u, C.need_check ? 1u : 0u);
}

// Small duals (m <= kFuseYMax, single GPU): the accepted step's y-side
// Halpern/average update (k_halpern_y) runs in this kernel after the
// decision, saving a graph node per iteration where node latency dominates
// (PAPER.md:918).  Same formula, same bits.
constexpr int64_t kFuseYMax = 2048;
struct FusedY {
  int64_t m;
  const double* yh; const double* y0; double* y; double* ysum;
  const double* kxh; const double* kx0; double* kxc;     // K x carried with the same step
};

// y-side reflected Halpern step and average sum of one row (Alg. 1 line 5-6,
// PAPER.md:606): y+ = a((1+beta) y^ - beta y) + c y0, ysum += eta y+.  Explicit
// roundings so k_decide's fused update and k_halpern_y (scalar or vectorised)
// produce the same bits whatever contraction the compiler would pick.
__device__ __forceinline__ double halpern_y_row(double a, double b, double c, double eta, double yh,
                                                double y, double y0, double& ysum) {
  const double t = __fma_rn(1.0 + b, yh, __dmul_rn(-b, y));
  const double yn = __fma_rn(a, t, __dmul_rn(c, y0));
  ysum = __fma_rn(eta, yn, ysum);
  return yn;
}

// The same step on the carried product K x (linearity of Alg. 1 line 6):
// K x+ = a((1+beta) K x^ - beta K x) + c K x0, explicit roundings (one
// function for k_decide's fused update and k_halpern_y).
__device__ __forceinline__ double halpern_kx_row(double a, double b, double c, double kxh, double kx, double kx0) {
  const double t = __fma_rn(1.0 + b, kxh, __dmul_rn(-b, kx));
  return __fma_rn(a, t, __dmul_rn(c, kx0));
}

__global__ void __launch_bounds__(kDecideThreads) k_decide(const double* __restrict__ part, int64_t nslots,
                                                           Ctl* ctl, unsigned long long h_retry,
                                                           unsigned long long h_check, int prereduced,
                                                           FusedY fy) {
  if (ctl->status != ST_RUNNING) {
    if (threadIdx.x == 0) set_graph_flags(h_retry, h_check, 0u, 0u);
    return;
  }
  if (prereduced) nslots = 0;
  // The decision is a serial chain of reads and writes of the control block;
  // done on a shared-memory copy (loaded while the partials are summed, stored
  // back by all threads) instead of ~10 dependent global round trips by one
  // thread (k_decide was ~10 us in the launch list, the reduction ~1.5 of it).
  static_assert(sizeof(Ctl) % sizeof(double) == 0, "Ctl is copied as doubles");
  constexpr int kCtlWords = sizeof(Ctl) / sizeof(double);
  __shared__ Ctl sC;
  for (int i = threadIdx.x; i < kCtlWords; i += blockDim.x)
    reinterpret_cast<double*>(&sC)[i] = reinterpret_cast<const double*>(ctl)[i];
  double red[3];
  block_sum3(part, nslots, red);               // ends with __syncthreads: sC is visible
  if (threadIdx.x == 0) decide_serial(sC, red, prereduced, h_retry, h_check);
  __syncthreads();
  if (fy.m > 0 && sC.status == ST_RUNNING && sC.accepted) {
    const double a = sC.ha, b = sC.hbeta, c = sC.hb, eta = sC.eta_used;
    for (int64_t i = threadIdx.x; i < fy.m; i += blockDim.x) {
      fy.y[i] = halpern_y_row(a, b, c, eta, fy.yh[i], fy.y[i], fy.y0[i], fy.ysum[i]);
      fy.kxc[i] = halpern_kx_row(a, b, c, fy.kxh[i], fy.kxc[i], fy.kx0[i]);
    }
  }
  for (int i = threadIdx.x; i < kCtlWords; i += blockDim.x)
    reinterpret_cast<double*>(ctl)[i] = reinterpret_cast<const double*>(&sC)[i];
}

// ---------------------------------------------------------------- SpMV epilogues
// One sweep over K computes K x^ (fresh); K x of the current iterate is carried
// by linearity (K x+ = a((1+beta) K x^ - beta K x) + c K x0 on
// an accepted step, the candidate's fresh product at a restart):
// Kxh = K x^; v = y + sigma (h~ - 2 K x^ + K x); y^ = P(v) for free / nonneg
// rows, v stored for block rows (projected by the block kernels).
// Accumulates ||y^ - y||^2 and <y^ - y, K x^ - K x> (line search).
struct EpiDualTrial {
  static constexpr int NA = kAcc;
  static constexpr int NX = 1;   // gathers x^ only; K x is carried (kxc, k_halpern_y)
  const double *y, *h;
  const uint8_t* rk;
  double *kxh, *kxd, *yh;
  const double* kxc;             // K x of the current iterate
  double sigma;
  int run;
  __device__ void init(const Ctl* c) { sigma = c->sigma; run = c->status == ST_RUNNING; }
  __device__ bool active() const { return run; }
  __device__ void row(int64_t i, double kxhat, double, Acc<NA>& a) {
    // read-only inputs through the non-coherent path: the compiler may then
    // issue them ahead of this and earlier rows' stores (kxh, yh, kxd)
    const double kx = __ldg(kxc + i), yi = __ldg(y + i), hi = __ldg(h + i);
    const uint8_t k = __ldg(rk + i);
    kxh[i] = kxhat;
    const double v = yi + sigma * (hi - 2.0 * kxhat + kx);
    if (k == EK_BLOCK) { yh[i] = v; kxd[i] = kxhat - kx; return; }
    const double p = k == EK_NONNEG ? fmax(v, 0.0) : v;
    yh[i] = p;
    const double d = p - yi;
    a.v[1] += d * d;
    a.v[2] += d * (kxhat - kx);
  }
};

// K^T y+ on an accepted step (y+ already formed by k_halpern_y), fused with
// ReflectedHalpern on x and the step-weighted average
// (reading A8):  x+ = a((1+b) x^ - b x) + c x0, xsum += eta x+,
// and the fresh product K^T y+ for the next primal step.
struct EpiHalpernX {
  static constexpr int NA = 1;
  static constexpr int NX = 1;
  const double *xh, *x0;
  double *x, *kty, *xsum;
  double a, b, c, eta;
  int run;
  __device__ void init(const Ctl* C) {
    run = C->status == ST_RUNNING && C->accepted;
    a = C->ha; c = C->hb; b = C->hbeta; eta = C->eta_used;
  }
  __device__ bool active() const { return run; }
  __device__ void row(int64_t j, double dot, double, Acc<NA>&) {
    // x and xsum are read and then written by this thread only, xh and x0 are
    // read-only here: all four through the read-only path, so the compiler may
    // issue them ahead of earlier rows' stores (short K^T rows: Fisher's 1e7)
    const double xhj = __ldg(xh + j), xj = __ldg(x + j), x0j = __ldg(x0 + j), xsj = __ldg(xsum + j);
    const double xn = a * ((1.0 + b) * xhj - b * xj) + c * x0j;
    x[j] = xn;
    kty[j] = dot;
    xsum[j] = xsj + eta * xn;
  }
};

// x-side ReflectedHalpern + average after the all-reduce of K^T y+ (row-sharded
// path; the single-GPU path fuses this into the K^T sweep as EpiHalpernX).
__global__ void __launch_bounds__(kThreads) k_halpern_x(int64_t n, const double* __restrict__ xh,
                                                        const double* __restrict__ x0,
                                                        const double* __restrict__ ktyp,
                                                        double* __restrict__ x, double* __restrict__ kty,
                                                        double* __restrict__ xsum, const Ctl* ctl) {
  if (ctl->status != ST_RUNNING || !ctl->accepted) return;
  const double a = ctl->ha, b = ctl->hbeta, c = ctl->hb, eta = ctl->eta_used;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double xn = a * ((1.0 + b) * xh[j] - b * x[j]) + c * x0[j];
    x[j] = xn;
    kty[j] = ktyp[j];
    xsum[j] += eta * xn;
  }
}

// Plain product store.
struct EpiStore {
  static constexpr int NA = 1;
  static constexpr int NX = 1;
  double* out;
  __device__ void init(const Ctl*) {}
  __device__ bool active() const { return true; }
  __device__ void row(int64_t i, double dot, double, Acc<NA>&) { out[i] = dot; }
};

// Product store only on an accepted step (row-sharded K^T y+ partial).
struct EpiStoreAcc {
  static constexpr int NA = 1;
  static constexpr int NX = 1;
  double* out;
  int run;
  __device__ void init(const Ctl* C) { run = C->status == ST_RUNNING && C->accepted; }
  __device__ bool active() const { return run; }
  __device__ void row(int64_t i, double dot, double, Acc<NA>&) { out[i] = dot; }
};

// Product store of the first component of an interleaved-pair gather (autotune).
struct EpiStore2 {
  static constexpr int NA = 1;
  static constexpr int NX = 3;
  double* out;
  __device__ void init(const Ctl*) {}
  __device__ bool active() const { return true; }
  __device__ void row(int64_t i, double dot, double, Acc<NA>&) { out[i] = dot; }
};

// y-side ReflectedHalpern + average: y+, ysum.
__global__ void __launch_bounds__(kThreads) k_halpern_y(int64_t m, const double* __restrict__ yh,
                                                        const double* __restrict__ y0,
                                                        double* __restrict__ y,
                                                        double* __restrict__ ysum,
                                                        const double* __restrict__ kxh,
                                                        const double* __restrict__ kx0,
                                                        double* __restrict__ kxc, const Ctl* ctl) {
  if (ctl->status != ST_RUNNING || !ctl->accepted) return;
  const double a = ctl->ha, b = ctl->hbeta, c = ctl->hb, eta = ctl->eta_used;
  auto upd = [&](double yhi, double yi, double y0i, double& ysi) {
    return halpern_y_row(a, b, c, eta, yhi, yi, y0i, ysi);
  };
  // 16-byte loads, two pairs (4 rows) per thread and step: 8 loads in flight
  // per thread instead of 4 scalar ones.  The same arithmetic per row, so the
  // result is bit-identical to the scalar loop and to k_decide's fused update (the buffers are cudaMalloc'd,
  // 256-B aligned; the odd tail row is done by the first thread).
  const int64_t np = m >> 1, T = (int64_t)gridDim.x * blockDim.x;
  const double2* yh2 = reinterpret_cast<const double2*>(yh);
  const double2* y02 = reinterpret_cast<const double2*>(y0);
  double2* y2 = reinterpret_cast<double2*>(y);
  double2* ys2 = reinterpret_cast<double2*>(ysum);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += 2 * T) {
    const int64_t j = i + T;
    const bool two = j < np;
    const double2 h0 = yh2[i], v0 = y2[i], o0 = y02[i];
    double2 s0 = ys2[i];
    double2 h1{}, v1{}, o1{}, s1{};
    if (two) { h1 = yh2[j]; v1 = y2[j]; o1 = y02[j]; s1 = ys2[j]; }
    double2 n0;
    n0.x = upd(h0.x, v0.x, o0.x, s0.x);
    n0.y = upd(h0.y, v0.y, o0.y, s0.y);
    y2[i] = n0; ys2[i] = s0;
    if (two) {
      double2 n1;
      n1.x = upd(h1.x, v1.x, o1.x, s1.x);
      n1.y = upd(h1.y, v1.y, o1.y, s1.y);
      y2[j] = n1; ys2[j] = s1;
    }
  }
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t i = m - 1;
    y[i] = upd(yh[i], y[i], y0[i], ysum[i]);
  }
  // the carried K x (same coefficients)
  const double2* kh2 = reinterpret_cast<const double2*>(kxh);
  const double2* k02 = reinterpret_cast<const double2*>(kx0);
  double2* kc2 = reinterpret_cast<double2*>(kxc);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += T) {
    const double2 h = kh2[i], v = kc2[i], o = k02[i];
    kc2[i] = make_double2(halpern_kx_row(a, b, c, h.x, v.x, o.x), halpern_kx_row(a, b, c, h.y, v.y, o.y));
  }
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t i = m - 1;
    kxc[i] = halpern_kx_row(a, b, c, kxh[i], kxc[i], kx0[i]);
  }
}

// ---------------------------------------------------------------- Eq. 9 residuals
// Per candidate c the 10 reduction values are:
//   0 max|res - P_C(res)| 1 max|Gx| 2 max|P_C(res)| 3 sum y h 4 sum (y - y0)^2
//   5 max|lam - P(lam)|   6 max|G^T y| 7 sum c x  8 sum box dual terms 9 sum (x - x0)^2
__device__ __forceinline__ bool kkt_is_max(int i) {
  const int r = i % 10;
  return r == 0 || r == 1 || r == 2 || r == 5 || r == 6;
}

__device__ __forceinline__ void write_kkt_partials(double* kv, double* part, int64_t slot) {
  __shared__ double red[kKAcc][kThreads / 32];
  for (int i = 0; i < kKAcc; ++i) {
    double s = kv[i];
    const bool mx = kkt_is_max(i);
    for (int o = 16; o >= 1; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, s, o);
      s = mx ? fmax(s, t) : s + t;
    }
    if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (threadIdx.x < kKAcc) {
    const bool mx = kkt_is_max(threadIdx.x);
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = mx ? fmax(s, red[threadIdx.x][w]) : s + red[threadIdx.x][w];
    part[slot * kKAcc + threadIdx.x] = s;
  }
}

struct KktCand {
  const double *x, *y, *kx, *kty;   // scaled iterate and its products
  double *res, *lam;                // scratch for block rows / block columns
};

// Rows: err_p terms (Gx = r (K~ x~), res = Gx - h, C_b with unit scaling) and
// the y^T h part of the dual objective.
__global__ void __launch_bounds__(kThreads) k_kkt_rows(int64_t m, const uint8_t* __restrict__ rk,
                                                       const double* __restrict__ r,
                                                       const double* __restrict__ h,
                                                       const double* __restrict__ y0, KktCand c0,
                                                       KktCand c1, int ncand, double* part,
                                                       int64_t slot0) {
  double kv[kKAcc];
  for (int i = 0; i < kKAcc; ++i) kv[i] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t k = rk[i];
    const double ri = r[i], hi = h[i];
    for (int c = 0; c < ncand; ++c) {
      const KktCand& C = c ? c1 : c0;
      double* v = kv + 10 * c;
      const double gx = ri * C.kx[i];
      const double res = gx - hi;
      v[1] = fmax(v[1], fabs(gx));
      if (k == EK_BLOCK) C.res[i] = res;
      else {
        const double p = k == EK_NONNEG ? fmax(res, 0.0) : 0.0;
        v[0] = fmax(v[0], fabs(res - p));
        v[2] = fmax(v[2], fabs(p));
      }
      const double yi = C.y[i];
      v[3] += (yi / ri) * hi;
      const double dy = yi - y0[i];
      v[4] += dy * dy;
    }
  }
  write_kkt_partials(kv, part, slot0 + blockIdx.x);
}

// Columns: err_d terms (lambda = c - G^T y, G^T y = q (K~^T y~); Lambda of Eq. 3
// for box coordinates, K_p^* for cone coordinates), c^T x and the box part of the
// dual objective with lambda~_1 = P_Lambda(lambda_1) (reading A13).
__global__ void __launch_bounds__(kThreads) k_kkt_cols(int64_t n, const uint8_t* __restrict__ ek,
                                                       const double* __restrict__ q,
                                                       const double* __restrict__ c,
                                                       const double* __restrict__ l,
                                                       const double* __restrict__ u,
                                                       const double* __restrict__ x0, KktCand c0,
                                                       KktCand c1, int ncand, double* part,
                                                       int64_t slot0) {
  double kv[kKAcc];
  for (int i = 0; i < kKAcc; ++i) kv[i] = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t k = ek[j];
    const double qj = q[j], cj = c[j];
    for (int cc = 0; cc < ncand; ++cc) {
      const KktCand& C = cc ? c1 : c0;
      double* v = kv + 10 * cc;
      const double gty = qj * C.kty[j];
      const double lam = cj - gty;
      v[6] = fmax(v[6], fabs(gty));
      const double xj = C.x[j];
      v[7] += cj * (xj / qj);
      const double dx = xj - x0[j];
      v[9] += dx * dx;
      double p;
      switch (k) {
        case EK_FREE: p = 0.0; break;
        case EK_LO0: case EK_LO: p = fmax(lam, 0.0); break;
        case EK_UP: p = fmin(lam, 0.0); break;
        case EK_BOTH: p = lam; break;
        case EK_ZERO: p = lam; break;            // dual of {0} is R^d
        case EK_NONNEG: p = fmax(lam, 0.0); break;
        default: C.lam[j] = lam; p = lam; break; // block: handled by the block kernel
      }
      v[5] = fmax(v[5], fabs(lam - p));
      if (k == EK_LO || k == EK_BOTH) v[8] += l[j] * fmax(p, 0.0);
      if (k == EK_UP || k == EK_BOTH) v[8] -= u[j] * fmax(-p, 0.0);
    }
  }
  write_kkt_partials(kv, part, slot0 + blockIdx.x);
}

// Reduce the KKT partial slots into ctl->kred (row-sharded runs all-reduce the
// row-side entries 10c+0..2 (max) and 10c+3..4 (sum) before k_kkt_decide).
__global__ void __launch_bounds__(kThreads) k_kkt_reduce(const double* __restrict__ part, int64_t nslots,
                                                         Ctl* ctl) {
  __shared__ double red[kKAcc][kThreads];
  double acc[kKAcc];
  for (int i = 0; i < kKAcc; ++i) acc[i] = 0.0;
  for (int64_t s = threadIdx.x; s < nslots; s += blockDim.x)
    for (int i = 0; i < kKAcc; ++i) {
      const double v = part[s * kKAcc + i];
      acc[i] = kkt_is_max(i) ? fmax(acc[i], v) : acc[i] + v;
    }
  for (int i = 0; i < kKAcc; ++i) red[i][threadIdx.x] = acc[i];
  __syncthreads();
  for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int i = 0; i < kKAcc; ++i)
        red[i][threadIdx.x] = kkt_is_max(i) ? fmax(red[i][threadIdx.x], red[i][threadIdx.x + w])
                                            : red[i][threadIdx.x] + red[i][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < kKAcc) ctl->kred[threadIdx.x] = red[threadIdx.x][0];
}

// Form Eq. 9 for each candidate and run GetRestartCandidate / restart
// condition / PrimalWeightUpdate / termination (
// SPEC.md:387-413; readings A10-A15).  mode 0: evaluate only; 1: full check.
__global__ void k_kkt_decide(int ncand, int mode, double hnorm, double cnorm, Ctl* ctl) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* red = ctl->kred;
  Ctl& C = *ctl;
  if (mode == 1) C.checks++;
  double e[2] = {kInf, kInf};
  for (int c = 0; c < ncand; ++c) {
    auto R = [&](int i) { return red[10 * c + i]; };
    const double err_p = R(0) / (1.0 + fmax(hnorm, fmax(R(1), R(2))));
    const double err_d = R(5) / (1.0 + fmax(cnorm, R(6)));
    const double pobj = R(7), dobj = R(3) + R(8);
    const double gap = fabs(pobj - dobj) / (1.0 + fmax(fabs(pobj), fabs(dobj)));
    C.kkt[c][0] = err_p; C.kkt[c][1] = err_d; C.kkt[c][2] = gap; C.kkt[c][3] = pobj; C.kkt[c][4] = dobj;
    C.dist[c][0] = sqrt(R(9));
    C.dist[c][1] = sqrt(R(4));
    e[c] = fmax(err_p, fmax(err_d, gap));
  }
  C.restart = 0;
  C.best_flag = 0;
  if (mode == 0) return;
  const int use_avg = (ncand == 2 && e[1] <= e[0]) ? 1 : 0;   // tie -> average
  C.use_avg = use_avg;
  const double ec = e[use_avg];
  if (ec < C.best_e) {
    C.best_e = ec;
    C.best_flag = 1;
    for (int i = 0; i < 5; ++i) C.best_kkt[i] = C.kkt[use_avg][i];
  }
  if (ec <= C.tol) {
    C.done = 1;
    if (C.stop_at_tol) C.status = ST_OPTIMAL;   // graph mode: later launches become no-ops
  }
  if (C.vanilla) return;
  const bool rs = ec <= C.suff * C.e_anchor ||
                  (C.e_prev >= 0.0 && ec <= C.nec * C.e_anchor && ec > C.e_prev) ||
                  (double)C.k >= C.art * (double)C.total;
  C.e_prev = ec;
  if (rs) {
    const double dxn = C.dist[use_avg][0], dyn = C.dist[use_avg][1];
    if (dxn > 1e-10 && dyn > 1e-10) C.omega = exp(0.5 * log(dyn / dxn) + 0.5 * log(C.omega));
    C.e_anchor = ec;
    C.k = 0;
    C.Wsum = 0.0;
    C.beta = C.beta_max;
    C.e_prev = -1.0;
    C.restarts++;
    C.restart = 1;
    C.tau = C.eta / C.omega;
    C.sigma = C.eta * C.omega;
  }
}

// Restart / best / candidate copies selected by the finalize decision.
struct RestartArgs {
  int64_t n, m;
  const double *cx[2], *cy[2], *ckty[2], *ckx[2];
  double *x, *x0, *y, *y0, *kty, *xsum, *ysum, *kxc, *kx0;
  double *bx, *by, *candx, *candy;
};
__global__ void __launch_bounds__(kThreads) k_restart_copy(RestartArgs A, const Ctl* ctl) {
  const int u = ctl->use_avg;
  const bool rs = ctl->restart, bf = ctl->best_flag;
  const int64_t N = A.n > A.m ? A.n : A.m;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    if (j < A.n) {
      const double xv = A.cx[u][j];
      A.candx[j] = xv;
      if (bf) A.bx[j] = xv;
      if (rs) {
        A.x[j] = xv; A.x0[j] = xv; A.kty[j] = A.ckty[u][j]; A.xsum[j] = 0.0;
      }
    }
    if (j < A.m) {
      const double yv = A.cy[u][j];
      A.candy[j] = yv;
      if (bf) A.by[j] = yv;
      if (rs) {
        A.y[j] = yv; A.y0[j] = yv; A.ysum[j] = 0.0;
        const double kv = A.ckx[u][j];          // the candidate's fresh product K x
        A.kxc[j] = kv; A.kx0[j] = kv;
      }
    }
  }
}

// ---------------------------------------------------------------- Ruiz / Pock-Chambolle
// For every row i of a CSR (of K or of K^T): out_i = max_p |v_p|/(s_i t_col)
// (mode 0) or sum_p (mode 1).  One warp per row.  Rows of K^T are columns of
// K, so the same kernel serves both sides.
__global__ void __launch_bounds__(kThreads) k_row_norms(int64_t rows, const int32_t* __restrict__ ptr,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ srow,
                                                        const double* __restrict__ scol, int mode,
                                                        double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < rows;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double si = srow[i];
    double a = 0.0;
    for (int32_t p = ptr[i] + lane; p < ptr[i + 1]; p += 32) {
      const double t = fabs(val[p]) / (si * scol[col[p]]);
      a = mode ? a + t : fmax(a, t);
    }
    for (int o = 16; o >= 1; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, a, o);
      a = mode ? a + t : fmax(a, t);
    }
    if (lane == 0) out[i] = a;
  }
}
// s_i *= sqrt(norm_i) (1 where the norm is 0)
__global__ void k_apply_root(int64_t n, const double* __restrict__ nrm, double* __restrict__ s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s[i] *= nrm[i] > 0.0 ? sqrt(nrm[i]) : 1.0;
}
// RSOC leading pair: geometric mean of the first two divisors
__global__ void k_rsoc_geomean(const int64_t* __restrict__ offs, int64_t nb, double* __restrict__ s) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = offs[b];
    const double g = sqrt(s[a] * s[a + 1]);
    s[a] = g; s[a + 1] = g;
  }
}
// K~ values: v_p = G_p / (s_row * s_col)
__global__ void __launch_bounds__(kThreads) k_scale_vals(int64_t rows, const int32_t* __restrict__ ptr,
                                                         const int32_t* __restrict__ col,
                                                         double* __restrict__ val,
                                                         const double* __restrict__ srow,
                                                         const double* __restrict__ scol) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < rows;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double si = srow[i];
    for (int32_t p = ptr[i] + lane; p < ptr[i + 1]; p += 32) val[p] = val[p] / (si * scol[col[p]]);
  }
}
// out_i = a_i * op b_i : 0 divide, 1 multiply
__global__ void k_ewise(int64_t n, const double* __restrict__ a, const double* __restrict__ b, int op,
                        double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = op == 0 ? a[i] / b[i] : a[i] * b[i];
}
__global__ void k_fill(int64_t n, double v, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}
// Deterministic single-CTA reductions: mode 0 max|a|, 1 sum a^2, 2 max a
__global__ void __launch_bounds__(kThreads) k_reduce(int64_t n, const double* __restrict__ a, int mode,
                                                     double* __restrict__ out) {
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = a[i];
    s = mode == 0 ? fmax(s, fabs(v)) : mode == 1 ? s + v * v : fmax(s, v);
  }
  __shared__ double red[kThreads];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
    if ((int)threadIdx.x < w) {
      const double t = red[threadIdx.x + w];
      red[threadIdx.x] = mode == 1 ? red[threadIdx.x] + t : fmax(red[threadIdx.x], t);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}
// scaled bounds: lt = q l, ut = q u (reading A2)
__global__ void k_bounds(int64_t n1, const double* __restrict__ q, const double* __restrict__ l,
                         const double* __restrict__ u, double* __restrict__ lt, double* __restrict__ ut) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n1; j += (int64_t)gridDim.x * blockDim.x) {
    lt[j] = q[j] * l[j];
    ut[j] = q[j] * u[j];
  }
}
// CSR transpose helpers
__global__ void k_row_ids(int64_t rows, const int32_t* __restrict__ ptr, int32_t* __restrict__ rid) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    for (int32_t p = ptr[i]; p < ptr[i + 1]; ++p) rid[p] = (int32_t)i;
}
__global__ void k_gather_t(int64_t nnz, const int32_t* __restrict__ perm, const int32_t* __restrict__ rid,
                           const double* __restrict__ val, int32_t* __restrict__ tcol,
                           double* __restrict__ tval) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = perm[p];
    tcol[p] = rid[s];
    tval[p] = val[s];
  }
}
__global__ void k_gather_vals(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ src,
                              double* __restrict__ dst) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    dst[p] = perm[p] >= 0 ? src[perm[p]] : 0.0;   // -1: quad padding
}
__global__ void k_iota(int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}
__global__ void k_count_cols(int64_t nnz, const int32_t* __restrict__ col, int32_t* __restrict__ cnt) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[p], 1);
}

}  // namespace pdcs
