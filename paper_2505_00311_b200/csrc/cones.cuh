// cones.cuh — projections onto diagonally rescaled cones, device side.
//
//  * Rescaled SOC / RSOC (Theorem 1; proof 1185-1249).
//    The paper finds the multiplier lambda of Eq. 7 by bisection.
//    Here the same root is found with Newton on the reciprocal norm:
//        t > 0:  psi(lam) = 1/||p(lam)|| - (1-2 lam)/t,   p_i = dh_i x_i/(dh_i^2 + 2 lam)
//        t < 0:  psi(mu)  = 1/||p(mu)||  - (1-mu)/|t|,    p_i = dh_i x_i/(1 + mu dh_i^2),
//                lam = 1/(2 mu)   (reading A16)
//    1/||(H + s I)^-1 g|| is concave in s (the Moré-Sorensen secular function),
//    so psi is concave increasing and Newton from the left end converges
//    monotonically to the unique root, usually in 3-6 passes over the block.
//    Recovery y = (I + 2 lam Dh^-2)^-1 x, s = ||Dh^-1 y|| (A16).
//    Each pass is one team-wide reduction; the team is a thread, a warp, a CTA
//    or the whole grid (cooperative) depending on the block size (PAPER.md:713,
//    "thread-wise / block-wise / grid-wise").
//  * Rescaled exponential cone (Theorem 4), one thread per
//    cone.  Root of the pole-free determinant form of h(rho)
//    (reading A18) by safeguarded Newton inside the Eq. 16 bracket, recovery by
//    orthogonal coefficient, nearest of {root point, face point, t-raised point, 0}.
//  * Dual exponential cone by the Remark.
#pragma once
#include <cooperative_groups.h>
#include "internal.cuh"

namespace pdcs {

// ------------------------------------------------------------------ teams
struct ThreadTeam {
  __device__ int rank() const { return 0; }
  __device__ int size() const { return 1; }
  __device__ void sum2(double&, double&) {}
};

struct WarpTeam {
  int lane;
  __device__ int rank() const { return lane; }
  __device__ int size() const { return 32; }
  __device__ void sum2(double& a, double& b) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
  }
};

// CTA team: all threads of the block; sm holds 2 * (blockDim/32) doubles.
struct CtaTeam {
  double* sm;
  __device__ int rank() const { return threadIdx.x; }
  __device__ int size() const { return blockDim.x; }
  __device__ void sum2(double& a, double& b) {
    WarpTeam w{(int)(threadIdx.x & 31)};
    w.sum2(a, b);
    const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { sm[wid] = a; sm[nw + wid] = b; }
    __syncthreads();
    a = 0.0; b = 0.0;
    for (int i = 0; i < nw; ++i) { a += sm[i]; b += sm[nw + i]; }
  }
};

// Cluster team: the kClusterCtas CTAs of a thread-block cluster.  Each pass's
// CTA sums are exchanged through distributed shared memory and added in rank
// order, so every CTA gets the same bits.  sm holds 2 * (blockDim/32) + 2 doubles.
struct ClusterTeam {
  double* sm;
  __device__ int rank() const { return (int)cooperative_groups::this_cluster().block_rank() * blockDim.x + threadIdx.x; }
  __device__ int size() const { return (int)cooperative_groups::this_cluster().num_blocks() * blockDim.x; }
  __device__ void sum2(double& a, double& b) {
    CtaTeam c{sm};
    c.sum2(a, b);
    auto cl = cooperative_groups::this_cluster();
    const int slot = 2 * (blockDim.x >> 5);
    if (threadIdx.x == 0) { sm[slot] = a; sm[slot + 1] = b; }
    cl.sync();
    double sa = 0.0, sb = 0.0;
    for (unsigned int r = 0; r < cl.num_blocks(); ++r) {
      const double* p = cl.map_shared_rank(sm, r);
      sa += p[slot];
      sb += p[slot + 1];
    }
    cl.sync();                       // the slots may be rewritten by the next pass
    a = sa;
    b = sb;
  }
};

// Whole-grid team (cooperative launch).  gbuf holds 2 buffers x 2 x gridDim doubles.
constexpr int kGridCache = 8;   // elements per thread the grid team keeps in shared memory
struct GridTeam {
  double* sm;      // >= 2*(blockDim/32) + 2 doubles of shared memory
  double* gbuf;
  int parity;
  double* cache;   // 2 * kGridCache * blockDim doubles of dynamic shared memory (or nullptr)
  __device__ int rank() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ int size() const { return gridDim.x * blockDim.x; }
  __device__ void sum2(double& a, double& b) {
    CtaTeam c{sm};
    c.sum2(a, b);
    double* buf = gbuf + (size_t)parity * 2 * gridDim.x;
    parity ^= 1;
    if (threadIdx.x == 0) { buf[2 * blockIdx.x] = a; buf[2 * blockIdx.x + 1] = b; }
    cooperative_groups::this_grid().sync();
    // every CTA reduces the per-CTA partials in the same fixed order, all its
    // threads loading one (a, b) pair each (one 16-B load instead of a warp's
    // serial walk over ~20 pairs: one L2 latency per pass instead of ~20)
    double sa = 0.0, sb = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
      const double2 p = __ldcg(reinterpret_cast<const double2*>(buf) + i);
      sa += p.x;
      sb += p.y;
    }
    c.sum2(sa, sb);
    a = sa;
    b = sb;
  }
};

// ------------------------------------------------------------------ rescaled SOC / RSOC
// Src: double v(int64_t i) (pre-projection value of block element i, unrotated),
//      double D(int64_t i) (divisor of element i).
// Dst: void put(int64_t i, double val) (projected value of element i).
// Preconditions: d >= 2 (SOC) / >= 3 (RSOC); all team members call uniformly.
enum SocMode { SM_ZERO = 0, SM_IDENT = 1, SM_HALF = 2, SM_LAM = 3, SM_MU = 4 };

// Per-thread element cache of a team (only the grid team has one): the
// member's first kGridCache elements are staged once in shared memory and
// every later pass reads them from there instead of from L2 / HBM.
template <class Team> __device__ __forceinline__ double* team_cache(Team&) { return nullptr; }
__device__ __forceinline__ double* team_cache(GridTeam& t) { return t.cache; }

#ifndef PDCS_WARM_DELTA
#define PDCS_WARM_DELTA 0.1           // relative margin below the previous root (0.02: Lasso grid team +12%, 0.1 neutral; mixed +1.9%)
#endif
// warm (optional): this block's multiplier from its previous projection of the
// same kind (> 0: lambda-form root, < 0: mu-form root negated, 0: none).  The
// Newton iteration then starts below it (10% relative) instead of at 0,
// and falls back to 0 if that start is not below the new root; the root it
// converges to is the same one (the stopping rule does not depend on the start).
template <class Team, class Src, class Dst>
__device__ __forceinline__ void soc_team(Team& tm, int64_t d, bool rsoc, bool unit, const Src& src,
                                         Dst& dst, int* newton_iters = nullptr, double* warm = nullptr) {
  const double v0 = src.v(0), v1 = src.v(1);
  const double t = rsoc ? (v0 + v1) * kRsqrt2 : v0;
  const double x1 = rsoc ? (v0 - v1) * kRsqrt2 : v1;
  const double D0 = unit ? 1.0 : src.D(0);
  const int r = tm.rank(), S = tm.size();
  auto X = [&](int64_t i) { return i == 1 ? x1 : src.v(i); };
  auto H = [&](int64_t i) { return unit ? 1.0 : src.D(i) / D0; };   // dhat_i
  // elements of this member in order i = 1 + r, 1 + r + S, ...: the first KC
  // from the team's shared-memory cache (same values, same order: same bits)
  double* const cache = team_cache(tm);
  const int KC = cache ? kGridCache : 0, CT = blockDim.x, ct = threadIdx.x;
  if (cache) {
    int64_t i = 1 + r;
    for (int k = 0; k < KC && i < d; ++k, i += S) {
      cache[k * CT + ct] = X(i);
      cache[(KC + k) * CT + ct] = H(i);
    }
  }
  auto each = [&](auto&& f) {
    int64_t i = 1 + r;
    for (int k = 0; k < KC && i < d; ++k, i += S) f(i, cache[k * CT + ct], cache[(KC + k) * CT + ct]);
    for (; i < d; i += S) f(i, X(i), H(i));
  };
  // pass 1: ||dh x||^2 and ||x/dh||^2 (Thm 1 case tests)
  double a = 0.0, b = 0.0;
  each([&](int64_t, double x, double h) {
    const double p = h * x, q = x / h;
    a += p * p;
    b += q * q;
  });
  tm.sum2(a, b);
  const double n_times = sqrt(a), n_over = sqrt(b);
  int mode;
  if (t <= 0.0 && n_times <= -t) mode = SM_ZERO;        // case (i)
  else if (n_over <= t) mode = SM_IDENT;                 // case (ii)
  else if (t == 0.0) mode = SM_HALF;                     // case (iii)
  else mode = t > 0.0 ? SM_LAM : SM_MU;                  // case (iv)
  if (mode == SM_ZERO || mode == SM_IDENT) {
    for (int64_t i = 1 + r; i < d; i += S) {
      if (i == 1) {
        dst.put(0, mode == SM_ZERO ? 0.0 : v0);
        dst.put(1, mode == SM_ZERO ? 0.0 : v1);
      } else {
        dst.put(i, mode == SM_ZERO ? 0.0 : src.v(i));
      }
    }
    return;
  }
  double s_out, par = 0.0;
  if (unit) {
    // textbook SOC: ((t + ||x||)/2) (1, x/||x||); here n_times == n_over
    s_out = 0.5 * (t + n_times);
    each([&](int64_t i, double x, double) {
      const double y = s_out * x / n_times;
      if (i == 1) {
        if (rsoc) { dst.put(0, (s_out + y) * kRsqrt2); dst.put(1, (s_out - y) * kRsqrt2); }
        else { dst.put(0, s_out); dst.put(1, y); }
      } else {
        dst.put(i, y);
      }
    });
    return;
  }
  int its = 0;
  if (mode == SM_LAM || mode == SM_MU) {
    const double at = fabs(t);
    bool warm_try = false;
    if (warm) {
      const double w = *warm;
      const double wp = mode == SM_LAM ? w : -w;
      if (wp > 0.0 && wp < (mode == SM_LAM ? 0.5 : 1.0)) { par = wp * (1.0 - PDCS_WARM_DELTA); warm_try = true; }
    }
    for (; its < 64; ++its) {
      double S0 = 0.0, S1 = 0.0;
      each([&](int64_t, double x, double h) {
        const double h2 = h * h;
        double p, w;
        if (mode == SM_LAM) { const double rd = 1.0 / (h2 + 2.0 * par); p = h * x * rd; w = p * p * rd; }
        else { const double rd = 1.0 / (1.0 + par * h2); p = h * x * rd; w = p * p * h2 * rd; }
        S0 += p * p;
        S1 += w;
      });
      tm.sum2(S0, S1);
      const double nrm = sqrt(S0);
      double psi, dpsi;
      if (mode == SM_LAM) {
        psi = 1.0 / nrm - (1.0 - 2.0 * par) / at;
        dpsi = 2.0 * S1 / (S0 * nrm) + 2.0 / at;
      } else {
        psi = 1.0 / nrm - (1.0 - par) / at;
        dpsi = S1 / (S0 * nrm) + 1.0 / at;
      }
      if (!(psi < 0.0)) {                       // at (or past, by rounding) the root
        if (warm_try) { warm_try = false; par = 0.0; continue; }   // the warm start was above it
        break;
      }
      warm_try = false;
      const double step = -psi / dpsi;
      const double cap = mode == SM_LAM ? 0.5 : 1.0;
      double np = par + step;
      if (!(np < cap)) np = 0.5 * (par + cap);
      if (!(np > par)) break;
      const bool conv = step <= 4e-16 * np;
      par = np;
      if (conv) { ++its; break; }
    }
  }
  if (newton_iters) *newton_iters = its;
  if (warm && tm.rank() == 0) *warm = mode == SM_LAM ? par : mode == SM_MU ? -par : 0.0;
  // recovery: y_i, s = ||y/dh|| (reading A16)
  auto Y = [&](double x, double h) {
    const double h2 = h * h;
    if (mode == SM_HALF) return x / (1.0 + 1.0 / h2);
    if (mode == SM_LAM) return h2 * x / (h2 + 2.0 * par);
    return par * h2 * x / (1.0 + par * h2);
  };
  double ss = 0.0, dummy = 0.0;
  each([&](int64_t, double x, double h) {
    const double q = Y(x, h) / h;
    ss += q * q;
  });
  tm.sum2(ss, dummy);
  s_out = sqrt(ss);
  each([&](int64_t i, double x, double h) {
    const double y = Y(x, h);
    if (i == 1) {
      if (rsoc) { dst.put(0, (s_out + y) * kRsqrt2); dst.put(1, (s_out - y) * kRsqrt2); }
      else { dst.put(0, s_out); dst.put(1, y); }
    } else {
      dst.put(i, y);
    }
  });
}

// ------------------------------------------------------------------ exponential cone
// Membership with additive slack (Eq. 12-13; reading A20).
__device__ __forceinline__ bool d_in_exp(double r, double s, double t, double tol) {
  if (s > 0.0 && t >= s * exp(r / s) - tol) return true;
  return fabs(s) <= tol && r <= tol && t >= -tol;
}
__device__ __forceinline__ bool d_in_exp_dual(double r, double s, double t, double tol) {
  if (r < 0.0 && 2.718281828459045 * t >= -r * exp(s / r) - tol) return true;
  return fabs(r) <= tol && s >= -tol && t >= -tol;
}

// det[v0, u, w] e^{-|rho|}, its rho-derivative with the same scaling, and the
// magnitude of its terms.  u = (dr rho, ds, dt e^rho), w = (1/dr, (1-rho)/ds,
// -e^-rho/dt) span the Moreau pair of Eq. 17, <u, w> = 0.
struct ExpDet { double g, dg, mag; };
// Ratios of the divisors, computed once per cone (the same quotients as
// inline: bit-identical, 6 fp64 divisions fewer per determinant evaluation).
struct ExpRatios {
  double dr, ds, sd_t, dt_s, dt_r, dr_t, dr_s, ds_r;   // ds/dt, dt/ds, dt/dr, dr/dt, dr/ds, ds/dr
  __device__ ExpRatios(double dr_, double ds_, double dt_)
      : dr(dr_), ds(ds_), sd_t(ds_ / dt_), dt_s(dt_ / ds_), dt_r(dt_ / dr_), dr_t(dr_ / dt_), dr_s(dr_ / ds_),
        ds_r(ds_ / dr_) {}
};
__device__ __forceinline__ ExpDet exp_det(double r0, double s0, double t0, const ExpRatios& q, double rho) {
  const double e0 = exp(-fabs(rho));
  const double ep = rho >= 0.0 ? 1.0 : e0 * e0;     // e^{rho - |rho|}
  const double em = rho >= 0.0 ? e0 * e0 : 1.0;     // e^{-rho - |rho|}
  const double cr = -q.sd_t * em - q.dt_s * (1.0 - rho) * ep;
  const double cs = q.dt_r * ep + q.dr_t * rho * em;
  const double ct = (q.dr * rho * (1.0 - rho) / q.ds - q.ds_r) * e0;
  const double dcr = q.sd_t * em + q.dt_s * rho * ep;
  const double dcs = q.dt_r * ep + q.dr_t * (1.0 - rho) * em;
  const double dct = q.dr * (1.0 - 2.0 * rho) / q.ds * e0;
  ExpDet o;
  o.g = r0 * cr + s0 * cs + t0 * ct;
  o.dg = r0 * dcr + s0 * dcs + t0 * dct;
  o.mag = fabs(r0 * cr) + fabs(s0 * cs) + fabs(t0 * ct);
  return o;
}
__device__ __forceinline__ int det_sign(const ExpDet& e) {
  if (!(fabs(e.g) > 16.0 * 2.220446049250313e-16 * e.mag)) return 0;   // rounding noise
  return e.g < 0.0 ? -1 : 1;
}

// P_{D K_exp}(v0), Theorem 4 with reading A18.
// proj_exp_quick: cases 1-3 (membership tests and the r0, s0 <= 0 face);
// false when the root case 4 is needed (proj_exp_case4).  proj_exp_d is the
// two in sequence; the thread-class kernel runs them as two passes so that the
// lanes of a warp that need the root finder are packed together.
__device__ __forceinline__ bool proj_exp_quick(double r0, double s0, double t0, double dr, double ds, double dt,
                                               double& o0, double& o1, double& o2) {
  {  // case 1: D^-1 v0 in K_exp
    const double w0 = r0 / dr, w1 = s0 / ds, w2 = t0 / dt;
    const double tol = 1e-12 * sqrt(w0 * w0 + w1 * w1 + w2 * w2);
    if (d_in_exp(w0, w1, w2, tol)) { o0 = r0; o1 = s0; o2 = t0; return true; }
  }
  {  // case 2: -D v0 in K_exp^*
    const double w0 = -dr * r0, w1 = -ds * s0, w2 = -dt * t0;
    const double tol = 1e-12 * sqrt(w0 * w0 + w1 * w1 + w2 * w2);
    if (d_in_exp_dual(w0, w1, w2, tol)) { o0 = 0.0; o1 = 0.0; o2 = 0.0; return true; }
  }
  if (r0 <= 0.0 && s0 <= 0.0) { o0 = r0; o1 = 0.0; o2 = fmax(t0, 0.0); return true; }   // case 3
  return false;
}
__device__ __noinline__ void proj_exp_case4(double r0, double s0, double t0, double dr, double ds, double dt,
                                            double& o0, double& o1, double& o2) {
  const ExpRatios q(dr, ds, dt);
  // case 4: bracket (Eq. 16); an end whose det is rounding
  // noise is the root.
  double rho = __builtin_nan("");
  double lo = 0.0, hi = 0.0;
  int slo = 0, shi = 0;
  bool found = false;
  if (r0 > 0.0 && s0 > 0.0) {
    const double a3 = r0 * ds / (s0 * dr), a4 = 1.0 - s0 * ds / (r0 * dr);
    lo = fmin(a3, a4); hi = fmax(a3, a4);
    if (lo == hi) { rho = lo; found = true; }
    else {
      slo = det_sign(exp_det(r0, s0, t0, q, lo));
      shi = det_sign(exp_det(r0, s0, t0, q, hi));
      if (slo == 0) { rho = lo; found = true; } else if (shi == 0) { rho = hi; found = true; }
    }
  } else if (s0 > 0.0) {          // r0 <= 0 < s0: (-inf, a3)
    hi = r0 * ds / (s0 * dr);
    shi = det_sign(exp_det(r0, s0, t0, q, hi));
    if (shi == 0) { rho = hi; found = true; }
    else {
      for (int j = 0; j < 200; ++j) {      // doubling, cap 200 (A19)
        lo = hi - ldexp(1.0, j);
        slo = det_sign(exp_det(r0, s0, t0, q, lo));
        if (slo != shi) break;
      }
      if (slo == 0) { rho = lo; found = true; }
    }
  } else {                        // s0 <= 0 < r0: (a4, inf)
    lo = 1.0 - s0 * ds / (r0 * dr);
    slo = det_sign(exp_det(r0, s0, t0, q, lo));
    if (slo == 0) { rho = lo; found = true; }
    else {
      for (int j = 0; j < 200; ++j) {
        hi = lo + ldexp(1.0, j);
        shi = det_sign(exp_det(r0, s0, t0, q, hi));
        if (shi != slo) break;
      }
      if (shi == 0) { rho = hi; found = true; }
    }
  }
  bool have = found;
  if (!found && slo != shi) {
    // safeguarded Newton inside [lo, hi] (bisection when Newton leaves the
    // bracket or stalls)
    have = true;
    rho = 0.5 * (lo + hi);
    double dxold = hi - lo, dx = dxold;
    for (int it = 0; it < 200; ++it) {
      const ExpDet e = exp_det(r0, s0, t0, q, rho);
      const int s = det_sign(e);
      if (s == 0) break;
      if (s == slo) lo = rho; else hi = rho;
      const double nr = rho - e.g / e.dg;
      if (!(nr > lo && nr < hi) || fabs(2.0 * e.g) > fabs(dxold * e.dg)) {
        dxold = dx;
        dx = 0.5 * (hi - lo);
        rho = lo + dx;
      } else {
        dxold = dx;
        dx = rho - nr;
        rho = nr;
      }
      if (!(rho > lo && rho < hi)) { rho = 0.5 * (lo + hi); if (!(rho > lo && rho < hi)) break; }
      if (fabs(dx) <= 2.220446049250313e-16 * fabs(rho)) break;
    }
  }
  // candidates: root point, face (min(r0,0), 0, t0^+), t-raised point, 0
  // nearest by the sign of <p - q, p + q - 2 v0> (reading P7; the squared
  // distances themselves can tie to the ulp while the points differ)
  double b0 = 0.0, b1 = 0.0, b2 = 0.0;
  auto consider = [&](double a, double b, double c) {
    if (!isfinite(a) || !isfinite(b) || !isfinite(c)) return;
    const double diff = (a - b0) * (a + b0 - 2.0 * r0) + (b - b1) * (b + b1 - 2.0 * s0) +
                        (c - b2) * (c + b2 - 2.0 * t0);
    if (diff < 0.0) { b0 = a; b1 = b; b2 = c; }
  };
  if (have && isfinite(rho)) {
    const double sc = exp(-fmax(rho, 0.0));
    const double u0 = dr * rho * sc, u1 = ds * sc, u2 = dt * exp(rho - fmax(rho, 0.0));
    const double uu = u0 * u0 + u1 * u1 + u2 * u2;
    const double sp = (r0 * u0 + s0 * u1 + t0 * u2) / uu;
    if (sp > 0.0) consider(sp * u0, sp * u1, sp * u2);
  }
  consider(fmin(r0, 0.0), 0.0, fmax(t0, 0.0));
  if (s0 > 0.0) {
    const double w0 = r0 / dr, w1 = s0 / ds, w2 = t0 / dt;
    consider(r0, s0, dt * fmax(w2, w1 * exp(w0 / w1)));
  }
  o0 = b0; o1 = b1; o2 = b2;
}

__device__ __noinline__ void proj_exp_d(double r0, double s0, double t0, double dr, double ds,
                                        double dt, double& o0, double& o1, double& o2) {
  if (proj_exp_quick(r0, s0, t0, dr, ds, dt, o0, o1, o2)) return;
  proj_exp_case4(r0, s0, t0, dr, ds, dt, o0, o1, o2);
}

// P_{D K_exp^*}(v) = v + P_{D^-1 K_exp}(-v)  (Remark)
// phase 0: whole; 1: quick cases only (false: case 4 needed); 2: case 4 only.
__device__ __forceinline__ bool proj_dexp_d(double r0, double s0, double t0, double dr, double ds,
                                            double dt, double& o0, double& o1, double& o2, int phase = 0) {
  double p0, p1, p2;
  if (phase == 1) {
    if (!proj_exp_quick(-r0, -s0, -t0, 1.0 / dr, 1.0 / ds, 1.0 / dt, p0, p1, p2)) return false;
  } else if (phase == 2) {
    proj_exp_case4(-r0, -s0, -t0, 1.0 / dr, 1.0 / ds, 1.0 / dt, p0, p1, p2);
  } else {
    proj_exp_d(-r0, -s0, -t0, 1.0 / dr, 1.0 / ds, 1.0 / dt, p0, p1, p2);
  }
  o0 = r0 + p0; o1 = s0 + p1; o2 = t0 + p2;
  return true;
}

}  // namespace pdcs
