// ============================================================================
//  PDCS CPU ORACLE  —  TEST INFRASTRUCTURE ONLY
// ----------------------------------------------------------------------------
//  A plain, slow, single-threaded C++ transcription of the PDCS method of
//  arxiv 2505.00311 used to check the CUDA path.  Only tests/,
//  __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
//  may load it.  It shares NO code, header, table or constant generator with
//  paper_2505_00311_b200/ (the product); both implement the same paper.
//
//  Precision: fp64 throughout (the paper states none; BASELINE.json: fp64).
//
//  Map of this file (each function cites the passage it follows):
//    spmv / spmv_t ............ PAPER.md:577-578 (Eq. 5 products)
//    proj_box ................. PAPER.md:577 (P_[l,u])
//    proj_soc_unit ............ PAPER.md:590 (textbook SOC)
//    proj_soc_scaled .......... PAPER.md:651-661 (Thm 1), proof 1185-1249;
//                               readings A16 (mu-form, s = ||y/dhat||), A17
//    proj_rsoc_scaled ......... PAPER.md:591 + SPEC.md:242-243 (rotation)
//    proj_exp_scaled .......... PAPER.md:1272-1311 (Thm 4), 1262-1268 (Lemma 2);
//                               reading A18 (pole-free determinant root)
//    proj_dual_exp_scaled ..... PAPER.md:1318-1327 (Remark)
//    in_exp / in_exp_dual ..... PAPER.md:1254-1259 (Eq. 12-13); reading A20
//    ruiz_scale ............... PAPER.md:646-648 (§3)
//    Solver::inner_step ....... PAPER.md:603-607 (Alg. 1 lines 4-7)
//    Solver::check ............ PAPER.md:602, 608, 611 (Alg. 1 lines 3, 8, 11),
//                               SPEC.md:387-413, 433-440
//    kkt ...................... PAPER.md:819-827 (Eq. 9)
//
//  "parity unpinned" items: the multi-step iterate sequence of
//  Alg. 1 (no closed form exists beyond the per-step pins in tests/).
// ============================================================================
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <vector>
#include <limits>
#include <chrono>
#include <algorithm>

namespace orc {

using std::vector;
static const double INF = std::numeric_limits<double>::infinity();

enum { K_ZERO = 0, K_NONNEG = 1, K_SOC = 2, K_RSOC = 3, K_EXP = 4, K_DUAL_EXP = 5 };

// ---------------------------------------------------------------- linear algebra
struct Csr {
  int64_t m = 0, n = 0;
  vector<int64_t> ptr;
  vector<int32_t> col;
  vector<double> val;
};

// y = A x, row-major entry order.
static void spmv(const Csr& A, const double* x, double* y) {
  for (int64_t i = 0; i < A.m; ++i) {
    double s = 0.0;
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) s += A.val[p] * x[A.col[p]];
    y[i] = s;
  }
}

// Transpose as a CSR of A^T (column layout).
static Csr transpose(const Csr& A) {
  Csr T;
  T.m = A.n; T.n = A.m;
  T.ptr.assign(A.n + 1, 0);
  for (int64_t p = 0; p < A.ptr[A.m]; ++p) T.ptr[A.col[p] + 1]++;
  for (int64_t j = 0; j < A.n; ++j) T.ptr[j + 1] += T.ptr[j];
  T.col.resize(A.ptr[A.m]);
  T.val.resize(A.ptr[A.m]);
  vector<int64_t> fill(T.ptr.begin(), T.ptr.end() - 1);
  for (int64_t i = 0; i < A.m; ++i)
    for (int64_t p = A.ptr[i]; p < A.ptr[i + 1]; ++p) {
      int64_t q = fill[A.col[p]]++;
      T.col[q] = (int32_t)i;
      T.val[q] = A.val[p];
    }
  return T;
}

static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double nrm2(const double* a, int64_t n) { return std::sqrt(dot(a, a, n)); }
static double nrminf(const double* a, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s = std::max(s, std::fabs(a[i]));
  return s;
}

// ---------------------------------------------------------------- projections
static int64_t g_rootfail = 0;   // root-finder failures (reported, never absorbed)

// Box: clamp.
static inline double proj_box(double v, double l, double u) { return std::min(std::max(v, l), u); }

// Unit SOC, textbook 3-case formula.  v = (t, x).
static void proj_soc_unit(int64_t d, const double* v, double* out) {
  double t = v[0];
  double nx = nrm2(v + 1, d - 1);
  if (nx <= t) { for (int64_t i = 0; i < d; ++i) out[i] = v[i]; return; }
  if (nx <= -t) { for (int64_t i = 0; i < d; ++i) out[i] = 0.0; return; }
  double a = 0.5 * (t + nx);
  out[0] = a;
  for (int64_t i = 1; i < d; ++i) out[i] = a * v[i] / nx;
}

// Projection onto D K_soc (Theorem 1).  v = (t, x), Dg =
// (d_1, ..., d_{n+1}) the diagonal of D; dhat_i = d_{i+1}/d_1.
// Cases in the theorem's order:
//  (i)  t <= 0 and ||dhat x|| <= -t           -> 0
//  (ii) ||x / dhat|| <= t                     -> (t, x)
//  (iii) t == 0, x != 0  -> (||x/(dhat+1/dhat)||, x/(1+dhat^-2))
//  (iv) root of Eq. 7.  Reading A16: for t > 0 bisect
//       phi+(lam) = (1-2lam)||dhat x/(dhat^2+2lam)|| - t on (0, 1/2);
//       for t < 0 bisect phi-(mu) = ||(1-mu) dhat x/(1+mu dhat^2)|| - |t| on
//       (0, 1) with lam = 1/(2mu) (Eq. 7 times (1-2lam)^2, square-rooted).
//       y = (I + 2 lam Dhat^-2)^-1 x; s = ||Dhat^-1 y|| (A16).
static void proj_soc_scaled(int64_t d, const double* v, const double* Dg, double* out) {
  const double t = v[0];
  const double* x = v + 1;
  const int64_t nx = d - 1;
  vector<double> dh(nx);
  for (int64_t i = 0; i < nx; ++i) dh[i] = Dg[i + 1] / Dg[0];
  double s_times = 0.0, s_over = 0.0;
  for (int64_t i = 0; i < nx; ++i) {
    s_times += (dh[i] * x[i]) * (dh[i] * x[i]);
    s_over += (x[i] / dh[i]) * (x[i] / dh[i]);
  }
  double n_times = std::sqrt(s_times), n_over = std::sqrt(s_over);
  if (t <= 0.0 && n_times <= -t) {                       // case (i)
    for (int64_t i = 0; i < d; ++i) out[i] = 0.0;
    return;
  }
  if (n_over <= t) {                                      // case (ii)
    for (int64_t i = 0; i < d; ++i) out[i] = v[i];
    return;
  }
  vector<double> y(nx);
  if (t == 0.0) {                                         // case (iii)
    for (int64_t i = 0; i < nx; ++i) y[i] = x[i] / (1.0 + 1.0 / (dh[i] * dh[i]));
  } else if (t > 0.0) {                                   // case (iv), t > 0
    auto phi = [&](double lam) {
      double s = 0.0;
      for (int64_t i = 0; i < nx; ++i) {
        double q = dh[i] * x[i] / (dh[i] * dh[i] + 2.0 * lam);
        s += q * q;
      }
      return (1.0 - 2.0 * lam) * std::sqrt(s) - t;
    };
    double lo = 0.0, hi = 0.5;                            // phi(lo) > 0 > phi(hi)
    for (int it = 0; it < 200; ++it) {
      double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      double f = phi(mid);
      if (f > 0.0) lo = mid; else if (f < 0.0) hi = mid; else { lo = hi = mid; break; }
    }
    double lam = 0.5 * (lo + hi);
    for (int64_t i = 0; i < nx; ++i) {
      double d2 = dh[i] * dh[i];
      y[i] = d2 * x[i] / (d2 + 2.0 * lam);
    }
  } else {                                                // case (iv), t < 0
    const double at = -t;
    auto phi = [&](double mu) {
      double s = 0.0;
      for (int64_t i = 0; i < nx; ++i) {
        double q = (1.0 - mu) * dh[i] * x[i] / (1.0 + mu * dh[i] * dh[i]);
        s += q * q;
      }
      return std::sqrt(s) - at;
    };
    double lo = 0.0, hi = 1.0;
    for (int it = 0; it < 200; ++it) {
      double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      double f = phi(mid);
      if (f > 0.0) lo = mid; else if (f < 0.0) hi = mid; else { lo = hi = mid; break; }
    }
    double mu = 0.5 * (lo + hi);
    for (int64_t i = 0; i < nx; ++i) {
      double d2 = dh[i] * dh[i];
      y[i] = mu * d2 * x[i] / (1.0 + mu * d2);
    }
  }
  double s = 0.0;
  for (int64_t i = 0; i < nx; ++i) s += (y[i] / dh[i]) * (y[i] / dh[i]);
  out[0] = std::sqrt(s);
  for (int64_t i = 0; i < nx; ++i) out[i + 1] = y[i];
}

// Rotated SOC {(a,b,z): a,b >= 0, ||z||^2 <= 2ab} through the
// orthogonal map (a,b) -> ((a+b)/sqrt2, (a-b)/sqrt2).
// The rescaled form requires Dg[0] == Dg[1] (reading A21).
static void proj_rsoc_scaled(int64_t d, const double* v, const double* Dg, double* out) {
  vector<double> w(v, v + d), o(d);
  w[0] = (v[0] + v[1]) * M_SQRT1_2;
  w[1] = (v[0] - v[1]) * M_SQRT1_2;
  if (Dg) proj_soc_scaled(d, w.data(), Dg, o.data());
  else proj_soc_unit(d, w.data(), o.data());
  for (int64_t i = 2; i < d; ++i) out[i] = o[i];
  out[0] = (o[0] + o[1]) * M_SQRT1_2;
  out[1] = (o[0] - o[1]) * M_SQRT1_2;
}

// Membership with additive slack (Eq. 12-13; reading A20).
static bool in_exp(double r, double s, double t, double tol) {
  if (s > 0.0 && t >= s * std::exp(r / s) - tol) return true;
  return std::fabs(s) <= tol && r <= tol && t >= -tol;
}
static bool in_exp_dual(double r, double s, double t, double tol) {
  if (r < 0.0 && M_E * t >= -r * std::exp(s / r) - tol) return true;
  return std::fabs(r) <= tol && s >= -tol && t >= -tol;
}

// det[v0, u(rho), w(rho)] * exp(-|rho|) with u = (dr rho, ds, dt e^rho) and
// w = (1/dr, (1-rho)/ds, -e^-rho/dt): the two directions of Eq. 17
// (PAPER.md:1308), <u, w> = 0.  v0 in span{u, w} <=> det = 0 <=> the t-equation
// h(rho) = 0 of Eq. 14 holds (reading A18: pole-free form of h).  *mag gets
// the sum of the absolute terms, so |det| <= 16 eps mag is rounding noise.
static double exp_det(double r0, double s0, double t0, double dr, double ds, double dt,
                      double rho, double* mag = nullptr) {
  double a = std::fabs(rho);
  double ep = std::exp(rho - a), em = std::exp(-rho - a), e0 = std::exp(-a);
  double cr = -(ds / dt) * em - (dt / ds) * (1.0 - rho) * ep;
  double cs = (dt / dr) * ep + (dr / dt) * rho * em;
  double ct = (dr * rho * (1.0 - rho) / ds - ds / dr) * e0;
  if (mag) *mag = std::fabs(r0 * cr) + std::fabs(s0 * cs) + std::fabs(t0 * ct);
  return r0 * cr + s0 * cs + t0 * ct;
}

// Sign of det at rho: -1, +1, or 0 when |det| is below rounding noise.
static int exp_det_sign(double r0, double s0, double t0, double dr, double ds, double dt,
                        double rho) {
  double mag;
  double g = exp_det(r0, s0, t0, dr, ds, dt, rho, &mag);
  if (!(std::fabs(g) > 16.0 * std::numeric_limits<double>::epsilon() * mag)) return 0;
  return g < 0.0 ? -1 : 1;
}

// Projection onto D K_exp (Theorem 4).
static void proj_exp_scaled(const double* v0, const double* D, double* out) {
  const double r0 = v0[0], s0 = v0[1], t0 = v0[2];
  const double dr = D[0], ds = D[1], dt = D[2];
  // case 1: v0 in D K_exp  <=>  D^-1 v0 in K_exp
  {
    double w0 = r0 / dr, w1 = s0 / ds, w2 = t0 / dt;
    double tol = 1e-12 * std::sqrt(w0 * w0 + w1 * w1 + w2 * w2);
    if (in_exp(w0, w1, w2, tol)) { out[0] = r0; out[1] = s0; out[2] = t0; return; }
  }
  // case 2: v0 in -D^-1 K_exp^*  <=>  -D v0 in K_exp^*
  {
    double w0 = -dr * r0, w1 = -ds * s0, w2 = -dt * t0;
    double tol = 1e-12 * std::sqrt(w0 * w0 + w1 * w1 + w2 * w2);
    if (in_exp_dual(w0, w1, w2, tol)) { out[0] = out[1] = out[2] = 0.0; return; }
  }
  // case 3: r0 <= 0, s0 <= 0  ->  (r0, 0, t0^+)
  if (r0 <= 0.0 && s0 <= 0.0) { out[0] = r0; out[1] = 0.0; out[2] = std::max(t0, 0.0); return; }
  // case 4: root of det on the bracket of Eq. 16.  An end
  // whose det is rounding noise is taken as the root (rho* is not separable
  // from it in floating point).
  auto sg = [&](double rho) { return exp_det_sign(r0, s0, t0, dr, ds, dt, rho); };
  double rho = NAN;
  double lo = 0.0, hi = 0.0;
  int slo = 0, shi = 0;
  if (r0 > 0.0 && s0 > 0.0) {
    double a3 = r0 * ds / (s0 * dr), a4 = 1.0 - s0 * ds / (r0 * dr);
    lo = std::min(a3, a4); hi = std::max(a3, a4);
    if (lo == hi) rho = lo;
    else {
      slo = sg(lo); shi = sg(hi);
      if (slo == 0) rho = lo; else if (shi == 0) rho = hi;
    }
  } else if (s0 > 0.0) {            // r0 <= 0 < s0: (-inf, a3), expand lo
    hi = r0 * ds / (s0 * dr);
    shi = sg(hi);
    if (shi == 0) rho = hi;
    else {
      for (int j = 0; j < 200; ++j) {   // doubling, cap 200 (reading A19)
        lo = hi - std::ldexp(1.0, j);
        slo = sg(lo);
        if (slo != shi) break;
      }
      if (slo == 0) rho = lo;
    }
  } else {                          // s0 <= 0 < r0: (a4, inf), expand hi
    lo = 1.0 - s0 * ds / (r0 * dr);
    slo = sg(lo);
    if (slo == 0) rho = lo;
    else {
      for (int j = 0; j < 200; ++j) {
        hi = lo + std::ldexp(1.0, j);
        shi = sg(hi);
        if (shi != slo) break;
      }
      if (shi == 0) rho = hi;
    }
  }
  bool have_root = true;
  if (std::isnan(rho)) {
    if (slo == shi) have_root = false;
    else {
      for (int it = 0; it < 400; ++it) {     // bisection to adjacent doubles
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        int sm = sg(mid);
        if (sm == 0) { lo = hi = mid; break; }
        if (sm == slo) lo = mid; else hi = mid;
      }
      rho = 0.5 * (lo + hi);
    }
  }
  // candidates (reading A18): root point, face point, t-raised point, 0.
  // "Nearest" is decided by the sign of ||p - v0||^2 - ||q - v0||^2 =
  // <p - q, p + q - 2 v0> (reading P7): the two squared distances can differ
  // by less than one ulp of their common part (a far-away t0) while the
  // points differ in r, s at 1e-6 relative.
  double best[3] = {0.0, 0.0, 0.0};              // candidate 0
  auto consider = [&](double a, double b, double c) {
    if (!std::isfinite(a) || !std::isfinite(b) || !std::isfinite(c)) return;
    double diff = (a - best[0]) * (a + best[0] - 2.0 * r0) + (b - best[1]) * (b + best[1] - 2.0 * s0) +
                  (c - best[2]) * (c + best[2] - 2.0 * t0);
    if (diff < 0.0) { best[0] = a; best[1] = b; best[2] = c; }
  };
  if (have_root && std::isfinite(rho)) {
    // v_p = (<v0,u>/||u||^2) u (orthogonal coefficient), u scaled by e^-max(rho,0)
    double sc = std::exp(-std::max(rho, 0.0));
    double u0 = dr * rho * sc, u1 = ds * sc, u2 = dt * std::exp(rho - std::max(rho, 0.0));
    double uu = u0 * u0 + u1 * u1 + u2 * u2;
    double sp = (r0 * u0 + s0 * u1 + t0 * u2) / uu;
    if (sp > 0.0) consider(sp * u0, sp * u1, sp * u2);
  } else {
    ++g_rootfail;
  }
  // face {s = 0, r <= 0, t >= 0} of K_exp (invariant under D)
  consider(std::min(r0, 0.0), 0.0, std::max(t0, 0.0));
  // t raised to the boundary in D^-1 coordinates (needs s > 0)
  if (s0 > 0.0) {
    double w0 = r0 / dr, w1 = s0 / ds, w2 = t0 / dt;
    double tb = std::max(w2, w1 * std::exp(w0 / w1));
    consider(r0, s0, dt * tb);
  }
  out[0] = best[0]; out[1] = best[1]; out[2] = best[2];
}

// Projection onto D K_exp^* = v0 + P_{D^-1 K_exp}(-v0) (Remark).
static void proj_dual_exp_scaled(const double* v0, const double* D, double* out) {
  double nv[3] = {-v0[0], -v0[1], -v0[2]};
  double Di[3] = {1.0 / D[0], 1.0 / D[1], 1.0 / D[2]};
  double p[3];
  proj_exp_scaled(nv, Di, p);
  out[0] = v0[0] + p[0]; out[1] = v0[1] + p[1]; out[2] = v0[2] + p[2];
}

static const double ONE3[3] = {1.0, 1.0, 1.0};

// ---------------------------------------------------------------- Alg. 1 scalar rules
// Line-search bound: eta_bar = (w||dx||^2 + ||dy||^2/w) / (2|<dy, K dx>|).
static double ls_bound(double num, double cross) {
  double den = std::fabs(cross);
  return den > 0.0 ? num / (2.0 * den) : INF;
}
// ReflectedHalpern coefficients: z+ = a((1+beta) zh - beta z) + b z0.
static void halpern_coef(int64_t k, double* a, double* b) {
  *a = (double)(k + 1) / (double)(k + 2);
  *b = 1.0 / (double)(k + 2);
}
// Restart condition (reading A11).
// e_prev < 0 means "no previous check in this epoch".
static bool restart_rule(double e, double e_anchor, double e_prev, int64_t k, int64_t total,
                         double suff, double nec, double art) {
  return e <= suff * e_anchor || (e_prev >= 0.0 && e <= nec * e_anchor && e > e_prev) ||
         (double)k >= art * (double)total;
}
// AdaptiveReflectionParameter (Alg. 1 line 5, reading A9):
// non-overlapping windows of W inner iterations within the epoch; res is the
// fixed-point residual ||z^ - z||_omega of inner iteration k.  The residual of the
// window's first iteration is remembered; at the window's last iteration beta is
// halved when the residual there exceeds the remembered one.
static double reflection_beta(int64_t k, int64_t W, double res, double* r_start, double beta) {
  if (k % W == 0) *r_start = res;
  if (k % W == W - 1 && res > *r_start) beta *= 0.5;
  return beta;
}
// GetRestartCandidate (Alg. 1 line 8, reading A14):
// the candidate with the smaller aggregate Eq. 9 error; a tie goes to the average.
static bool candidate_is_average(double e_current, double e_average) {
  return e_average <= e_current;
}
// PrimalWeightUpdate (theta = 1/2; reading A12).
static double primal_weight(double dxn, double dyn, double omega) {
  if (dxn > 1e-10 && dyn > 1e-10) return std::exp(0.5 * std::log(dyn / dxn) + 0.5 * std::log(omega));
  return omega;
}

// ---------------------------------------------------------------- problem
struct Cone { int32_t kind; int64_t dim; int64_t off; };

struct Params {            // layout mirrors the product's pdcs_params (independent copy)
  double tol; int64_t max_iters; double time_limit_s;
  int32_t ruiz_iters; int32_t pock_chambolle; int32_t check_interval; int32_t vanilla_pdhg;
  double eta0; double omega0; double beta_max; int32_t refl_window; int32_t pad0;
  double restart_suff, restart_nec, restart_art;
  double ls_shrink, ls_grow; int32_t ls_max_rejects; int32_t verbose;
};
struct Kkt { double err_p, err_d, err_gap, pobj, dobj; };
struct Result {
  int32_t status; int32_t pad; Kkt kkt;
  int64_t iters, trials, restarts, spmv_K, spmv_KT;
  double eta, omega, beta, solve_seconds;
};
enum { ST_OPTIMAL = 0, ST_ITER_LIMIT = 1, ST_TIME_LIMIT = 2, ST_NUMERICAL = 3, ST_RUNNING = 4 };

struct Problem {
  int64_t m, n, n1;
  Csr G, GT;
  vector<double> c, h, l, u;
  vector<Cone> pc, rc;
};

// Ruiz (10 rounds) + Pock-Chambolle (alpha = 1) rescaling (
// SPEC.md:274, 305-308; reading A2: r, q are divisors, K~ = diag(1/r) G diag(1/q)).
// The working matrix of every round is formed afresh as |G_ij|/(r_i q_j).
static void ruiz_scale(const Problem& P, int ruiz_iters, int pc, vector<double>& r,
                       vector<double>& q) {
  r.assign(P.m, 1.0);
  q.assign(P.n, 1.0);
  vector<double> rm(P.m), cm(P.n);
  for (int it = 0; it < ruiz_iters; ++it) {
    std::fill(rm.begin(), rm.end(), 0.0);
    std::fill(cm.begin(), cm.end(), 0.0);
    for (int64_t i = 0; i < P.m; ++i)
      for (int64_t p = P.G.ptr[i]; p < P.G.ptr[i + 1]; ++p) {
        int64_t j = P.G.col[p];
        double a = std::fabs(P.G.val[p]) / (r[i] * q[j]);
        rm[i] = std::max(rm[i], a);
        cm[j] = std::max(cm[j], a);
      }
    for (int64_t i = 0; i < P.m; ++i) r[i] *= rm[i] > 0.0 ? std::sqrt(rm[i]) : 1.0;
    for (int64_t j = 0; j < P.n; ++j) q[j] *= cm[j] > 0.0 ? std::sqrt(cm[j]) : 1.0;
  }
  if (pc) {
    std::fill(rm.begin(), rm.end(), 0.0);
    std::fill(cm.begin(), cm.end(), 0.0);
    for (int64_t i = 0; i < P.m; ++i)
      for (int64_t p = P.G.ptr[i]; p < P.G.ptr[i + 1]; ++p) {
        int64_t j = P.G.col[p];
        double a = std::fabs(P.G.val[p]) / (r[i] * q[j]);
        rm[i] += a;
        cm[j] += a;
      }
    for (int64_t i = 0; i < P.m; ++i) r[i] *= rm[i] > 0.0 ? std::sqrt(rm[i]) : 1.0;
    for (int64_t j = 0; j < P.n; ++j) q[j] *= cm[j] > 0.0 ? std::sqrt(cm[j]) : 1.0;
  }
  // RSOC leading pair: geometric mean (reading A21)
  for (const Cone& c : P.pc)
    if (c.kind == K_RSOC) {
      int64_t a = P.n1 + c.off;
      double g = std::sqrt(q[a] * q[a + 1]);
      q[a] = g; q[a + 1] = g;
    }
  for (const Cone& c : P.rc)
    if (c.kind == K_RSOC) {
      int64_t a = c.off;
      double g = std::sqrt(r[a] * r[a + 1]);
      r[a] = g; r[a + 1] = g;
    }
}

// ---------------------------------------------------------------- solver
struct Solver {
  Problem P;
  Params prm;
  // scaled data
  Csr K, KT;
  vector<double> r, q, ct, ht, lt, ut;
  // iterate state (scaled space)
  vector<double> x, y, xh, yh, x0, y0, xsum, ysum;
  double Wsum = 0.0;
  double eta = 0.0, eta_init = 0.0, omega = 1.0, beta = 1.0;
  int64_t k = 0, total = 0, trials = 0, restarts = 0, nK = 0, nKT = 0;
  double r_start = 0.0, e_anchor = 0.0, e_prev = -1.0;
  int status = ST_RUNNING;
  double best_e = INF;
  vector<double> best_x, best_y, cand_x, cand_y;
  Kkt last_cur{}, last_avg{}, best_kkt{};
  vector<int32_t> trace;        // decisions: 1 accept,0 reject,10+cand,20+restart
  double vanilla_step = 0.0;
  double last_num = 0.0, last_cross = 0.0, last_cross_abs = 0.0;

  // x in X~ = [q l, q u] x prod diag(q_B) K_B  (Eq. 5 primal projection)
  void proj_X(double* v) const {
    for (int64_t j = 0; j < P.n1; ++j) v[j] = proj_box(v[j], lt[j], ut[j]);
    for (const Cone& c : P.pc) {
      double* b = v + P.n1 + c.off;
      const double* D = q.data() + P.n1 + c.off;
      project_block(c.kind, c.dim, b, D, /*dual_side=*/false);
    }
  }
  // y in prod diag(r_b) C_b^*  (Eq. 5 dual projection, reading A1)
  void proj_Y(double* v) const {
    for (const Cone& c : P.rc) {
      double* b = v + c.off;
      const double* D = r.data() + c.off;
      project_block(c.kind, c.dim, b, D, /*dual_side=*/true);
    }
  }
  // Project one block onto diag(D) K (primal side) or diag(D) K^* (row side).
  static void project_block(int kind, int64_t d, double* b, const double* D, bool dual_side) {
    vector<double> o(d);
    switch (kind) {
      case K_ZERO:
        if (!dual_side) for (int64_t i = 0; i < d; ++i) b[i] = 0.0;   // x in {0}; y free
        return;
      case K_NONNEG:
        for (int64_t i = 0; i < d; ++i) b[i] = std::max(b[i], 0.0);
        return;
      case K_SOC:
        proj_soc_scaled(d, b, D, o.data());
        break;
      case K_RSOC:
        proj_rsoc_scaled(d, b, D, o.data());
        break;
      case K_EXP:          // primal: D K_exp ; row (C = K_exp): y in D K_exp^*
        if (dual_side) proj_dual_exp_scaled(b, D, o.data()); else proj_exp_scaled(b, D, o.data());
        break;
      case K_DUAL_EXP:     // primal: D K_exp^* ; row (C = K_exp^*): y in D K_exp
        if (dual_side) proj_exp_scaled(b, D, o.data()); else proj_dual_exp_scaled(b, D, o.data());
        break;
    }
    for (int64_t i = 0; i < d; ++i) b[i] = o[i];
  }

  // ------------------------------------------------------------ Eq. 9 (original space)
  Kkt kkt(const double* xs, const double* ys) const {
    const int64_t m = P.m, n = P.n, n1 = P.n1;
    vector<double> xo(n), yo(m), Gx(m), Gty(n);
    for (int64_t j = 0; j < n; ++j) xo[j] = xs[j] / q[j];
    for (int64_t i = 0; i < m; ++i) yo[i] = ys[i] / r[i];
    spmv(P.G, xo.data(), Gx.data());
    spmv(P.GT, yo.data(), Gty.data());
    // err_p: distance of Gx - h to C = K_d^* (unit scaling)
    vector<double> res(m), pr(m);
    for (int64_t i = 0; i < m; ++i) res[i] = Gx[i] - P.h[i];
    for (const Cone& c : P.rc) {
      const double* v = res.data() + c.off;
      double* o = pr.data() + c.off;
      switch (c.kind) {
        case K_ZERO: for (int64_t i = 0; i < c.dim; ++i) o[i] = 0.0; break;
        case K_NONNEG: for (int64_t i = 0; i < c.dim; ++i) o[i] = std::max(v[i], 0.0); break;
        case K_SOC: proj_soc_unit(c.dim, v, o); break;
        case K_RSOC: proj_rsoc_scaled(c.dim, v, nullptr, o); break;
        case K_EXP: proj_exp_scaled(v, ONE3, o); break;
        case K_DUAL_EXP: proj_dual_exp_scaled(v, ONE3, o); break;
      }
    }
    double num_p = 0.0;
    for (int64_t i = 0; i < m; ++i) num_p = std::max(num_p, std::fabs(res[i] - pr[i]));
    double den_p = 1.0 + std::max(nrminf(P.h.data(), m), std::max(nrminf(Gx.data(), m), nrminf(pr.data(), m)));
    // err_d: lambda = c - G^T y; lambda_1 vs Lambda (Eq. 3), lambda_2 vs K_p^*
    vector<double> lam(n);
    for (int64_t j = 0; j < n; ++j) lam[j] = P.c[j] - Gty[j];
    double num_d = 0.0, dual_obj_box = 0.0;
    for (int64_t j = 0; j < n1; ++j) {
      bool fl = std::isfinite(P.l[j]), fu = std::isfinite(P.u[j]);
      double pl;                                         // P_Lambda (Eq. 3)
      if (!fl && !fu) pl = 0.0;
      else if (!fl) pl = std::min(lam[j], 0.0);
      else if (!fu) pl = std::max(lam[j], 0.0);
      else pl = lam[j];
      num_d = std::max(num_d, std::fabs(lam[j] - pl));
      // dual objective with lambda~_1 = P_Lambda(lambda_1) (reading A13)
      if (fl) dual_obj_box += P.l[j] * std::max(pl, 0.0);
      if (fu) dual_obj_box -= P.u[j] * std::max(-pl, 0.0);
    }
    for (const Cone& c : P.pc) {
      const double* v = lam.data() + n1 + c.off;
      vector<double> o(c.dim);
      switch (c.kind) {                                  // K_p^* blocks
        case K_ZERO: for (int64_t i = 0; i < c.dim; ++i) o[i] = v[i]; break;   // R^d
        case K_NONNEG: for (int64_t i = 0; i < c.dim; ++i) o[i] = std::max(v[i], 0.0); break;
        case K_SOC: proj_soc_unit(c.dim, v, o.data()); break;
        case K_RSOC: proj_rsoc_scaled(c.dim, v, nullptr, o.data()); break;
        case K_EXP: proj_dual_exp_scaled(v, ONE3, o.data()); break;
        case K_DUAL_EXP: proj_exp_scaled(v, ONE3, o.data()); break;
      }
      for (int64_t i = 0; i < c.dim; ++i) num_d = std::max(num_d, std::fabs(v[i] - o[i]));
    }
    double den_d = 1.0 + std::max(nrminf(P.c.data(), n), nrminf(Gty.data(), n));
    double pobj = dot(P.c.data(), xo.data(), n);
    double dobj = dot(yo.data(), P.h.data(), m) + dual_obj_box;
    Kkt K;
    K.err_p = num_p / den_p;
    K.err_d = num_d / den_d;
    K.err_gap = std::fabs(pobj - dobj) / (1.0 + std::max(std::fabs(pobj), std::fabs(dobj)));
    K.pobj = pobj;
    K.dobj = dobj;
    return K;
  }
  static double kmax(const Kkt& k) { return std::max(k.err_p, std::max(k.err_d, k.err_gap)); }

  // ------------------------------------------------------------ setup
  void setup() {
    const int64_t m = P.m, n = P.n;
    if (!prm.vanilla_pdhg && (prm.ruiz_iters > 0 || prm.pock_chambolle))
      ruiz_scale(P, prm.ruiz_iters, prm.pock_chambolle, r, q);
    else { r.assign(m, 1.0); q.assign(n, 1.0); }
    K = P.G;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t p = K.ptr[i]; p < K.ptr[i + 1]; ++p) K.val[p] = P.G.val[p] / (r[i] * q[K.col[p]]);
    KT = transpose(K);
    ct.resize(n); ht.resize(m); lt.resize(P.n1); ut.resize(P.n1);
    for (int64_t j = 0; j < n; ++j) ct[j] = P.c[j] / q[j];
    for (int64_t i = 0; i < m; ++i) ht[i] = P.h[i] / r[i];
    for (int64_t j = 0; j < P.n1; ++j) { lt[j] = q[j] * P.l[j]; ut[j] = q[j] * P.u[j]; }
    // initial point z00 = (P_X(0), 0) (reading A4)
    x.assign(n, 0.0); y.assign(m, 0.0);
    proj_X(x.data());
    xh = x; yh = y; x0 = x; y0 = y;
    xsum.assign(n, 0.0); ysum.assign(m, 0.0); Wsum = 0.0;
    if (prm.vanilla_pdhg) {
      // tau = sigma = 0.9/||G||_2 by power iteration
      double nrm = prm.eta0 > 0.0 ? 0.9 / prm.eta0 : power_norm();
      vanilla_step = prm.eta0 > 0.0 ? prm.eta0 : (nrm > 0.0 ? 0.9 / nrm : 1.0);
      eta = eta_init = vanilla_step;
      omega = 1.0;
    } else {
      // eta0 = 1/||K~||_inf (reading A5)
      double mx = 0.0;
      for (int64_t i = 0; i < m; ++i) {
        double s = 0.0;
        for (int64_t p = K.ptr[i]; p < K.ptr[i + 1]; ++p) s += std::fabs(K.val[p]);
        mx = std::max(mx, s);
      }
      eta = prm.eta0 > 0.0 ? prm.eta0 : (mx > 0.0 ? 1.0 / mx : 1.0);
      eta_init = eta;
      // omega0 (reading A6)
      double cn = nrminf(ct.data(), n), hn = nrminf(ht.data(), m);
      if (prm.omega0 > 0.0) omega = prm.omega0;
      else if (cn > 0.0 && hn > 0.0) omega = std::min(std::max(cn / hn, 1e-4), 1e4);
      else omega = 1.0;
    }
    beta = prm.beta_max;
    e_anchor = kmax(kkt(x.data(), y.data()));
    e_prev = -1.0;
  }

  // ||G||_2 estimate: power iteration on G^T G, start 1/sqrt(n)
  double power_norm() {
    const int64_t n = P.n, m = P.m;
    vector<double> v(n, 1.0 / std::sqrt((double)std::max<int64_t>(n, 1))), Gv(m), w(n);
    double lam = 0.0;
    for (int it = 0; it < 20; ++it) {
      spmv(K, v.data(), Gv.data());
      spmv(KT, Gv.data(), w.data());
      double nw = nrm2(w.data(), n);
      if (nw == 0.0) return 0.0;
      double prev = lam;
      lam = nw;
      for (int64_t j = 0; j < n; ++j) v[j] = w[j] / nw;
      if (it > 0 && std::fabs(lam - prev) < 1e-4 * lam) break;
    }
    return std::sqrt(lam);
  }

  // One PDHG step (Eq. 5) from (x, y) with steps tau, sigma.
  // Products recomputed fresh (3 SpMVs, reading A28).
  void one_pdhg(double tau, double sigma, vector<double>& Kxh, vector<double>& Kx) {
    const int64_t m = P.m, n = P.n;
    vector<double> KTy(n);
    spmv(KT, y.data(), KTy.data()); nKT++;
    for (int64_t j = 0; j < n; ++j) xh[j] = x[j] - tau * (ct[j] - KTy[j]);
    proj_X(xh.data());
    Kxh.resize(m); Kx.resize(m);
    spmv(K, xh.data(), Kxh.data()); nK++;
    spmv(K, x.data(), Kx.data()); nK++;
    for (int64_t i = 0; i < m; ++i) yh[i] = y[i] + sigma * (ht[i] - 2.0 * Kxh[i] + Kx[i]);
    proj_Y(yh.data());
  }

  // One accepted inner iteration of Alg. 1 (lines 4-7).
  bool inner_step() {
    const int64_t m = P.m, n = P.n;
    vector<double> Kxh, Kx;
    if (prm.vanilla_pdhg) {
      one_pdhg(vanilla_step, vanilla_step, Kxh, Kx);
      trials++;
      x = xh; y = yh;
      k++; total++;
      return true;
    }
    // AdaptiveStepPDHG (line 4): line search (reading A7)
    int rejects = 0;
    double eta_used = 0.0, num = 0.0;
    for (;;) {
      double tau = eta / omega, sigma = eta * omega;
      one_pdhg(tau, sigma, Kxh, Kx);
      double dxx = 0.0, dyy = 0.0, cross = 0.0;
      for (int64_t j = 0; j < n; ++j) { double d = xh[j] - x[j]; dxx += d * d; }
      for (int64_t i = 0; i < m; ++i) {
        double d = yh[i] - y[i];
        dyy += d * d;
        cross += d * (Kxh[i] - Kx[i]);
      }
      num = omega * dxx + dyy / omega;
      double etabar = ls_bound(num, cross);
      last_num = num; last_cross = cross;
      last_cross_abs = 0.0;
      for (int64_t i = 0; i < m; ++i) last_cross_abs += std::fabs((yh[i] - y[i]) * (Kxh[i] - Kx[i]));
      trials++;
      if (eta <= etabar) {
        trace.push_back(1);
        eta_used = eta;
        eta = std::min(prm.ls_grow * eta, etabar);
        break;
      }
      trace.push_back(0);
      eta *= prm.ls_shrink;
      rejects++;
      if (eta < 1e-12 * eta_init || rejects > prm.ls_max_rejects) { status = ST_NUMERICAL; return false; }
    }
    // AdaptiveReflectionParameter (line 5): window rule (reading A9)
    beta = reflection_beta(k, prm.refl_window, std::sqrt(num), &r_start, beta);
    // ReflectedHalpern (line 6, PAPER.md:606 verbatim)
    double a, b;
    halpern_coef(k, &a, &b);
    for (int64_t j = 0; j < n; ++j) x[j] = a * ((1.0 + beta) * xh[j] - beta * x[j]) + b * x0[j];
    for (int64_t i = 0; i < m; ++i) y[i] = a * ((1.0 + beta) * yh[i] - beta * y[i]) + b * y0[i];
    // step-weighted average (line 7; reading A8: weight = step that produced z)
    for (int64_t j = 0; j < n; ++j) xsum[j] += eta_used * x[j];
    for (int64_t i = 0; i < m; ++i) ysum[i] += eta_used * y[i];
    Wsum += eta_used;
    k++; total++;
    return true;
  }

  // Residual check every check_interval inner iterations:
  // GetRestartCandidate (line 8), restart condition (line 3), PrimalWeightUpdate
  // (line 11).  Returns true when the termination criterion holds.
  bool check() {
    const int64_t m = P.m, n = P.n;
    if (prm.vanilla_pdhg) {
      Kkt kc = kkt(x.data(), y.data());
      last_cur = kc;
      double e = kmax(kc);
      if (e < best_e) { best_e = e; best_x = x; best_y = y; best_kkt = kc; }
      return e <= prm.tol;
    }
    // candidates (reading A10): current = z^ (feasible), average = P(zbar)
    Kkt kc = kkt(xh.data(), yh.data());
    vector<double> xa(n), ya(m);
    for (int64_t j = 0; j < n; ++j) xa[j] = xsum[j] / Wsum;
    for (int64_t i = 0; i < m; ++i) ya[i] = ysum[i] / Wsum;
    proj_X(xa.data());
    proj_Y(ya.data());
    nK++; nKT++;                       // products of the average candidate
    Kkt ka = kkt(xa.data(), ya.data());
    last_cur = kc; last_avg = ka;
    double ec = kmax(kc), ea = kmax(ka);
    bool use_avg = candidate_is_average(ec, ea);
    trace.push_back(use_avg ? 11 : 10);
    const vector<double>& xc = use_avg ? xa : xh;
    const vector<double>& yc = use_avg ? ya : yh;
    double e = use_avg ? ea : ec;
    cand_x = xc; cand_y = yc;
    if (e < best_e) { best_e = e; best_x = xc; best_y = yc; best_kkt = use_avg ? ka : kc; }
    const bool done = e <= prm.tol;
    bool restart = restart_rule(e, e_anchor, e_prev, k, total, prm.restart_suff, prm.restart_nec,
                                prm.restart_art);
    e_prev = e;
    trace.push_back(restart ? 21 : 20);
    if (restart) {
      // PrimalWeightUpdate (reading A12)
      double dxn = 0.0, dyn = 0.0;
      for (int64_t j = 0; j < n; ++j) { double d = xc[j] - x0[j]; dxn += d * d; }
      for (int64_t i = 0; i < m; ++i) { double d = yc[i] - y0[i]; dyn += d * d; }
      dxn = std::sqrt(dxn); dyn = std::sqrt(dyn);
      omega = primal_weight(dxn, dyn, omega);
      x0 = xc; y0 = yc; x = xc; y = yc;
      e_anchor = e;
      k = 0;
      std::fill(xsum.begin(), xsum.end(), 0.0);
      std::fill(ysum.begin(), ysum.end(), 0.0);
      Wsum = 0.0;
      beta = prm.beta_max;
      e_prev = -1.0;
      restarts++;
    }
    return done;
  }

  void iterate(int64_t nsteps) {
    for (int64_t s = 0; s < nsteps && status == ST_RUNNING; ++s) {
      if (!inner_step()) return;
      if (k > 0 && k % prm.check_interval == 0) check();
    }
  }

  Result solve() {
    auto t0 = std::chrono::steady_clock::now();
    while (status == ST_RUNNING) {
      if (!inner_step()) break;
      if (k > 0 && k % prm.check_interval == 0) {
        if (check()) { status = ST_OPTIMAL; break; }
      }
      if (total >= prm.max_iters) { status = ST_ITER_LIMIT; break; }
      double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (prm.time_limit_s > 0 && el > prm.time_limit_s) { status = ST_TIME_LIMIT; break; }
    }
    Result R{};
    R.status = status;
    R.kkt = best_kkt;
    R.iters = total; R.trials = trials; R.restarts = restarts;
    R.spmv_K = nK; R.spmv_KT = nKT;
    R.eta = eta; R.omega = omega; R.beta = beta;
    R.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return R;
  }
};

}  // namespace orc

// ============================================================================
//  C ABI of the oracle (called from tests via ctypes).  orc_* names only.
// ============================================================================
using namespace orc;

extern "C" {

void orc_spmv(int64_t m, const int64_t* ptr, const int32_t* col, const double* val,
              const double* x, double* y) {
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) s += val[p] * x[col[p]];
    y[i] = s;
  }
}

void orc_spmv_t(int64_t m, int64_t n, const int64_t* ptr, const int32_t* col,
                const double* val, const double* y, double* x) {
  Csr A;
  A.m = m; A.n = n;
  A.ptr.assign(ptr, ptr + m + 1);
  A.col.assign(col, col + ptr[m]);
  A.val.assign(val, val + ptr[m]);
  Csr T = transpose(A);
  spmv(T, y, x);
}

void orc_proj_soc_unit(int64_t d, const double* v, double* out) { proj_soc_unit(d, v, out); }
void orc_proj_soc_scaled(int64_t d, const double* v, const double* D, double* out) {
  proj_soc_scaled(d, v, D, out);
}
void orc_proj_rsoc_scaled(int64_t d, const double* v, const double* D, double* out) {
  proj_rsoc_scaled(d, v, D, out);
}
void orc_proj_exp_scaled(const double* v, const double* D, double* out) { proj_exp_scaled(v, D, out); }
void orc_proj_dual_exp_scaled(const double* v, const double* D, double* out) {
  proj_dual_exp_scaled(v, D, out);
}
int orc_in_exp(const double* v, double tol) { return in_exp(v[0], v[1], v[2], tol); }
int orc_in_exp_dual(const double* v, double tol) { return in_exp_dual(v[0], v[1], v[2], tol); }
double orc_exp_det(const double* v, const double* D, double rho) {
  return exp_det(v[0], v[1], v[2], D[0], D[1], D[2], rho);
}
int64_t orc_rootfail_count(void) { return g_rootfail; }
double orc_ls_bound(double num, double cross) { return ls_bound(num, cross); }
void orc_halpern_coef(int64_t k, double* a, double* b) { halpern_coef(k, a, b); }
int orc_restart_rule(double e, double ea, double ep, int64_t k, int64_t total, double s, double n,
                     double a) { return restart_rule(e, ea, ep, k, total, s, n, a); }
double orc_primal_weight(double dxn, double dyn, double omega) { return primal_weight(dxn, dyn, omega); }
double orc_reflection_beta(int64_t k, int64_t W, double res, double* r_start, double beta) {
  return reflection_beta(k, W, res, r_start, beta);
}
int orc_candidate_is_average(double e_current, double e_average) {
  return candidate_is_average(e_current, e_average);
}
void orc_ruiz(int64_t m, int64_t n, int64_t n1, const int64_t* ptr, const int32_t* col,
              const double* val, const int32_t* pk, const int64_t* pdim, int64_t npc,
              const int32_t* rk, const int64_t* rdim, int64_t nrc, int ruiz_iters, int pc,
              double* r, double* q) {
  Problem P;
  P.m = m; P.n = n; P.n1 = n1;
  P.G.m = m; P.G.n = n;
  P.G.ptr.assign(ptr, ptr + m + 1);
  P.G.col.assign(col, col + ptr[m]);
  P.G.val.assign(val, val + ptr[m]);
  int64_t off = 0;
  for (int64_t b = 0; b < npc; ++b) { P.pc.push_back({pk[b], pdim[b], off}); off += pdim[b]; }
  off = 0;
  for (int64_t b = 0; b < nrc; ++b) { P.rc.push_back({rk[b], rdim[b], off}); off += rdim[b]; }
  vector<double> rr, qq;
  ruiz_scale(P, ruiz_iters, pc, rr, qq);
  std::copy(rr.begin(), rr.end(), r);
  std::copy(qq.begin(), qq.end(), q);
}

void* orc_create(int64_t m, int64_t n, int64_t n1, const int64_t* ptr, const int32_t* col,
                 const double* val, const double* c, const double* h, const double* l,
                 const double* u, const int32_t* pk, const int64_t* pdim, int64_t npc,
                 const int32_t* rk, const int64_t* rdim, int64_t nrc, const Params* prm) {
  Solver* S = new Solver();
  Problem& P = S->P;
  P.m = m; P.n = n; P.n1 = n1;
  P.G.m = m; P.G.n = n;
  P.G.ptr.assign(ptr, ptr + m + 1);
  P.G.col.assign(col, col + ptr[m]);
  P.G.val.assign(val, val + ptr[m]);
  P.GT = transpose(P.G);
  P.c.assign(c, c + n); P.h.assign(h, h + m);
  P.l.assign(l, l + n1); P.u.assign(u, u + n1);
  int64_t off = 0;
  for (int64_t b = 0; b < npc; ++b) { P.pc.push_back({pk[b], pdim[b], off}); off += pdim[b]; }
  off = 0;
  for (int64_t b = 0; b < nrc; ++b) { P.rc.push_back({rk[b], rdim[b], off}); off += rdim[b]; }
  S->prm = *prm;
  S->setup();
  return S;
}

void orc_destroy(void* h) { delete (Solver*)h; }
void orc_iterate(void* h, int64_t n) { ((Solver*)h)->iterate(n); }
int orc_status(void* h) { return ((Solver*)h)->status; }
void orc_solve(void* h, Result* out) { *out = ((Solver*)h)->solve(); }

// which: 0 current iterate z, 1 last PDHG output z^, 2 anchor, 3 best, 4 last candidate
// space: 0 scaled, 1 original
void orc_get_iterate(void* h, int which, int space, double* x, double* y) {
  Solver* S = (Solver*)h;
  const vector<double>* X = &S->x;
  const vector<double>* Y = &S->y;
  if (which == 1) { X = &S->xh; Y = &S->yh; }
  if (which == 2) { X = &S->x0; Y = &S->y0; }
  if (which == 3) { X = &S->best_x; Y = &S->best_y; }
  if (which == 4) { X = &S->cand_x; Y = &S->cand_y; }
  for (int64_t j = 0; j < S->P.n; ++j) x[j] = space ? (*X)[j] / S->q[j] : (*X)[j];
  for (int64_t i = 0; i < S->P.m; ++i) y[i] = space ? (*Y)[i] / S->r[i] : (*Y)[i];
}
void orc_get_scaling(void* h, double* r, double* q) {
  Solver* S = (Solver*)h;
  std::copy(S->r.begin(), S->r.end(), r);
  std::copy(S->q.begin(), S->q.end(), q);
}
// KKT (Eq. 9) of which (0 current z, 1 z^, 2 anchor, 3 best); out[5]
void orc_kkt(void* h, int which, double* out) {
  Solver* S = (Solver*)h;
  const vector<double>* X = &S->x;
  const vector<double>* Y = &S->y;
  if (which == 1) { X = &S->xh; Y = &S->yh; }
  if (which == 2) { X = &S->x0; Y = &S->y0; }
  if (which == 3) { X = &S->best_x; Y = &S->best_y; }
  Kkt k = S->kkt(X->data(), Y->data());
  out[0] = k.err_p; out[1] = k.err_d; out[2] = k.err_gap; out[3] = k.pobj; out[4] = k.dobj;
}
// Set the current iterate (scaled space); it also becomes the anchor.
void orc_set_iterate(void* h, const double* x, const double* y) {
  Solver* S = (Solver*)h;
  std::copy(x, x + S->P.n, S->x.begin());
  std::copy(y, y + S->P.m, S->y.begin());
  S->x0 = S->x; S->y0 = S->y; S->xh = S->x; S->yh = S->y;
  S->e_anchor = S->kmax(S->kkt(S->x.data(), S->y.data()));
  // a new epoch at the given point, as pdcs_set_iterate (include/pdcs.h)
  std::fill(S->xsum.begin(), S->xsum.end(), 0.0);
  std::fill(S->ysum.begin(), S->ysum.end(), 0.0);
  S->Wsum = 0.0; S->k = 0; S->beta = S->prm.beta_max; S->e_prev = -1.0;
}
// Full Alg. 1 state (scaled space) for checkpoint shadowing.
void orc_get_state(void* h, double* x, double* y, double* x0, double* y0, double* xs, double* ys,
                   double* sc) {
  Solver* S = (Solver*)h;
  std::copy(S->x.begin(), S->x.end(), x); std::copy(S->y.begin(), S->y.end(), y);
  std::copy(S->x0.begin(), S->x0.end(), x0); std::copy(S->y0.begin(), S->y0.end(), y0);
  std::copy(S->xsum.begin(), S->xsum.end(), xs); std::copy(S->ysum.begin(), S->ysum.end(), ys);
  const double v[13] = {S->eta, S->eta_init, S->omega, S->beta, S->Wsum, S->r_start, S->e_anchor,
                        S->e_prev, S->best_e, (double)S->k, (double)S->total, (double)S->trials,
                        (double)S->restarts};
  std::copy(v, v + 13, sc);
}
// Eq. 9 at an ORIGINAL-space point (x, y).
void orc_kkt_point(void* h, const double* x, const double* y, double* out) {
  Solver* S = (Solver*)h;
  vector<double> xs(S->P.n), ys(S->P.m);
  for (int64_t j = 0; j < S->P.n; ++j) xs[j] = x[j] * S->q[j];
  for (int64_t i = 0; i < S->P.m; ++i) ys[i] = y[i] * S->r[i];
  Kkt k = S->kkt(xs.data(), ys.data());
  out[0] = k.err_p; out[1] = k.err_d; out[2] = k.err_gap; out[3] = k.pobj; out[4] = k.dobj;
}
// Scalars: eta, omega, beta, k, total, trials, restarts, e_anchor, W
void orc_scalars(void* h, double* out) {
  Solver* S = (Solver*)h;
  out[0] = S->eta; out[1] = S->omega; out[2] = S->beta; out[3] = (double)S->k;
  out[4] = (double)S->total; out[5] = (double)S->trials; out[6] = (double)S->restarts;
  out[7] = S->e_anchor; out[8] = S->Wsum; out[9] = S->eta_init;
  const Kkt* ks[2] = {&S->last_cur, &S->last_avg};
  for (int c = 0; c < 2; ++c) {
    out[10 + 5 * c] = ks[c]->err_p; out[11 + 5 * c] = ks[c]->err_d; out[12 + 5 * c] = ks[c]->err_gap;
    out[13 + 5 * c] = ks[c]->pobj; out[14 + 5 * c] = ks[c]->dobj;
  }
  out[20] = S->e_prev; out[21] = S->best_e;
  out[22] = S->last_num; out[23] = S->last_cross; out[24] = S->last_cross_abs;
}
int64_t orc_trace(void* h, int32_t* out, int64_t cap) {
  Solver* S = (Solver*)h;
  int64_t nn = (int64_t)S->trace.size();
  for (int64_t i = 0; i < std::min(nn, cap); ++i) out[i] = S->trace[i];
  return nn;
}
}
