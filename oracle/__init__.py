"""PDCS CPU oracle — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/liboracle.so`` (single-threaded C++, fp64, built
from ``oracle/pdcs_oracle.cpp``).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
module.  It shares no code with the product package ``paper_2505_00311_b200``.

Parity-unpinned items are listed in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pdcs_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++ -O2, no fast-math, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


P_D = C.POINTER(C.c_double)
P_I64 = C.POINTER(C.c_int64)
P_I32 = C.POINTER(C.c_int32)


class Params(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int64), ("time_limit_s", C.c_double),
                ("ruiz_iters", C.c_int32), ("pock_chambolle", C.c_int32),
                ("check_interval", C.c_int32), ("vanilla_pdhg", C.c_int32),
                ("eta0", C.c_double), ("omega0", C.c_double), ("beta_max", C.c_double),
                ("refl_window", C.c_int32), ("pad0", C.c_int32),
                ("restart_suff", C.c_double), ("restart_nec", C.c_double),
                ("restart_art", C.c_double), ("ls_shrink", C.c_double), ("ls_grow", C.c_double),
                ("ls_max_rejects", C.c_int32), ("verbose", C.c_int32)]


class Kkt(C.Structure):
    _fields_ = [("err_p", C.c_double), ("err_d", C.c_double), ("err_gap", C.c_double),
                ("pobj", C.c_double), ("dobj", C.c_double)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_int32), ("kkt", Kkt),
                ("iters", C.c_int64), ("trials", C.c_int64), ("restarts", C.c_int64),
                ("spmv_K", C.c_int64), ("spmv_KT", C.c_int64), ("eta", C.c_double),
                ("omega", C.c_double), ("beta", C.c_double), ("solve_seconds", C.c_double)]


DEFAULTS = dict(tol=1e-6, max_iters=1_000_000, time_limit_s=0.0, ruiz_iters=10,
                pock_chambolle=1, check_interval=40, vanilla_pdhg=0, eta0=0.0, omega0=0.0,
                beta_max=1.0, refl_window=40, pad0=0, restart_suff=0.2, restart_nec=0.8,
                restart_art=0.36, ls_shrink=0.5, ls_grow=1.05, ls_max_rejects=60, verbose=0)


def make_params(**kw) -> Params:
    d = dict(DEFAULTS)
    d.update(kw)
    return Params(**d)


def _declare(L):
    L.orc_spmv.argtypes = [C.c_int64, P_I64, P_I32, P_D, P_D, P_D]
    L.orc_spmv_t.argtypes = [C.c_int64, C.c_int64, P_I64, P_I32, P_D, P_D, P_D]
    L.orc_proj_soc_unit.argtypes = [C.c_int64, P_D, P_D]
    L.orc_proj_soc_scaled.argtypes = [C.c_int64, P_D, P_D, P_D]
    L.orc_proj_rsoc_scaled.argtypes = [C.c_int64, P_D, P_D, P_D]
    L.orc_proj_exp_scaled.argtypes = [P_D, P_D, P_D]
    L.orc_proj_dual_exp_scaled.argtypes = [P_D, P_D, P_D]
    L.orc_in_exp.argtypes = [P_D, C.c_double]
    L.orc_in_exp_dual.argtypes = [P_D, C.c_double]
    L.orc_exp_det.argtypes = [P_D, P_D, C.c_double]
    L.orc_exp_det.restype = C.c_double
    L.orc_rootfail_count.restype = C.c_int64
    L.orc_ls_bound.argtypes = [C.c_double, C.c_double]
    L.orc_ls_bound.restype = C.c_double
    L.orc_halpern_coef.argtypes = [C.c_int64, P_D, P_D]
    L.orc_restart_rule.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64,
                                   C.c_double, C.c_double, C.c_double]
    L.orc_primal_weight.argtypes = [C.c_double, C.c_double, C.c_double]
    L.orc_primal_weight.restype = C.c_double
    L.orc_reflection_beta.argtypes = [C.c_int64, C.c_int64, C.c_double, P_D, C.c_double]
    L.orc_reflection_beta.restype = C.c_double
    L.orc_candidate_is_average.argtypes = [C.c_double, C.c_double]
    L.orc_ruiz.argtypes = [C.c_int64, C.c_int64, C.c_int64, P_I64, P_I32, P_D, P_I32, P_I64,
                           C.c_int64, P_I32, P_I64, C.c_int64, C.c_int, C.c_int, P_D, P_D]
    L.orc_set_iterate.argtypes = [C.c_void_p, P_D, P_D]
    L.orc_kkt_point.argtypes = [C.c_void_p, P_D, P_D, P_D]
    L.orc_get_state.argtypes = [C.c_void_p] + [P_D] * 7
    L.orc_create.argtypes = [C.c_int64, C.c_int64, C.c_int64, P_I64, P_I32, P_D, P_D, P_D, P_D,
                             P_D, P_I32, P_I64, C.c_int64, P_I32, P_I64, C.c_int64,
                             C.POINTER(Params)]
    L.orc_create.restype = C.c_void_p
    L.orc_destroy.argtypes = [C.c_void_p]
    L.orc_iterate.argtypes = [C.c_void_p, C.c_int64]
    L.orc_status.argtypes = [C.c_void_p]
    L.orc_solve.argtypes = [C.c_void_p, C.POINTER(Result)]
    L.orc_get_iterate.argtypes = [C.c_void_p, C.c_int, C.c_int, P_D, P_D]
    L.orc_get_scaling.argtypes = [C.c_void_p, P_D, P_D]
    L.orc_kkt.argtypes = [C.c_void_p, C.c_int, P_D]
    L.orc_scalars.argtypes = [C.c_void_p, P_D]
    L.orc_trace.argtypes = [C.c_void_p, P_I32, C.c_int64]
    L.orc_trace.restype = C.c_int64


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(P_D)


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(P_I64)


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(P_I32)


# ------------------------------------------------------------------ primitives
def spmv(row_ptr, col, val, x):
    m = len(row_ptr) - 1
    y = np.zeros(m)
    a, b, c, d = _i64(row_ptr), _i32(col), _d(val), _d(x)
    lib().orc_spmv(m, a[1], b[1], c[1], d[1], y.ctypes.data_as(P_D))
    return y


def spmv_t(row_ptr, col, val, y, n):
    m = len(row_ptr) - 1
    x = np.zeros(n)
    a, b, c, d = _i64(row_ptr), _i32(col), _d(val), _d(y)
    lib().orc_spmv_t(m, n, a[1], b[1], c[1], d[1], x.ctypes.data_as(P_D))
    return x


def proj_soc_unit(v):
    v = _d(v)
    out = np.zeros(len(v[0]))
    lib().orc_proj_soc_unit(len(v[0]), v[1], out.ctypes.data_as(P_D))
    return out


def proj_soc_scaled(v, D):
    v, D = _d(v), _d(D)
    out = np.zeros(len(v[0]))
    lib().orc_proj_soc_scaled(len(v[0]), v[1], D[1], out.ctypes.data_as(P_D))
    return out


def proj_rsoc_scaled(v, D=None):
    v = _d(v)
    out = np.zeros(len(v[0]))
    if D is None:
        lib().orc_proj_rsoc_scaled(len(v[0]), v[1], None, out.ctypes.data_as(P_D))
    else:
        D = _d(D)
        lib().orc_proj_rsoc_scaled(len(v[0]), v[1], D[1], out.ctypes.data_as(P_D))
    return out


def proj_exp_scaled(v, D=(1.0, 1.0, 1.0)):
    v, D = _d(v), _d(D)
    out = np.zeros(3)
    lib().orc_proj_exp_scaled(v[1], D[1], out.ctypes.data_as(P_D))
    return out


def proj_dual_exp_scaled(v, D=(1.0, 1.0, 1.0)):
    v, D = _d(v), _d(D)
    out = np.zeros(3)
    lib().orc_proj_dual_exp_scaled(v[1], D[1], out.ctypes.data_as(P_D))
    return out


def in_exp(v, tol=0.0):
    v = _d(v)
    return bool(lib().orc_in_exp(v[1], tol))


def in_exp_dual(v, tol=0.0):
    v = _d(v)
    return bool(lib().orc_in_exp_dual(v[1], tol))


def exp_det(v, D, rho):
    v, D = _d(v), _d(D)
    return lib().orc_exp_det(v[1], D[1], rho)


def rootfail_count():
    return int(lib().orc_rootfail_count())


def ls_bound(num, cross):
    return lib().orc_ls_bound(num, cross)


def halpern_coef(k):
    a, b = C.c_double(), C.c_double()
    lib().orc_halpern_coef(k, C.byref(a), C.byref(b))
    return a.value, b.value


def restart_rule(e, e_anchor, e_prev, k, total, suff=0.2, nec=0.8, art=0.36):
    return bool(lib().orc_restart_rule(e, e_anchor, e_prev, k, total, suff, nec, art))


def primal_weight(dxn, dyn, omega):
    return lib().orc_primal_weight(dxn, dyn, omega)


def reflection_beta(k, W, res, r_start, beta):
    """One application of the window rule; returns (beta', r_start')."""
    rs = C.c_double(r_start)
    b = lib().orc_reflection_beta(k, W, res, C.byref(rs), beta)
    return b, rs.value


def candidate_is_average(e_current, e_average):
    return bool(lib().orc_candidate_is_average(e_current, e_average))


def ruiz(prog, ruiz_iters=10, pc=1):
    r = np.zeros(prog.m)
    q = np.zeros(prog.n)
    k = [_i64(prog.row_ptr), _i32(prog.col_idx), _d(prog.vals), _i32(prog.pk), _i64(prog.pdim),
         _i32(prog.rk), _i64(prog.rdim)]
    lib().orc_ruiz(prog.m, prog.n, prog.n1, k[0][1], k[1][1], k[2][1], k[3][1], k[4][1],
                   len(prog.pk), k[5][1], k[6][1], len(prog.rk), ruiz_iters, pc,
                   r.ctypes.data_as(P_D), q.ctypes.data_as(P_D))
    return r, q


# ------------------------------------------------------------------ solver
class OracleSolver:
    """Handle over the oracle's Alg. 1 state machine (create -> iterate/solve)."""

    def __init__(self, prog, **params):
        L = lib()
        self.prog = prog
        self.params = make_params(**params)
        self._keep = [_i64(prog.row_ptr), _i32(prog.col_idx), _d(prog.vals), _d(prog.c),
                      _d(prog.h), _d(prog.l), _d(prog.u), _i32(prog.pk), _i64(prog.pdim),
                      _i32(prog.rk), _i64(prog.rdim)]
        k = self._keep
        self.h = L.orc_create(prog.m, prog.n, prog.n1, k[0][1], k[1][1], k[2][1], k[3][1],
                              k[4][1], k[5][1], k[6][1], k[7][1], k[8][1], len(prog.pk),
                              k[9][1], k[10][1], len(prog.rk), C.byref(self.params))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def iterate(self, n: int):
        lib().orc_iterate(self.h, n)
        return lib().orc_status(self.h)

    def solve(self) -> Result:
        r = Result()
        lib().orc_solve(self.h, C.byref(r))
        return r

    def get_iterate(self, which=0, space=0):
        x = np.zeros(self.prog.n)
        y = np.zeros(self.prog.m)
        lib().orc_get_iterate(self.h, which, space, x.ctypes.data_as(P_D), y.ctypes.data_as(P_D))
        return x, y

    def get_scaling(self):
        r = np.zeros(self.prog.m)
        q = np.zeros(self.prog.n)
        lib().orc_get_scaling(self.h, r.ctypes.data_as(P_D), q.ctypes.data_as(P_D))
        return r, q

    def kkt(self, which=0):
        out = np.zeros(5)
        lib().orc_kkt(self.h, which, out.ctypes.data_as(P_D))
        return dict(err_p=out[0], err_d=out[1], err_gap=out[2], pobj=out[3], dobj=out[4])

    def scalars(self):
        out = np.zeros(25)
        lib().orc_scalars(self.h, out.ctypes.data_as(P_D))
        keys = ["eta", "omega", "beta", "k", "total", "trials", "restarts", "e_anchor", "W",
                "eta0", "cur_err_p", "cur_err_d", "cur_err_gap", "cur_pobj", "cur_dobj",
                "avg_err_p", "avg_err_d", "avg_err_gap", "avg_pobj", "avg_dobj", "e_prev", "best_e",
                "last_num", "last_cross", "last_cross_abs"]
        return dict(zip(keys, out))

    def set_iterate(self, x, y):
        x, y = _d(x), _d(y)
        lib().orc_set_iterate(self.h, x[1], y[1])

    def get_state(self):
        n, m = self.prog.n, self.prog.m
        v = {k: np.zeros(n if k[0] == "x" else m) for k in ("x", "y", "x0", "y0", "xsum", "ysum")}
        sc = np.zeros(13)
        lib().orc_get_state(self.h, *[v[k].ctypes.data_as(P_D) for k in ("x", "y", "x0", "y0", "xsum",
                                                                         "ysum")], sc.ctypes.data_as(P_D))
        v["sc"] = sc
        return v

    def kkt_point(self, x, y):
        """Eq. 9 at an original-space point."""
        x, y = _d(x), _d(y)
        out = np.zeros(5)
        lib().orc_kkt_point(self.h, x[1], y[1], out.ctypes.data_as(P_D))
        return dict(err_p=out[0], err_d=out[1], err_gap=out[2], pobj=out[3], dobj=out[4])

    def trace(self):
        n = lib().orc_trace(self.h, None, 0)
        out = np.zeros(n, np.int32)
        lib().orc_trace(self.h, out.ctypes.data_as(P_I32), n)
        return out
