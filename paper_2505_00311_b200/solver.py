"""Convenience handle over the C ABI (no arithmetic of the method here)."""
from __future__ import annotations

import numpy as np

from . import _lib as L


def _result_dict(r) -> dict:
    return dict(status=L.SOLVE_STATUS.get(r.status, r.status), err_p=r.kkt.err_p,
                err_d=r.kkt.err_d, err_gap=r.kkt.err_gap, pobj=r.kkt.pobj, dobj=r.kkt.dobj,
                iters=r.iters, trials=r.trials, restarts=r.restarts, eta=r.eta, omega=r.omega,
                beta=r.beta, seconds=r.solve_seconds)


class PdcsSolver:
    """create -> set_cones on construction; iterate / solve / kkt / get_iterate after."""

    def __init__(self, prog, device: int = 0, stream=None, **params):
        self.prog = prog
        self.params = L.pdcs_default_params(**params)
        self._arrays = dict(
            row_ptr=np.ascontiguousarray(prog.row_ptr, np.int64),
            col=np.ascontiguousarray(prog.col_idx, np.int32),
            val=np.ascontiguousarray(prog.vals, np.float64),
            c=np.ascontiguousarray(prog.c, np.float64), h=np.ascontiguousarray(prog.h, np.float64),
            l=np.ascontiguousarray(prog.l, np.float64), u=np.ascontiguousarray(prog.u, np.float64))
        a = self._arrays
        self.ctx = L.pdcs_create(prog.m, prog.n, prog.n1, 0, prog.m, a["row_ptr"], a["col"], a["val"],
                                 a["c"], a["h"], a["l"], a["u"], self.params, device, stream)
        L.pdcs_set_cones(self.ctx, prog.pk, prog.pdim, prog.rk, prog.rdim)

    def close(self):
        if getattr(self, "ctx", None):
            L.pdcs_destroy(self.ctx)
            self.ctx = None

    __del__ = close

    def iterate(self, n: int) -> dict:
        return _result_dict(L.pdcs_iterate(self.ctx, n))

    def solve(self) -> dict:
        return _result_dict(L.pdcs_solve(self.ctx))

    def kkt(self, which=L.CURRENT) -> dict:
        k = L.pdcs_kkt(self.ctx, which)
        return dict(err_p=k.err_p, err_d=k.err_d, err_gap=k.err_gap, pobj=k.pobj, dobj=k.dobj)

    def get_iterate(self, which=L.CURRENT, space=L.SCALED):
        x = np.zeros(self.prog.n)
        y = np.zeros(self.prog.m)
        L.pdcs_get_iterate(self.ctx, which, space, x, y)
        return x, y

    def set_iterate(self, x, y):
        L.pdcs_set_iterate(self.ctx, np.ascontiguousarray(x, np.float64),
                           np.ascontiguousarray(y, np.float64))

    def get_scaling(self):
        r = np.zeros(self.prog.m)
        q = np.zeros(self.prog.n)
        L.pdcs_get_scaling(self.ctx, r, q)
        return r, q

    def enable_timing(self, on=True):
        L.pdcs_enable_timing(self.ctx, on)

    def kernel_times(self):
        return L.pdcs_kernel_times(self.ctx)

    def get_state(self):
        return L.pdcs_get_state(self.ctx, self.prog.n, self.prog.m)

    def set_state(self, st):
        L.pdcs_set_state(self.ctx, st)

    def scalars(self):
        return L.pdcs_get_scalars(self.ctx)

    def launch_count(self):
        return L.pdcs_launch_count(self.ctx)
