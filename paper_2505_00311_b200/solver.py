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

    def __init__(self, prog, device: int = 0, stream=None, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, rows=None, loopback=None, **params):
        """rows=(row_begin, row_end) selects this rank's shard (dist.partition_rows);
        nccl_id (128 bytes from pdcs_nccl_unique_id on rank 0) enables the
        NCCL path (also usable with world == 1); loopback (a group from
        pdcs_loopback_create) makes this rank one of N in-process ranks."""
        from . import dist
        self.prog = prog
        self.params = L.pdcs_default_params(**params)
        r0, r1 = rows if rows is not None else getattr(prog, "rows", (0, prog.m))
        self.rows = (r0, r1)
        sh = dist.shard(prog, r0, r1)
        self._arrays = dict(
            row_ptr=sh["row_ptr"], col=np.ascontiguousarray(sh["col"], np.int32),
            val=np.ascontiguousarray(sh["val"], np.float64),
            c=np.ascontiguousarray(prog.c, np.float64), h=np.ascontiguousarray(sh["h"], np.float64),
            l=np.ascontiguousarray(prog.l, np.float64), u=np.ascontiguousarray(prog.u, np.float64))
        a = self._arrays
        idbuf = None
        if nccl_id is not None:
            idbuf = np.frombuffer(bytes(nccl_id), dtype=np.uint8).copy()
        if loopback is not None:           # in-process loopback group (pdcs_loopback_create)
            self.ctx = L.pdcs_create_loopback(prog.m, prog.n, prog.n1, r0, r1, a["row_ptr"], a["col"],
                                              a["val"], a["c"], a["h"], a["l"], a["u"], self.params, device,
                                              stream, group=loopback, rank=rank)
        else:
            self.ctx = L.pdcs_create(prog.m, prog.n, prog.n1, r0, r1, a["row_ptr"], a["col"], a["val"],
                                     a["c"], a["h"], a["l"], a["u"], self.params, device, stream,
                                     nccl_unique_id=idbuf, rank=rank, world=world)
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

    def set_tolerance(self, tol: float, time_limit_s: float = 0.0):
        L.pdcs_set_tolerance(self.ctx, tol, time_limit_s)

    def kkt(self, which=L.CURRENT) -> dict:
        k = L.pdcs_kkt(self.ctx, which)
        return dict(err_p=k.err_p, err_d=k.err_d, err_gap=k.err_gap, pobj=k.pobj, dobj=k.dobj)

    def get_iterate(self, which=L.CURRENT, space=L.SCALED):
        x = np.zeros(self.prog.n)
        y = np.zeros(self.rows[1] - self.rows[0])
        L.pdcs_get_iterate(self.ctx, which, space, x, y)
        return x, y

    def set_iterate(self, x, y):
        L.pdcs_set_iterate(self.ctx, np.ascontiguousarray(x, np.float64),
                           np.ascontiguousarray(y, np.float64))

    def get_scaling(self):
        r = np.zeros(self.rows[1] - self.rows[0])
        q = np.zeros(self.prog.n)
        L.pdcs_get_scaling(self.ctx, r, q)
        return r, q

    def enable_timing(self, on=True):
        L.pdcs_enable_timing(self.ctx, on)

    def kernel_times(self):
        return L.pdcs_kernel_times(self.ctx)

    def get_state(self):
        return L.pdcs_get_state(self.ctx, self.prog.n, self.rows[1] - self.rows[0])

    def set_state(self, st):
        L.pdcs_set_state(self.ctx, st)

    def scalars(self):
        return L.pdcs_get_scalars(self.ctx)

    def launch_count(self):
        return L.pdcs_launch_count(self.ctx)
