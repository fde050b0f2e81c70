"""Thin ctypes binding over libpdcs.so (include/pdcs.h).

Argument marshalling only: every step of the method runs in the CUDA kernels
of the library.  There is no CPU fallback — if the shared library is missing
or no sm_100 device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDCS_LIB") or os.path.join(_HERE, "libpdcs.so")   # PDCS_LIB: tuning builds

P_D = C.POINTER(C.c_double)
P_I64 = C.POINTER(C.c_int64)
P_I32 = C.POINTER(C.c_int32)

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_DIM", 3: "ERR_BOUNDS", 4: "ERR_NONFINITE", 5: "ERR_CONE",
          6: "ERR_SHARD", 7: "ERR_CUDA", 8: "ERR_NCCL", 9: "ERR_NUMERICAL", 10: "ERR_STATE"}
SOLVE_STATUS = {0: "OPTIMAL", 1: "ITERATION_LIMIT", 2: "TIME_LIMIT", 3: "NUMERICAL_ERROR",
                4: "RUNNING"}
CURRENT, PDHG_OUT, ANCHOR, BEST, CANDIDATE = 0, 1, 2, 3, 4
SCALED, ORIGINAL = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1


class pdcs_params(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int64), ("time_limit_s", C.c_double),
                ("ruiz_iters", C.c_int32), ("pock_chambolle", C.c_int32),
                ("check_interval", C.c_int32), ("vanilla_pdhg", C.c_int32),
                ("eta0", C.c_double), ("omega0", C.c_double), ("beta_max", C.c_double),
                ("refl_window", C.c_int32), ("pad0", C.c_int32),
                ("restart_suff", C.c_double), ("restart_nec", C.c_double),
                ("restart_art", C.c_double), ("ls_shrink", C.c_double), ("ls_grow", C.c_double),
                ("ls_max_rejects", C.c_int32), ("verbose", C.c_int32)]


class pdcs_kkt_t(C.Structure):
    _fields_ = [("err_p", C.c_double), ("err_d", C.c_double), ("err_gap", C.c_double),
                ("pobj", C.c_double), ("dobj", C.c_double)]


class pdcs_result_t(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad", C.c_int32), ("kkt", pdcs_kkt_t),
                ("iters", C.c_int64), ("trials", C.c_int64), ("restarts", C.c_int64),
                ("spmv_K", C.c_int64), ("spmv_KT", C.c_int64), ("eta", C.c_double),
                ("omega", C.c_double), ("beta", C.c_double), ("solve_seconds", C.c_double)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class PdcsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libpdcs.so (built by paper_2505_00311_b200.build.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2505_00311_b200.build.build() "
                              "(the CUDA path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.pdcs_default_params.argtypes = [C.POINTER(pdcs_params)]
        L.pdcs_last_error.argtypes = [C.c_void_p]
        L.pdcs_last_error.restype = C.c_char_p
        L.pdcs_create.argtypes = [C.POINTER(C.c_void_p), C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(pdcs_params), C.c_int,
                                  C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int]
        L.pdcs_create_loopback.argtypes = [C.POINTER(C.c_void_p), C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(pdcs_params),
                                           C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        L.pdcs_set_allocator.argtypes = [ALLOC_FN, FREE_FN, C.c_void_p]
        L.pdcs_trim_memory.argtypes = []
        L.pdcs_trim_memory.restype = C.c_int64
        L.pdcs_loopback_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
        L.pdcs_loopback_destroy.argtypes = [C.c_void_p]
        L.pdcs_set_cones.argtypes = [C.c_void_p, P_I32, P_I64, C.c_int64, P_I32, P_I64, C.c_int64]
        L.pdcs_iterate.argtypes = [C.c_void_p, C.c_int64, C.POINTER(pdcs_result_t)]
        L.pdcs_kkt.argtypes = [C.c_void_p, C.c_int, C.POINTER(pdcs_kkt_t)]
        L.pdcs_solve.argtypes = [C.c_void_p, C.POINTER(pdcs_result_t)]
        L.pdcs_set_tolerance.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.pdcs_get_iterate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.pdcs_set_iterate.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.pdcs_get_scaling.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.pdcs_kernel_times.argtypes = [C.c_void_p, C.c_void_p, P_D, P_I64, C.c_int]
        L.pdcs_enable_timing.argtypes = [C.c_void_p, C.c_int]
        L.pdcs_get_state.argtypes = [C.c_void_p] + [C.c_void_p] * 6 + [P_D]
        L.pdcs_set_state.argtypes = [C.c_void_p] + [C.c_void_p] * 6 + [P_D]
        L.pdcs_get_scalars.argtypes = [C.c_void_p, P_D, C.c_int]
        L.pdcs_launch_count.argtypes = [C.c_void_p]
        L.pdcs_launch_count.restype = C.c_int64
        L.pdcs_destroy.argtypes = [C.c_void_p]
        L.pdcs_nccl_unique_id.argtypes = [C.c_void_p]
        L.pdcs_tiled_layout_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                                              C.c_void_p, C.c_int]
        L.pdcs_tiled_layout_stats.restype = C.c_int
        L.pdcs_tiled_build_host.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.pdcs_tiled_build_host.restype = C.c_int
        L.pdcs_tiled_device_check.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.pdcs_tiled_device_check.restype = C.c_int
        L.pdcs_tiled_devbuild_check.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.pdcs_tiled_devbuild_check.restype = C.c_int
        L.pdcs_proj_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, P_I32, P_I64, C.c_int64, C.c_int]
        L.pdcs_proj_run.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.pdcs_proj_info.argtypes = [C.c_void_p, P_I64, P_I64]
        L.pdcs_proj_info.restype = C.c_int
        L.pdcs_proj_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


EXPORTED = ["pdcs_default_params", "pdcs_create", "pdcs_set_cones", "pdcs_iterate", "pdcs_kkt",
            "pdcs_solve", "pdcs_get_iterate", "pdcs_set_iterate", "pdcs_get_scaling",
            "pdcs_kernel_times", "pdcs_enable_timing", "pdcs_launch_count", "pdcs_last_error",
            "pdcs_destroy", "pdcs_nccl_unique_id", "pdcs_get_scalars", "pdcs_get_state",
            "pdcs_set_state", "pdcs_tiled_layout_stats", "pdcs_proj_create", "pdcs_proj_run",
            "pdcs_proj_info", "pdcs_proj_destroy", "pdcs_set_tolerance", "pdcs_tiled_build_host",
            "pdcs_loopback_create", "pdcs_loopback_destroy", "pdcs_create_loopback", "pdcs_tiled_device_check",
            "pdcs_tiled_devbuild_check",
            "pdcs_set_allocator", "pdcs_trim_memory"]

STATE_KEYS = ["eta", "eta_init", "omega", "beta", "W", "r_start", "e_anchor", "e_prev", "best_e", "k",
              "total", "trials", "restarts"]

SCALAR_KEYS = ["eta", "omega", "beta", "k", "total", "trials", "restarts", "e_anchor", "W", "eta0",
               "cur_err_p", "cur_err_d", "cur_err_gap", "cur_pobj", "cur_dobj",
               "avg_err_p", "avg_err_d", "avg_err_gap", "avg_pobj", "avg_dobj",
               "e_prev", "best_e", "use_avg", "restart", "last_num", "last_cross",
               "tiled_K", "tune_K_csr_ms", "tune_K_tiled_ms", "tiled_KT", "tune_KT_csr_ms",
               "tune_KT_tiled_ms", "tiled_K_build_ms", "tiled_KT_build_ms", "setup_create_ms",
               "setup_cones_ms", "colperm", "panels_K", "tune_K_csr_ms_p", "tune_K_panel_ms", "panels_KT",
               "tune_KT_csr_ms_p", "tune_KT_panel_ms", "fused_K", "tune_K_fused_ms", "fused_KT",
               "tune_KT_fused_ms", "csr_u_K", "csr_u_KT"]


def _check(code, ctx=None):
    if code != 0:
        msg = lib().pdcs_last_error(ctx)
        raise PdcsError(code, msg.decode() if msg else "")


def _ptr(a):
    """Address of a contiguous numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- C-ABI names
def pdcs_default_params(**overrides) -> pdcs_params:
    p = pdcs_params()
    lib().pdcs_default_params(C.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def pdcs_create(m_global, n, n1, row_begin, row_end, row_ptr, col_idx, vals, c, h, l, u,
                params=None, device=0, stream=None, mem_kind=MEM_HOST, nccl_unique_id=None,
                rank=0, world=1):
    ctx = C.c_void_p()
    keep = [row_ptr, col_idx, vals, c, h, l, u]
    code = lib().pdcs_create(C.byref(ctx), m_global, n, n1, row_begin, row_end, _ptr(row_ptr),
                             _ptr(col_idx), _ptr(vals), _ptr(c), _ptr(h), _ptr(l), _ptr(u),
                             C.byref(params) if params is not None else None, device,
                             C.c_void_p(stream) if stream else None, mem_kind,
                             _ptr(nccl_unique_id), rank, world)
    del keep
    _check(code)
    return ctx


def pdcs_create_loopback(m_global, n, n1, row_begin, row_end, row_ptr, col_idx, vals, c, h, l, u,
                         params=None, device=0, stream=None, mem_kind=MEM_HOST, group=None, rank=0):
    ctx = C.c_void_p()
    keep = [row_ptr, col_idx, vals, c, h, l, u]
    code = lib().pdcs_create_loopback(C.byref(ctx), m_global, n, n1, row_begin, row_end, _ptr(row_ptr),
                                      _ptr(col_idx), _ptr(vals), _ptr(c), _ptr(h), _ptr(l), _ptr(u),
                                      C.byref(params) if params is not None else None, device,
                                      C.c_void_p(stream) if stream else None, mem_kind, group, rank)
    del keep
    _check(code)
    return ctx


_allocator_refs = None


def pdcs_trim_memory() -> int:
    """Release the library pool's unused device memory; returns the bytes released."""
    k = lib().pdcs_trim_memory()
    if k < 0:
        raise PdcsError(7, "pdcs_trim_memory failed")
    return int(k)


def pdcs_set_allocator(alloc=None, free=None):
    """alloc(nbytes) -> int device pointer, free(ptr) -> None (Python callables,
    e.g. torch's caching allocator); None, None restores cudaMalloc."""
    global _allocator_refs
    if alloc is None and free is None:
        _check(lib().pdcs_set_allocator(ALLOC_FN(), FREE_FN(), None))
        _allocator_refs = None
        return
    fa = ALLOC_FN(lambda nbytes, user: alloc(int(nbytes)) or None)
    ff = FREE_FN(lambda ptr, user: free(int(ptr)))
    _check(lib().pdcs_set_allocator(fa, ff, None))
    _allocator_refs = (fa, ff)          # keep the trampolines alive


def pdcs_loopback_create(world: int):
    g = C.c_void_p()
    _check(lib().pdcs_loopback_create(C.byref(g), world))
    return g


def pdcs_loopback_destroy(group):
    lib().pdcs_loopback_destroy(group)


def pdcs_set_cones(ctx, pk, pdim, rk, rdim):
    pk = np.ascontiguousarray(pk, np.int32)
    pdim = np.ascontiguousarray(pdim, np.int64)
    rk = np.ascontiguousarray(rk, np.int32)
    rdim = np.ascontiguousarray(rdim, np.int64)
    _check(lib().pdcs_set_cones(ctx, pk.ctypes.data_as(P_I32), pdim.ctypes.data_as(P_I64), len(pk),
                                rk.ctypes.data_as(P_I32), rdim.ctypes.data_as(P_I64), len(rk)), ctx)


def pdcs_iterate(ctx, n_inner) -> pdcs_result_t:
    r = pdcs_result_t()
    _check(lib().pdcs_iterate(ctx, n_inner, C.byref(r)), ctx)
    return r


def pdcs_solve(ctx) -> pdcs_result_t:
    r = pdcs_result_t()
    _check(lib().pdcs_solve(ctx, C.byref(r)), ctx)
    return r


def pdcs_tiled_build_host(row_ptr, col, rows, nvec, elem) -> dict:
    """Host-only timing of the tiled-format build (no device)."""
    out = np.zeros(3)
    rp = np.ascontiguousarray(row_ptr, np.int64); cl = np.ascontiguousarray(col, np.int32)
    n = lib().pdcs_tiled_build_host(rp.ctypes.data, cl.ctypes.data, rows, nvec, elem, out.ctypes.data)
    if n != 3:
        raise ValueError("pdcs_tiled_build_host: bad arguments")
    return dict(build_ms=out[0], ranges_ms=out[1], staged=int(out[2]))


def pdcs_tiled_device_check(row_ptr, col, rows, nvec, elem) -> dict:
    rp = np.ascontiguousarray(row_ptr, np.int64)
    c = np.ascontiguousarray(col, np.int32)
    out = np.zeros(5)
    k = lib().pdcs_tiled_device_check(_ptr(rp), _ptr(c), rows, nvec, elem, out.ctypes.data_as(P_D))
    if k != 5:
        raise PdcsError(7 if k < 0 else 1, "pdcs_tiled_device_check failed" if k < 0 else "not applicable")
    return dict(mismatches=out[0], host_ms=out[1], deferred_host_ms=out[2], device_ms=out[3], entries=out[4])


def pdcs_tiled_devbuild_check(row_ptr, col, rows, nvec, elem) -> dict:
    rp = np.ascontiguousarray(row_ptr, np.int64)
    c = np.ascontiguousarray(col, np.int32)
    out = np.zeros(5)
    k = lib().pdcs_tiled_devbuild_check(_ptr(rp), _ptr(c), rows, nvec, elem, out.ctypes.data_as(P_D))
    if k != 5:
        raise PdcsError(7 if k < 0 else 1, "pdcs_tiled_devbuild_check failed" if k < 0 else "not applicable")
    return dict(mismatches=out[0], host_ms=out[1], device_ms=out[2], staged=out[3], entries=out[4])


def pdcs_set_tolerance(ctx, tol, time_limit_s=0.0):
    _check(lib().pdcs_set_tolerance(ctx, float(tol), float(time_limit_s)), ctx)


def pdcs_kkt(ctx, which=CURRENT) -> pdcs_kkt_t:
    k = pdcs_kkt_t()
    _check(lib().pdcs_kkt(ctx, which, C.byref(k)), ctx)
    return k


def pdcs_get_iterate(ctx, which, space, x, y):
    _check(lib().pdcs_get_iterate(ctx, which, space, _ptr(x), _ptr(y)), ctx)


def pdcs_set_iterate(ctx, x, y):
    _check(lib().pdcs_set_iterate(ctx, _ptr(x), _ptr(y)), ctx)


def pdcs_get_scaling(ctx, r, q):
    _check(lib().pdcs_get_scaling(ctx, _ptr(r), _ptr(q)), ctx)


def pdcs_enable_timing(ctx, on=True):
    lib().pdcs_enable_timing(ctx, 1 if on else 0)


def pdcs_kernel_times(ctx, cap=64):
    names = (C.c_char * 32 * cap)()
    ms = np.zeros(cap)
    cnt = np.zeros(cap, np.int64)
    k = lib().pdcs_kernel_times(ctx, names, ms.ctypes.data_as(P_D), cnt.ctypes.data_as(P_I64), cap)
    return {bytes(names[i]).split(b"\0")[0].decode(): (float(ms[i]), int(cnt[i])) for i in range(k)}


def pdcs_get_state(ctx, n, m):
    """-> dict of scaled-space vectors x, y, x0, y0, xsum, ysum and the 13 scalars."""
    v = {k: np.zeros(n if k[0] == "x" else m) for k in ("x", "y", "x0", "y0", "xsum", "ysum")}
    sc = np.zeros(13)
    _check(lib().pdcs_get_state(ctx, *[_ptr(v[k]) for k in ("x", "y", "x0", "y0", "xsum", "ysum")],
                                sc.ctypes.data_as(P_D)), ctx)
    v["sc"] = sc
    return v


def pdcs_set_state(ctx, st):
    arrs = [np.ascontiguousarray(st[k], np.float64) for k in ("x", "y", "x0", "y0", "xsum", "ysum")]
    sc = np.ascontiguousarray(st["sc"], np.float64)
    _check(lib().pdcs_set_state(ctx, *[_ptr(a) for a in arrs], sc.ctypes.data_as(P_D)), ctx)


def pdcs_get_scalars(ctx) -> dict:
    out = np.zeros(len(SCALAR_KEYS))
    k = lib().pdcs_get_scalars(ctx, out.ctypes.data_as(P_D), len(SCALAR_KEYS))
    return dict(zip(SCALAR_KEYS[:k], out[:k]))


def pdcs_launch_count(ctx) -> int:
    return int(lib().pdcs_launch_count(ctx))


def pdcs_last_error(ctx=None) -> str:
    s = lib().pdcs_last_error(ctx)
    return s.decode() if s else ""


def pdcs_destroy(ctx):
    lib().pdcs_destroy(ctx)


def pdcs_nccl_unique_id():
    buf = (C.c_char * 128)()
    _check(lib().pdcs_nccl_unique_id(buf))
    return bytes(buf)


TILED_STAT_KEYS = ["nnz", "staged", "quads", "pads", "segments", "work_items", "lds_inst", "lds_wavefronts",
                   "build_ms", "lds_wavefront_bound", "structure_errors"]


def pdcs_tiled_layout_stats(row_ptr, col, nvec: int, elem: int) -> dict:
    """Host-only model of the tiled layout (no GPU): see include/pdcs.h."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    out = np.zeros(len(TILED_STAT_KEYS))
    k = lib().pdcs_tiled_layout_stats(rp.ctypes.data, cc.ctypes.data, rp.shape[0] - 1, int(nvec), int(elem),
                                      out.ctypes.data, len(TILED_STAT_KEYS))
    if k == 0:
        raise PdcsError(-1, "pdcs_tiled_layout_stats: bad arguments")
    return dict(zip(TILED_STAT_KEYS[:k], out[:k]))


# ---------------------------------------------------------------- standalone projections
TEAMS = {"auto": -1, "thread": 0, "warp": 1, "cta": 2, "cluster": 3, "grid": 4}


def pdcs_proj_create(kinds, dims, team=-1, device=0):
    """Plan of a multi-cone projection (include/pdcs.h): kinds/dims host arrays."""
    k = np.ascontiguousarray(kinds, np.int32)
    d = np.ascontiguousarray(dims, np.int64)
    h = C.c_void_p()
    team = TEAMS[team] if isinstance(team, str) else int(team)
    _check(lib().pdcs_proj_create(C.byref(h), int(device), k.ctypes.data_as(P_I32), d.ctypes.data_as(P_I64),
                                  k.shape[0], team))
    return h


def pdcs_proj_run(plan, D, v, out, stream=None):
    """out = P_{diag(D) K}(v); D, v, out device tensors / pointers (D None: unit)."""
    st = None if stream is None else C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    _check(lib().pdcs_proj_run(plan, None if D is None else _ptr(D), _ptr(v), _ptr(out), st))


def pdcs_proj_info(plan):
    counts = np.zeros(5, np.int64)
    grids = np.zeros(5, np.int64)
    lib().pdcs_proj_info(plan, counts.ctypes.data_as(P_I64), grids.ctypes.data_as(P_I64))
    return {"counts": counts.tolist(), "grids": grids.tolist()}


def pdcs_proj_destroy(plan):
    lib().pdcs_proj_destroy(plan)
