"""Row-sharded PDCS through libpdcs.so at world 2 and 4 on ONE GPU (-m gpu).

SURVEY §8(e): K is row-partitioned; the only exchanges are all-reduces.  The
ranks are `world` contexts of this process on cuda:0 joined by an in-process
loopback group (include/pdcs.h, pdcs_loopback_create), each driven from its own
host thread (ctypes releases the GIL).  Checked:
  * per-iterate parity of the assembled shards against the CPU oracle under
    checkpoint shadowing (the oracle's exact state is loaded into every rank
    every `seg` iterations; every 4th segment ends on an Eq. 9 check with its
    restart and primal-weight decisions), tolerance as tests/test_gpu_parity.py;
  * every rank holds bitwise-identical decisions: the control-block scalars and
    the replicated primal iterate are equal on all ranks after every segment;
  * a time-limited solve stops every rank at the same check.
"""
import threading

import numpy as np
import pytest

import oracle as O
from instances import gen_lasso, gen_mixed

pytestmark = pytest.mark.gpu

TOL = 1e-9
STOL = 1e-6


@pytest.fixture(scope="module")
def P():
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    return P


def on_all(fns):
    """Run one callable per rank concurrently; return their results in rank order."""
    out = [None] * len(fns)
    err = [None] * len(fns)

    def run(i):
        try:
            out[i] = fns[i]()
        except BaseException as e:   # noqa: BLE001 - re-raised below
            err[i] = e

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=900)
    for e in err:
        if e is not None:
            raise e
    return out


def make_ranks(P, prog, world, **params):
    from paper_2505_00311_b200 import dist as D
    parts = D.partition_rows(prog.row_ptr, prog.rk, prog.rdim, world)
    assert all(b > a for a, b in parts), parts
    group = P.pdcs_loopback_create(world)
    ranks = on_all([lambda r=r: P.PdcsSolver(prog, rank=r, world=world, rows=parts[r], loopback=group,
                                             **params) for r in range(world)])
    return group, parts, ranks


def rel(a, b):
    return np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))) if a.size else 0.0


DECISION_KEYS = ["eta", "omega", "beta", "k", "total", "trials", "restarts", "e_anchor", "W", "eta0",
                 "cur_err_p", "cur_err_d", "cur_err_gap", "cur_pobj", "cur_dobj", "avg_err_p", "avg_err_d",
                 "avg_err_gap", "avg_pobj", "avg_dobj", "e_prev", "best_e", "use_avg", "restart", "last_num",
                 "last_cross"]


def assert_ranks_identical(ranks):
    sc = [g.scalars() for g in ranks]
    for k in DECISION_KEYS:
        vals = [s[k] for s in sc]
        assert all(v == vals[0] or (np.isnan(v) and np.isnan(vals[0])) for v in vals), (k, vals)
    st = [g.get_state() for g in ranks]
    for s in st[1:]:
        assert np.array_equal(s["sc"], st[0]["sc"])
        for k in ("x", "x0", "xsum"):
            assert np.array_equal(s[k], st[0][k]), k


CASES = {
    "mixed": lambda: gen_mixed(600, 60, 240, seed=21, soc_dims=(3, 40)),
    "lasso": lambda: gen_lasso(400, 40, 0.2, seed=3),
}


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_loopback_shadow_parity_and_identical_decisions(P, name, world, monkeypatch):
    monkeypatch.setenv("PDCS_TILED", "0")     # the same SpMV format on every rank (setup autotune is timed)
    prog = CASES[name]()
    group, parts, ranks = make_ranks(P, prog, world)
    o = O.OracleSolver(prog)
    # scaling: each rank's r is the oracle's on its rows; q is global
    sc = on_all([lambda g=g: g.get_scaling() for g in ranks])
    ro, qo = o.get_scaling()
    for (a, b), (rg, qg) in zip(parts, sc):
        np.testing.assert_allclose(rg, ro[a:b], rtol=1e-13)
        np.testing.assert_allclose(qg, qo, rtol=1e-13)
    seg, steps = 10, 400
    worst = 0.0
    for s in range(0, steps, seg):
        so = o.get_state()
        loc = [dict(x=so["x"], y=so["y"][a:b], x0=so["x0"], y0=so["y0"][a:b], xsum=so["xsum"],
                    ysum=so["ysum"][a:b], sc=so["sc"]) for a, b in parts]
        on_all([lambda g=g, st=st: g.set_state(st) for g, st in zip(ranks, loc)])
        on_all([lambda g=g: g.iterate(seg) for g in ranks])
        o.iterate(seg)
        assert_ranks_identical(ranks)
        xo, yo = o.get_iterate(0)
        its = [g.get_iterate(P.CURRENT) for g in ranks]
        yg = np.concatenate([y for _, y in its])
        worst = max(worst, rel(its[0][0], xo), rel(yg, yo))
        sg, so2 = ranks[0].get_state(), o.get_state()
        assert np.array_equal(sg["sc"][9:], so2["sc"][9:]), (s, sg["sc"], so2["sc"])
        assert sg["sc"][3] == so2["sc"][3]
        for i in (0, 2, 4):
            assert abs(sg["sc"][i] - so2["sc"][i]) <= STOL * abs(so2["sc"][i]), (s, i)
    assert worst <= TOL, worst
    for g in ranks:
        g.close()
    P.pdcs_loopback_destroy(group)


@pytest.mark.parametrize("world", [2, 4])
def test_loopback_free_running_matches_single_gpu(P, world, monkeypatch):
    """The sharded path vs the unsharded one over the first 120 free-running
    iterations (checks and restart decisions included; the window where the
    oracle's own rounding sensitivity stays below 1e-9, P5): same
    decisions, iterates to 1e-9 (the row-sum order of K^T y differs)."""
    monkeypatch.setenv("PDCS_TILED", "0")
    prog = CASES["mixed"]()
    group, parts, ranks = make_ranks(P, prog, world)
    g0 = P.PdcsSolver(prog)
    for _ in range(3):
        on_all([lambda g=g: g.iterate(40) for g in ranks])
        g0.iterate(40)
        assert_ranks_identical(ranks)
        s0, s1 = g0.scalars(), ranks[0].scalars()
        assert s0["restarts"] == s1["restarts"] and s0["trials"] == s1["trials"]
        x0, y0 = g0.get_iterate(P.CURRENT)
        its = [g.get_iterate(P.CURRENT) for g in ranks]
        assert rel(its[0][0], x0) <= TOL and rel(np.concatenate([y for _, y in its]), y0) <= TOL


def test_loopback_solve_and_time_limit_stop_together(P, monkeypatch):
    """pdcs_solve on 2 ranks: the same status, iteration count and residuals on
    both, to tolerance; a time-limited solve stops both at the same check."""
    monkeypatch.setenv("PDCS_TILED", "0")
    prog = gen_mixed(400, 60, 200, seed=30, soc_dims=(3, 30))
    group, parts, ranks = make_ranks(P, prog, 2, tol=1e-7, max_iters=200000)
    res = on_all([lambda g=g: g.solve() for g in ranks])
    assert res[0]["status"] == "OPTIMAL" and res[0] == {**res[1], "seconds": res[0]["seconds"]}
    assert abs(res[0]["pobj"] - prog.obj_star) <= 1e-5 * (1 + abs(prog.obj_star))
    # a solve again reports the same finished result, iterate refuses until set_tolerance
    again = on_all([lambda g=g: g.solve() for g in ranks])
    assert again[0]["iters"] == res[0]["iters"] and again[0]["status"] == "OPTIMAL"
    with pytest.raises(P.PdcsError):
        ranks[0].iterate(1)
    # time limit: a tiny limit on a long solve stops both ranks at one check
    group, parts, ranks = make_ranks(P, gen_lasso(2000, 200, 0.05, seed=5, balance=False), 2, tol=1e-12,
                                     time_limit_s=0.5)
    res = on_all([lambda g=g: g.solve() for g in ranks])
    assert res[0]["status"] == res[1]["status"] == "TIME_LIMIT"
    assert res[0]["iters"] == res[1]["iters"] and res[0]["iters"] > 0


def test_loopback_failing_rank_does_not_hang_peers(P, monkeypatch):
    """A rank that fails before a collective aborts the group: the peer's call
    returns an error instead of waiting forever."""
    monkeypatch.setenv("PDCS_LOOPBACK_TIMEOUT_S", "60")
    prog = gen_mixed(200, 20, 80, seed=2, soc_dims=(3, 20))
    from paper_2505_00311_b200 import dist as D
    parts = D.partition_rows(prog.row_ptr, prog.rk, prog.rdim, 2)
    group = P.pdcs_loopback_create(2)

    def bad():
        # rank 1 passes inconsistent cones: set_cones fails before its first collective
        g = P.PdcsSolver.__new__(P.PdcsSolver)
        prog2 = gen_mixed(200, 20, 80, seed=2, soc_dims=(3, 20))
        prog2.rdim = prog2.rdim.copy()
        prog2.rdim[0] += 1
        P.PdcsSolver.__init__(g, prog2, rank=1, world=2, rows=parts[1], loopback=group)

    def good():
        P.PdcsSolver(prog, rank=0, world=2, rows=parts[0], loopback=group)

    out = [None, None]

    def wrap(i, f):
        try:
            f()
        except Exception as e:   # noqa: BLE001
            out[i] = e

    ts = [threading.Thread(target=wrap, args=(0, good)), threading.Thread(target=wrap, args=(1, bad))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts)
    assert isinstance(out[0], P.PdcsError) and isinstance(out[1], P.PdcsError), out


@pytest.mark.parametrize("world", [2, 3])
def test_chunked_overlapped_allreduce_is_bit_identical(P, world, monkeypatch):
    """The K^T y partial all-reduced in row chunks on a second stream, each
    overlapping the next chunk's sums (PDCS_AR_CHUNKS), gives the same bits as
    one all-reduce of the whole vector: the reduction is elementwise."""
    monkeypatch.setenv("PDCS_TILED", "0")
    prog = CASES["mixed"]()
    out = {}
    for chunks in ("1", "3"):
        monkeypatch.setenv("PDCS_AR_CHUNKS", chunks)
        group, parts, ranks = make_ranks(P, prog, world)
        on_all([lambda g=g: g.iterate(150) for g in ranks])
        assert_ranks_identical(ranks)
        out[chunks] = (ranks[0].get_state(), [g.get_iterate(P.CURRENT)[1] for g in ranks])
        for g in ranks:
            g.close()
        P.pdcs_loopback_destroy(group)
    (sa, ya), (sb, yb) = out["1"], out["3"]
    assert np.array_equal(sa["sc"], sb["sc"])
    for k in ("x", "x0", "xsum"):
        assert np.array_equal(sa[k], sb[k]), k
    assert all(np.array_equal(a, b) for a, b in zip(ya, yb))


def test_rank_local_configs4_shards_through_libpdcs(P, monkeypatch):
    """configs[4]'s recipe generated rank-locally (instances.gen_mixed_shard: each
    rank draws only its rows, c from summed partials) and solved as 3 loopback
    ranks: the same iterates as the one-process instance on one context (first
    120 iterations, 1e-9), identical decisions on every rank."""
    from instances import ConicProgram, mixed_full_layout, gen_mixed_shard
    from paper_2505_00311_b200 import dist as D
    monkeypatch.setenv("PDCS_TILED", "0")
    L = mixed_full_layout(2e-4, seed=5)
    world = 3
    parts = D.partition_rows(L.row_ptr, L.rk, L.rdim, world)
    partial = [gen_mixed_shard(L, pr) for pr in parts]
    csum = sum(sh.c - L.lam for sh in partial)            # the all-reduce of the G^T y* partials
    shards = [gen_mixed_shard(L, pr, allreduce=lambda a: csum.copy()) for pr in parts]
    group = P.pdcs_loopback_create(world)
    ranks = on_all([lambda r=r: P.PdcsSolver(shards[r], rank=r, world=world, loopback=group)
                    for r in range(world)])
    whole = gen_mixed_shard(L, (0, L.m))
    one = ConicProgram(m=L.m, n=L.n, n1=L.n1, row_ptr=whole.row_ptr, col_idx=whole.col_idx, vals=whole.vals,
                       c=shards[0].c, h=whole.h, l=L.l, u=L.u, pk=L.pk, pdim=L.pdim, rk=L.rk, rdim=L.rdim)
    g0 = P.PdcsSolver(one)
    for _ in range(3):
        on_all([lambda g=g: g.iterate(40) for g in ranks])
        g0.iterate(40)
        assert_ranks_identical(ranks)
        x0, y0 = g0.get_iterate(P.CURRENT)
        its = [g.get_iterate(P.CURRENT) for g in ranks]
        assert rel(its[0][0], x0) <= TOL and rel(np.concatenate([y for _, y in its]), y0) <= TOL
    assert ranks[0].scalars()["restarts"] == g0.scalars()["restarts"]
