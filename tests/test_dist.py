"""Row sharding: host-side partition logic and the sharded
decomposition of Eq. 5's products, checked on CPU with gloo (world 2) and the
oracle's SpMV; the NCCL path of libpdcs.so with a 1-rank communicator on GPU."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from instances import gen_fisher, gen_lasso, gen_mixed, gen_mpo
from paper_2505_00311_b200 import dist as D


@pytest.mark.parametrize("make", [lambda: gen_mixed(400, 50, 150, seed=3, soc_dims=(3, 40)),
                                  lambda: gen_fisher(30, 20, seed=1), lambda: gen_mpo(4, 15, seed=2),
                                  lambda: gen_lasso(200, 50, 0.2, seed=1)])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_partition_properties(make, world):
    prog = make()
    parts = D.partition_rows(prog.row_ptr, prog.rk, prog.rdim, world)
    assert len(parts) == world and parts[0][0] == 0 and parts[-1][1] == prog.m
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c and a <= b
    # no SOC/RSOC/EXP block straddles a cut
    starts = np.concatenate([[0], np.cumsum(prog.rdim)])
    for k, s, e in zip(prog.rk, starts[:-1], starts[1:]):
        if k >= 2:
            for _, b in parts[:-1]:
                assert not (s < b < e)
    # balance: every shard within max-block-nnz of the ideal share
    nnz = [prog.row_ptr[b] - prog.row_ptr[a] for a, b in parts]
    rp = prog.row_ptr
    biggest = max(rp[e] - rp[s] for s, e in zip(starts[:-1], starts[1:]))
    assert max(nnz) - prog.nnz / world <= biggest + 1


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    prog = gen_mixed(300, 40, 120, seed=7, soc_dims=(3, 30))
    parts = D.partition_rows(prog.row_ptr, prog.rk, prog.rdim, world)
    a, b = parts[rank]
    sh = D.shard(prog, a, b)
    rng = np.random.default_rng(0)
    y = rng.standard_normal(prog.m)
    x = rng.standard_normal(prog.n)
    dy = rng.standard_normal(prog.m)
    # local K^T y partial + all-reduce == full K^T y (the accept-step exchange)
    part = O.spmv_t(sh["row_ptr"], sh["col"], sh["val"], y[a:b], prog.n)
    t = torch.from_numpy(part.copy())
    dist.all_reduce(t)
    full = O.spmv_t(prog.row_ptr, prog.col_idx, prog.vals, y, prog.n)
    ok1 = np.allclose(t.numpy(), full, rtol=1e-13, atol=1e-13)
    # local rows of K x are exactly the global rows (no exchange needed)
    kx = O.spmv(sh["row_ptr"], sh["col"], sh["val"], x)
    ok2 = np.array_equal(kx, O.spmv(prog.row_ptr, prog.col_idx, prog.vals, x)[a:b])
    # line-search sums over the shards (the per-trial all-reduce of 2 scalars)
    s = torch.tensor([dy[a:b] @ dy[a:b], dy[a:b] @ kx])
    dist.all_reduce(s)
    kx_full = O.spmv(prog.row_ptr, prog.col_idx, prog.vals, x)
    ok3 = np.allclose(s.numpy(), [dy @ dy, dy @ kx_full], rtol=1e-12)
    # identical decisions: the all-reduced scalars are bitwise equal on all ranks
    g = [torch.zeros(2, dtype=s.dtype) for _ in range(world)]
    dist.all_gather(g, s)
    ok4 = all(torch.equal(g[0], gi) for gi in g)
    q.put((rank, ok1, ok2, ok3, ok4))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_sharded_products():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(all(r[1:]) for r in res), res


@pytest.mark.gpu
@pytest.mark.parametrize("tiled", ["auto", "1"])
def test_nccl_path_single_rank_matches_local(tiled, monkeypatch):
    """The row-sharded code path (NCCL all-reduces, unfused K^T + Halpern,
    pre-reduced decisions) with a 1-rank communicator reproduces the local path
    (tiled = "1": both sweeps forced through the column-tiled formats)."""
    import torch  # noqa: F401  (loads libnccl.so.2 the library reuses)
    import paper_2505_00311_b200 as P
    if tiled != "auto":
        monkeypatch.setenv("PDCS_TILED", tiled)
        monkeypatch.setenv("PDCS_TILE_KB", "1")
    prog = gen_mixed(400, 60, 200, seed=11, soc_dims=(3, 60))
    uid = P.pdcs_nccl_unique_id()
    g1 = P.PdcsSolver(prog, nccl_id=uid, rank=0, world=1)
    g0 = P.PdcsSolver(prog)
    g1.iterate(300)
    g0.iterate(300)
    x1, y1 = g1.get_iterate(P.CURRENT)
    x0, y0 = g0.get_iterate(P.CURRENT)
    d = max(np.abs(x1 - x0).max() / (1 + np.abs(x0).max()), np.abs(y1 - y0).max() / (1 + np.abs(y0).max()))
    assert d <= 1e-12, d
    assert g1.scalars()["restarts"] == g0.scalars()["restarts"]


@pytest.mark.gpu
def test_nccl_graph_path_bit_identical_to_host_loop(monkeypatch):
    """The row-sharded iteration recorded into the CUDA graph with the NCCL
    all-reduces inside (the default) gives the same bits as the host-driven
    loop (PDCS_DIST_GRAPH=0), and the graph really is used."""
    import torch  # noqa: F401
    import paper_2505_00311_b200 as P
    prog = gen_mixed(400, 60, 200, seed=12, soc_dims=(3, 60))
    out = {}
    monkeypatch.setenv("PDCS_AR_CHUNKS", "3")      # the chunked, overlapped all-reduce inside the graph
    for mode in ("1", "0"):
        monkeypatch.setenv("PDCS_DIST_GRAPH", mode)
        g = P.PdcsSolver(prog, nccl_id=P.pdcs_nccl_unique_id(), rank=0, world=1)
        g.iterate(200)
        out[mode] = (g.get_iterate(P.CURRENT), g.scalars(), P.pdcs_last_error(g.ctx))
        g.close()
    (xa, ya), sa, ea = out["1"]
    (xb, yb), sb, _ = out["0"]
    assert "graph build failed" not in ea, ea
    assert np.array_equal(xa, xb) and np.array_equal(ya, yb)
    assert sa["trials"] == sb["trials"] and sa["restarts"] == sb["restarts"]


def _shard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from instances import mixed_full_layout, gen_mixed_shard

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    L = mixed_full_layout(5e-4, seed=3)
    parts = D.partition_rows(L.row_ptr, L.rk, L.rdim, world)
    sh = gen_mixed_shard(L, parts[rank], allreduce=allreduce)
    got = [None] * world
    dist.all_gather_object(got, (sh.rows, sh.row_ptr, sh.col_idx, sh.vals, sh.h, sh.y_star, sh.c))
    q.put((rank, got if rank == 0 else None, sh.nnz))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_rank_local_mixed_generator(world):
    """BASELINE configs[4] generated rank-locally (instances.gen_mixed_shard):
    each rank draws only its rows; c = G^T y* + lam* from an all-reduce of the
    ranks' partials.  The assembled shards are the single-process instance
    (G and h bitwise, c to rounding) and the planted pair is optimal: Eq. 9 at
    (x*, y*) <= 1e-13 through the oracle, objective = c^T x*."""
    from instances import ConicProgram, mixed_full_layout, gen_mixed_shard
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    got = res[0][1]
    L = mixed_full_layout(5e-4, seed=3)
    one = gen_mixed_shard(L, (0, L.m))
    rows = [g[0] for g in got]
    assert rows[0][0] == 0 and rows[-1][1] == L.m and all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    col = np.concatenate([g[2] for g in got])
    val = np.concatenate([g[3] for g in got])
    h = np.concatenate([g[4] for g in got])
    ys = np.concatenate([g[5] for g in got])
    rp = np.concatenate([[0]] + [g[1][1:] + off for g, off in
                                 zip(got, np.cumsum([0] + [int(g[1][-1]) for g in got[:-1]]))])
    assert np.array_equal(rp, one.row_ptr) and np.array_equal(col, one.col_idx)
    assert np.array_equal(val, one.vals) and np.array_equal(h, one.h) and np.array_equal(ys, one.y_star)
    c = got[0][6]
    assert all(np.array_equal(g[6], c) for g in got)                   # every rank holds the same c
    np.testing.assert_allclose(c, one.c, rtol=1e-13, atol=1e-13 * np.abs(one.c).max())
    prog = ConicProgram(m=L.m, n=L.n, n1=L.n1, row_ptr=rp, col_idx=col, vals=val, c=c, h=h, l=L.l, u=L.u,
                        pk=L.pk, pdim=L.pdim, rk=L.rk, rdim=L.rdim)
    k = O.OracleSolver(prog, ruiz_iters=0, pock_chambolle=0).kkt_point(L.x_star, ys)
    assert max(k["err_p"], k["err_d"], k["err_gap"]) <= 1e-13, k
    assert abs(k["pobj"] - float(c @ L.x_star)) <= 1e-12 * (1 + abs(k["pobj"]))
