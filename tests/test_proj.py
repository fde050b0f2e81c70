"""Standalone multi-cone projection (pdcs_proj_*, include/pdcs.h; PAPER.md:713-780
Figs. 3-4) against the oracle's per-block projections.

Every team (the solver's size classes, and each of thread / warp / CTA /
cluster / grid forced for all SOC/RSOC blocks, the paper's thread-, block- and
grid-wise strategies) must give the oracle's P_{diag(D) K}(v) blockwise to
1e-12 relative (fp64; the GPU uses Newton where the oracle bisects to adjacent
doubles, reading P4).
"""
import numpy as np
import pytest

import oracle as O
from instances import SOC, RSOC, EXP, DUAL_EXP

TOL = 1e-12


def _blocks(rng):
    kinds, dims = [], []
    for d in (2, 3, 5, 17, 32, 33, 100, 512, 513, 600, 4096, 4097, 9000, 140000):
        kinds.append(SOC); dims.append(d)
    for d in (3, 4, 40, 700, 6000):
        kinds.append(RSOC); dims.append(d)
    for _ in range(300):
        kinds.append(EXP if rng.random() < 0.6 else DUAL_EXP); dims.append(3)
    order = rng.permutation(len(kinds))
    return np.array(kinds, np.int32)[order], np.array(dims, np.int64)[order]


def _inputs(rng, kinds, dims, scaled):
    n = int(dims.sum())
    v = rng.standard_normal(n) * 10.0 ** rng.uniform(-2, 2, size=n)
    D = rng.uniform(0.5, 2.0, size=n) if scaled else None
    off = 0
    for b, (k, d) in enumerate(zip(kinds, dims)):
        if k == RSOC and D is not None:
            D[off + 1] = D[off]                        # reading A21: equal leading divisors
        if k in (SOC, RSOC) and b % 3 == 0:            # cases (i)/(ii): inside the cone / the polar
            v[off] = (1.0 if b % 2 else -1.0) * 3.0 * np.linalg.norm(v[off + 1:off + d]) * 4.0
        off += d
    return v, D


def _oracle(kinds, dims, v, D):
    out = np.empty_like(v)
    off = 0
    for k, d in zip(kinds, dims):
        vb = v[off:off + d]
        Db = np.ones(d) if D is None else D[off:off + d]
        if k == SOC:
            out[off:off + d] = O.proj_soc_scaled(vb, Db)
        elif k == RSOC:
            out[off:off + d] = O.proj_rsoc_scaled(vb, Db)
        elif k == EXP:
            out[off:off + d] = O.proj_exp_scaled(vb, Db)
        else:
            out[off:off + d] = O.proj_dual_exp_scaled(vb, Db)
        off += d
    return out


def _blockwise_err(kinds, dims, g, o, v):
    worst, off = 0.0, 0
    for d in dims:
        e = np.max(np.abs(g[off:off + d] - o[off:off + d])) / (1.0 + np.max(np.abs(v[off:off + d])))
        worst = max(worst, e)
        off += d
    return worst


def test_proj_create_rejects_bad_blocks():
    """Argument checks run before any device work (no GPU needed)."""
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    for kinds, dims in (([SOC], [1]), ([RSOC], [2]), ([EXP], [4]), ([0], [3]), ([7], [3])):
        with pytest.raises(P.PdcsError) as e:
            P.pdcs_proj_create(kinds, dims)
        assert e.value.code == 5, e.value          # PDCS_ERR_CONE
    with pytest.raises(P.PdcsError) as e:
        P.pdcs_proj_create([SOC], [4], team=9)
    assert e.value.code == 1                        # PDCS_ERR_ARG


@pytest.mark.gpu
@pytest.mark.parametrize("scaled", [True, False])
@pytest.mark.parametrize("team", ["auto", "thread", "warp", "cta", "cluster", "grid"])
def test_proj_teams_match_oracle(team, scaled):
    import torch
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    rng = np.random.default_rng(7)
    kinds, dims = _blocks(rng)
    v, D = _inputs(rng, kinds, dims, scaled)
    ref = _oracle(kinds, dims, v, D)
    plan = P.pdcs_proj_create(kinds, dims, team=team)
    try:
        info = P.pdcs_proj_info(plan)
        nsoc = int(np.sum((kinds == SOC) | (kinds == RSOC)))
        if team != "auto":
            assert info["counts"][P._lib.TEAMS[team]] >= nsoc
        vd = torch.from_numpy(v).cuda()
        Dd = None if D is None else torch.from_numpy(D).cuda()
        out = torch.full_like(vd, float("nan"))
        P.pdcs_proj_run(plan, Dd, vd, out)
        torch.cuda.synchronize()
        g = out.cpu().numpy()
    finally:
        P.pdcs_proj_destroy(plan)
    assert np.all(np.isfinite(g))
    err = _blockwise_err(kinds, dims, g, ref, v)
    assert err <= TOL, err


@pytest.mark.gpu
def test_proj_exp_far_below_face_nearest_candidate():
    """Reading P7 on the GPU: exp / dual-exp blocks far below the cone next to
    the s = 0 face, where the candidates' squared distances tie to the ulp
    (the first block is the mixed cfg 5 case of
    test_oracle_pins.test_exp_nearest_candidate_when_distances_tie_to_the_ulp).
    The GPU must pick the oracle's (and the 60-digit reference's) point."""
    import torch
    import paper_2505_00311_b200 as P
    rng = np.random.default_rng(11)
    vs = [np.array([-53.848289446000855, 5.317878561776792, -533.0367249585])]
    Ds = [np.array([25.540130991958577, 59.559580156562696, 414.0600653716415])]
    for _ in range(200):
        Ds.append(10 ** rng.uniform(-1, 2.5, 3))
        vs.append(np.array([-rng.uniform(5, 80), rng.uniform(0.5, 8), -rng.uniform(100, 5000)]))
    kinds = np.array([EXP] * len(vs) + [DUAL_EXP] * len(vs), np.int32)
    dims = np.full(kinds.shape[0], 3, np.int64)
    v = np.concatenate(vs + [-a for a in vs])
    D = np.concatenate(Ds + [1.0 / d for d in Ds])
    plan = P.pdcs_proj_create(kinds, dims)
    out = torch.full((v.shape[0],), float("nan"), dtype=torch.float64, device="cuda")
    P.pdcs_proj_run(plan, torch.from_numpy(D).cuda(), torch.from_numpy(v).cuda(), out)
    torch.cuda.synchronize()
    P.pdcs_proj_destroy(plan)
    g = out.cpu().numpy()
    o = _oracle(kinds, dims, v, D)
    assert _blockwise_err(kinds, dims, g, o, v) <= TOL
