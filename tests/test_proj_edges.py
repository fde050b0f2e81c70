"""Edge cases of the cone projections on the DEVICE (-m gpu), against the oracle.

The oracle pins these cases on the CPU (tests/test_oracle_pins.py); here the
CUDA kernels get the same inputs through pdcs_proj_run (every team: the
solver's size classes and each forced team) and must match the oracle's
P_{diag(D) K}(v) blockwise to 1e-12:
  * SOC case (iii) t == 0 exactly (Thm 1), x != 0;
  * |t| = 1e-13 ||x|| and 1e-300 (reading A16, the mu-form regression);
  * v = 0, and v = (t, 0) with t > 0 / t < 0 (x = 0 blocks);
  * the exp point of SPEC.md:197 (a3 = a4, the pole surface of h; reading A25);
  * exp points on the s = 0 face, with r / t of either sign, and far out in
    the bracket-expansion branches (a3 << 0, a4 >> 1; reading P2);
  * divisors spread over 10^[-4, 4] (d-hat far from 1).
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from instances import SOC, RSOC, EXP, DUAL_EXP

pytestmark = pytest.mark.gpu
TOL = 1e-12
HERE = os.path.dirname(os.path.abspath(__file__))


def _soc_cases(rng):
    vs, Ds = [], []
    for d in (3, 17, 40, 700, 5000):        # thread, warp, CTA classes
        for t in (0.0, 1e-13, -1e-13, 1e-300, -1e-300):
            x = rng.standard_normal(d - 1) * 10.0 ** rng.uniform(-2, 2, d - 1)
            tt = t * np.linalg.norm(x) if abs(t) > 1e-200 else t
            vs.append(np.concatenate([[tt], x]))
            Ds.append(10.0 ** rng.uniform(-4, 4, d))
        for t in (0.0, 2.0, -2.0):          # x = 0 blocks
            vs.append(np.concatenate([[t], np.zeros(d - 1)]))
            Ds.append(10.0 ** rng.uniform(-4, 4, d))
    return vs, Ds


def _exp_cases(rng):
    G = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))
    e = G["exp_degenerate"][0]
    vs = [np.array(e["v"], float)]
    Ds = [np.array(e["d"], float)]
    for r0 in (-3.0, 0.0, 2.0):             # s = 0 face
        for t0 in (-1.5, 0.0, 4.0):
            vs.append(np.array([r0, 0.0, t0])); Ds.append(np.ones(3))
            vs.append(np.array([r0, 0.0, t0])); Ds.append(10.0 ** rng.uniform(-4, 4, 3))
    for _ in range(40):                     # far expansion branches
        vs.append(np.array([-10.0 ** rng.uniform(1, 3), rng.uniform(1e-3, 1.0), rng.uniform(-1, 1)]))
        Ds.append(10.0 ** rng.uniform(-2, 2, 3))
        vs.append(np.array([10.0 ** rng.uniform(0.5, 2), rng.uniform(1e-3, 1.0), rng.uniform(0, 5)]))
        Ds.append(10.0 ** rng.uniform(-2, 2, 3))
        vs.append(rng.standard_normal(3) * 10.0 ** rng.uniform(-3, 3))
        Ds.append(10.0 ** rng.uniform(-4, 4, 3))
    vs.append(np.zeros(3)); Ds.append(np.ones(3))
    return vs, Ds


def _oracle(kinds, dims, v, D):
    out = np.empty_like(v)
    off = 0
    f = {SOC: O.proj_soc_scaled, RSOC: O.proj_rsoc_scaled, EXP: O.proj_exp_scaled,
         DUAL_EXP: O.proj_dual_exp_scaled}
    for k, d in zip(kinds, dims):
        out[off:off + d] = f[k](v[off:off + d], D[off:off + d])
        off += d
    return out


@pytest.mark.parametrize("team", ["auto", "thread", "warp", "cta", "cluster", "grid"])
def test_projection_edge_cases_match_oracle(team):
    import torch
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    rng = np.random.default_rng(5)
    sv, sD = _soc_cases(rng)
    ev, eD = _exp_cases(rng)
    kinds = [SOC] * len(sv) + [EXP] * len(ev) + [DUAL_EXP] * len(ev)
    vs = sv + ev + [-v for v in ev]
    Ds = sD + eD + [1.0 / d for d in eD]
    dims = np.array([len(v) for v in vs], np.int64)
    kinds = np.array(kinds, np.int32)
    v = np.concatenate(vs)
    D = np.concatenate(Ds)
    ref = _oracle(kinds, dims, v, D)
    plan = P.pdcs_proj_create(kinds, dims, team=team)
    try:
        out = torch.full((v.shape[0],), float("nan"), dtype=torch.float64, device="cuda")
        P.pdcs_proj_run(plan, torch.from_numpy(D).cuda(), torch.from_numpy(v).cuda(), out)
        torch.cuda.synchronize()
        g = out.cpu().numpy()
    finally:
        P.pdcs_proj_destroy(plan)
    assert np.all(np.isfinite(g))
    off, worst, where = 0, 0.0, None
    for b, d in enumerate(dims):
        e = np.max(np.abs(g[off:off + d] - ref[off:off + d])) / (1.0 + np.max(np.abs(v[off:off + d])))
        if e > worst:
            worst, where = e, (b, int(kinds[b]), int(d), v[off:off + min(d, 3)])
        off += d
    assert worst <= TOL, (worst, where)
