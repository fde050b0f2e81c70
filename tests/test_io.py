"""Instance I/O: JSON round trip, the CBF
subset reader, and its mapping onto Eq. 1 pinned by optimal values that are
known in closed form (solved by the CPU oracle here, by the CUDA path in the
gpu test)."""
import math
import os

import numpy as np
import pytest

from instances import gen_mixed, ZERO, NONNEG, SOC, RSOC, EXP
from instances.io import (from_cbf, from_json, to_json, read_instance, write_json, to_cbf_solution,
                          InstanceError, UnsupportedFeature)


def test_json_round_trip_byte_identical(tmp_path):
    prog = gen_mixed(60, 12, 40, seed=3)          # every box type incl. +-inf bounds
    assert np.isinf(prog.l).any() and np.isinf(prog.u).any()
    p1 = tmp_path / "a.json"
    write_json(prog, str(p1))
    back = read_instance(str(p1))
    p2 = tmp_path / "b.json"
    write_json(back, str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    for k in ("row_ptr", "col_idx", "vals", "c", "h", "l", "u", "pk", "pdim", "rk", "rdim"):
        assert np.array_equal(getattr(prog, k), getattr(back, k)), k


def test_json_minimal_lp_and_errors():
    txt = ('{"n1":1,"n2":0,"m":1,"c":[1.0],"h":[2.0],"l":[0.0],"u":["inf"],'
           '"primal_cones":[],"dual_cones":[{"kind":"nonneg","dim":1}],'
           '"G":{"rows":[0],"cols":[0],"vals":[1.0]}}\n')
    p = from_json(txt)
    assert to_json(p) == txt
    with pytest.raises(InstanceError, match="'psd'"):
        from_json(txt.replace('"nonneg"', '"psd"'))
    with pytest.raises(InstanceError, match="l > u"):
        from_json(txt.replace('"u":["inf"]', '"u":[-1.0]'))
    with pytest.raises(InstanceError, match="sum to"):
        from_json(txt.replace('"dim":1', '"dim":2'))
    with pytest.raises(InstanceError, match="parse error"):
        from_json(txt[:-5])


Q_CBF = """# min x1 s.t. (x1, x2, x3) in Q, x2 = 3, x3 = 4   -> x1 = 5
VER
3
OBJSENSE
MIN
VAR
3 1
Q 3
CON
2 1
L= 2
OBJACOORD
1
0 1.0
ACOORD
2
0 1 1.0
1 2 1.0
BCOORD
2
0 -3.0
1 -4.0
"""


def test_cbf_q_cone_matches_hand_built():
    p = from_cbf(Q_CBF)
    assert (p.m, p.n, p.n1) == (2, 3, 0)
    assert p.pk.tolist() == [SOC] and p.pdim.tolist() == [3]
    assert p.rk.tolist() == [ZERO] and p.rdim.tolist() == [2]
    G = p.dense()
    assert np.array_equal(G, np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]))
    assert np.array_equal(p.h, [3.0, 4.0])               # G x - h = A x + b
    assert np.array_equal(p.c, [1.0, 0.0, 0.0])
    # the same program through JSON
    assert to_json(from_json(to_json(p))) == to_json(p)


def test_cbf_unsupported_and_empty():
    with pytest.raises(InstanceError, match="empty program"):
        from_cbf("VER\n3\n")
    with pytest.raises(UnsupportedFeature, match="PSD"):
        from_cbf("VER\n3\nPSDCON\n1\n2\n")
    with pytest.raises(UnsupportedFeature, match="integer"):
        from_cbf("VER\n3\nVAR\n1 1\nF 1\nINT\n1\n0\n")
    with pytest.raises(UnsupportedFeature, match="'SVECPSD'"):
        from_cbf("VER\n3\nVAR\n3 1\nSVECPSD 3\n")
    with pytest.raises(InstanceError, match="EXP variable cone must have dim 3"):
        from_cbf("VER\n3\nVAR\n4 1\nEXP 4\n")


def _cbf(var_cones, con_cones, obj, acoord, bcoord, sense="MIN"):
    nv = sum(d for _, d in var_cones)
    nc = sum(d for _, d in con_cones)
    out = ["VER", "3", "OBJSENSE", sense, "VAR", f"{nv} {len(var_cones)}"]
    out += [f"{k} {d}" for k, d in var_cones]
    if con_cones:
        out += ["CON", f"{nc} {len(con_cones)}"] + [f"{k} {d}" for k, d in con_cones]
    out += ["OBJACOORD", str(len(obj))] + [f"{j} {v!r}" for j, v in obj]
    out += ["ACOORD", str(len(acoord))] + [f"{i} {j} {v!r}" for i, j, v in acoord]
    out += ["BCOORD", str(len(bcoord))] + [f"{i} {v!r}" for i, v in bcoord]
    return "\n".join(out) + "\n"


# (cbf text, CBF objective at the optimum, optimal x in CBF order or None).
# Each optimum is a closed form of the cone's definition, so a wrong
# orientation / sign / permutation in the mapping changes the answer.
CASES = {
    # EXP: x1 >= x2 exp(x3 / x2) with x2 = 1, x3 = 1 -> min x1 = e
    "exp_var": (_cbf([("EXP", 3)], [("L=", 2)], [(0, 1.0)], [(0, 1, 1.0), (1, 2, 1.0)],
                     [(0, -1.0), (1, -1.0)]), math.e, [math.e, 1.0, 1.0]),
    # EXP constraint on (z, 2, 0.5) with z free: z >= 2 exp(0.25)
    "exp_con": (_cbf([("F", 1)], [("EXP", 3)], [(0, 1.0)], [(0, 0, 1.0)], [(1, 2.0), (2, 0.5)]),
                2.0 * math.exp(0.25), None),
    # QR: 2 x1 x2 >= x3^2 with x2 = 1, x3 = 2 -> min x1 = 2
    "qr_var": (_cbf([("QR", 3)], [("L=", 2)], [(0, 1.0)], [(0, 1, 1.0), (1, 2, 1.0)],
                    [(0, -1.0), (1, -2.0)]), 2.0, [2.0, 1.0, 2.0]),
    # MAX x1 + x2 s.t. x1 - 3 <= 0 (L- row), x2 in [0, inf) with x1 + 2 x2 <= 7: 3 + 2 = 5
    "max_lminus": (_cbf([("F", 1), ("L+", 1)], [("L-", 1), ("L+", 1)], [(0, 1.0), (1, 1.0)],
                        [(0, 0, 1.0), (1, 0, -1.0), (1, 1, -2.0)], [(0, -3.0), (1, 7.0)], sense="MAX"),
                   5.0, [3.0, 2.0]),
    # Q with a free row block dropped: min x1, (x1, x2, x3) in Q, x2 = 3, x3 = 4 -> 5
    "q_free_row": (_cbf([("Q", 3)], [("F", 1), ("L=", 2)], [(0, 1.0)],
                        [(0, 0, 5.0), (1, 1, 1.0), (2, 2, 1.0)], [(1, -3.0), (2, -4.0)]), 5.0,
                   [5.0, 3.0, 4.0]),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_cbf_mapping_closed_form_optima_oracle(name):
    import oracle as O
    text, opt, xstar = CASES[name]
    p = from_cbf(text, name)
    o = O.OracleSolver(p, tol=1e-9, max_iters=200000)
    r = o.solve()
    assert r.status == 0, name
    obj = p.obj_sign * (r.kkt.pobj + p.obj_const)
    assert abs(obj - opt) <= 1e-6 * (1 + abs(opt)), (name, obj, opt)
    if xstar is not None:
        x, _ = o.get_iterate(3, 1)                # best point, original space
        assert np.allclose(to_cbf_solution(p, x), xstar, atol=1e-5), (name, to_cbf_solution(p, x))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_cbf_mapping_closed_form_optima_gpu(name):
    from paper_2505_00311_b200 import build
    build.build()
    import paper_2505_00311_b200 as P
    text, opt, xstar = CASES[name]
    p = from_cbf(text, name)
    g = P.PdcsSolver(p, tol=1e-9, max_iters=200000)
    r = g.solve()
    assert r["status"] == "OPTIMAL", (name, r)
    obj = p.obj_sign * (r["pobj"] + p.obj_const)
    assert abs(obj - opt) <= 1e-6 * (1 + abs(opt)), (name, obj, opt)
    if xstar is not None:
        x, _ = g.get_iterate(P.BEST, P.ORIGINAL)
        assert np.allclose(to_cbf_solution(p, x), xstar, atol=1e-5), (name, to_cbf_solution(p, x))
