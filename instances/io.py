"""Instance I/O: the JSON instance file and a CBF subset reader.

Host-side plumbing only (no arithmetic of the method): external conic programs
are turned into a ``ConicProgram`` that feeds the C ABI (``PdcsSolver``) or the
oracle.  Formats follow SPEC.md:595-622:

* JSON (``write_json`` / ``read_json``): ``{n1, n2, m, c, h, l, u,
  primal_cones: [{kind, dim}], dual_cones: [{kind, dim}], G: {rows, cols,
  vals}}``.  ``dual_cones`` is the row-cone list C_b (``G x - h in C_b``,
  reading A1).  Floats are written with ``repr`` (shortest round-trip decimal);
  +-inf bounds as the strings "inf" / "-inf".  write -> read -> write is
  byte-identical.
* CBF subset (``read_cbf``): records VER, OBJSENSE, VAR, CON,
  OBJACOORD, OBJBCOORD, ACOORD, BCOORD with cones F, L+, L-, L=, Q, QR, EXP.
  Integer and PSD/power-cone records raise ``UnsupportedFeature`` (never a
  silent skip).  A CBF problem  min c^T x + c0  s.t.  A x + b in K_con,
  x in K_var  maps to Eq. 1 as:

    - variables: F / L+ / L- / L= become box coordinates [l, u] =
      (-inf, inf) / [0, inf) / (-inf, 0] / [0, 0] and are moved to the front
      (x_1, n1 of them); Q / QR / EXP blocks become primal cones (x_2) in file
      order.  ``prog.var_perm[j]`` is the CBF index of our coordinate j.
    - constraints: G = A, h = -b, so G x - h = A x + b in C_b.  L= -> Zero,
      L+ -> NonNeg, L- -> NonNeg with the rows negated, Q -> SOC, QR -> RSOC,
      EXP -> Exp; F rows constrain nothing and are dropped.
    - CBF's EXP cone is {(x1, x2, x3): x1 >= x2 exp(x3 / x2), x2 > 0}; ours
      (Eq. 12) is {(r, s, t): t >= s exp(r / s), s > 0}, so a
      block is stored reversed: (r, s, t) = (x3, x2, x1).
    - QR is {(x1, x2, z): 2 x1 x2 >= ||z||^2, x1, x2 >= 0}, the same as our
      RSOC (reading A22).
    - OBJSENSE MAX negates c (and the constant); ``prog.obj_const`` holds c0
      and ``prog.obj_sign`` the sense, so the CBF objective is
      obj_sign * (c^T x + obj_const).
"""
from __future__ import annotations

import json
import math

import numpy as np

from .program import ConicProgram, ZERO, NONNEG, SOC, RSOC, EXP, DUAL_EXP, KIND_NAMES, csr_from_coo

KIND_BY_NAME = {v: k for k, v in KIND_NAMES.items()}


class InstanceError(ValueError):
    """Parse or validation error (with line / element context)."""


class UnsupportedFeature(InstanceError):
    """A CBF record or cone outside the supported subset."""


# ------------------------------------------------------------------ validation
def validate(prog: ConicProgram) -> None:
    """Collect every violation and raise one InstanceError."""
    errs = []
    if prog.m < 0 or prog.n < 0 or not 0 <= prog.n1 <= prog.n:
        errs.append(f"bad sizes m={prog.m} n={prog.n} n1={prog.n1}")
    if prog.row_ptr.shape != (prog.m + 1,) or prog.row_ptr[0] != 0 or np.any(np.diff(prog.row_ptr) < 0):
        errs.append("row_ptr is not a CSR row pointer of length m+1")
    nnz = int(prog.row_ptr[-1]) if prog.row_ptr.size else 0
    if prog.col_idx.shape != (nnz,) or prog.vals.shape != (nnz,):
        errs.append("col_idx / vals length != nnz")
    elif nnz and (prog.col_idx.min() < 0 or prog.col_idx.max() >= prog.n):
        errs.append("column index out of range")
    for name, arr, ln in (("c", prog.c, prog.n), ("h", prog.h, prog.m), ("l", prog.l, prog.n1),
                          ("u", prog.u, prog.n1)):
        if arr.shape != (ln,):
            errs.append(f"{name} has length {arr.shape[0]}, expected {ln}")
    for name, arr in (("c", prog.c), ("h", prog.h), ("G", prog.vals)):
        if not np.all(np.isfinite(arr)):
            errs.append(f"{name} has non-finite entries")
    if prog.l.shape == prog.u.shape:
        bad = np.nonzero(prog.l > prog.u)[0]
        if bad.size:
            errs.append(f"l > u at {bad[:5].tolist()}")
        if np.any(np.isnan(prog.l)) or np.any(np.isnan(prog.u)) or np.any(prog.l == np.inf) \
                or np.any(prog.u == -np.inf):
            errs.append("bounds contain NaN, l = +inf or u = -inf")
    for side, kinds, dims, total in (("primal", prog.pk, prog.pdim, prog.n - prog.n1),
                                     ("row", prog.rk, prog.rdim, prog.m)):
        for b, (k, d) in enumerate(zip(kinds.tolist(), dims.tolist())):
            mind = {ZERO: 1, NONNEG: 1, SOC: 2, RSOC: 3, EXP: 3, DUAL_EXP: 3}.get(k)
            if mind is None:
                errs.append(f"{side} cone {b}: unknown kind {k}")
            elif d < mind or (k in (EXP, DUAL_EXP) and d != 3):
                errs.append(f"{side} cone {b}: bad dim {d} for {KIND_NAMES[k]}")
        if int(np.sum(dims)) != total:
            errs.append(f"{side} cone dims sum to {int(np.sum(dims))}, expected {total}")
    if errs:
        raise InstanceError("; ".join(errs))


# ------------------------------------------------------------------ JSON
def _num(v: float):
    v = float(v)
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return v


def _fromnum(v, where: str) -> float:
    if isinstance(v, str):
        if v in ("inf", "-inf"):
            return math.inf if v == "inf" else -math.inf
        raise InstanceError(f"{where}: bad number {v!r}")
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise InstanceError(f"{where}: bad number {v!r}")
    return float(v)


def to_json(prog: ConicProgram) -> str:
    rows = np.repeat(np.arange(prog.m, dtype=np.int64), np.diff(prog.row_ptr))
    doc = {
        "n1": int(prog.n1), "n2": int(prog.n - prog.n1), "m": int(prog.m),
        "c": [_num(v) for v in prog.c], "h": [_num(v) for v in prog.h],
        "l": [_num(v) for v in prog.l], "u": [_num(v) for v in prog.u],
        "primal_cones": [{"kind": KIND_NAMES[int(k)], "dim": int(d)} for k, d in zip(prog.pk, prog.pdim)],
        "dual_cones": [{"kind": KIND_NAMES[int(k)], "dim": int(d)} for k, d in zip(prog.rk, prog.rdim)],
        "G": {"rows": rows.tolist(), "cols": prog.col_idx.astype(np.int64).tolist(),
              "vals": [_num(v) for v in prog.vals]},
    }
    return json.dumps(doc, separators=(",", ":"), allow_nan=False) + "\n"


def write_json(prog: ConicProgram, path: str) -> None:
    with open(path, "w") as f:
        f.write(to_json(prog))


def from_json(text: str, name: str = "json") -> ConicProgram:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise InstanceError(f"{name}: JSON parse error at line {e.lineno} col {e.colno}: {e.msg}") from None
    if not isinstance(doc, dict):
        raise InstanceError(f"{name}: top level must be an object")
    for key in ("n1", "n2", "m", "c", "h", "l", "u", "primal_cones", "dual_cones", "G"):
        if key not in doc:
            raise InstanceError(f"{name}: missing key {key!r}")
    n1, n2, m = int(doc["n1"]), int(doc["n2"]), int(doc["m"])
    n = n1 + n2

    def vec(key):
        v = doc[key]
        if not isinstance(v, list):
            raise InstanceError(f"{name}: {key} must be a list")
        return np.array([_fromnum(x, f"{name}: {key}[{i}]") for i, x in enumerate(v)], dtype=np.float64)

    def cones(key):
        kinds, dims = [], []
        for i, blk in enumerate(doc[key]):
            kname = blk.get("kind") if isinstance(blk, dict) else None
            if kname not in KIND_BY_NAME:
                raise InstanceError(f"{name}: {key}[{i}]: unknown cone kind {kname!r}")
            kinds.append(KIND_BY_NAME[kname])
            dims.append(int(blk.get("dim", -1)))
        return np.array(kinds, np.int32), np.array(dims, np.int64)

    G = doc["G"]
    rows = np.asarray(G.get("rows", []), dtype=np.int64)
    cols = np.asarray(G.get("cols", []), dtype=np.int64)
    vals = np.array([_fromnum(x, f"{name}: G.vals[{i}]") for i, x in enumerate(G.get("vals", []))],
                    dtype=np.float64)
    if not rows.shape == cols.shape == vals.shape:
        raise InstanceError(f"{name}: G.rows / cols / vals lengths differ")
    if rows.size and (rows.min() < 0 or rows.max() >= m or cols.min() < 0 or cols.max() >= n):
        raise InstanceError(f"{name}: G index out of range")
    pk, pdim = cones("primal_cones")
    rk, rdim = cones("dual_cones")
    row_ptr, col_idx, v = _merge_dups(m, n, rows, cols, vals)
    prog = ConicProgram(m=m, n=n, n1=n1, row_ptr=row_ptr, col_idx=col_idx, vals=v, c=vec("c"),
                        h=vec("h"), l=vec("l"), u=vec("u"), pk=pk, pdim=pdim, rk=rk, rdim=rdim,
                        name=name)
    validate(prog)
    return prog


def read_json(path: str) -> ConicProgram:
    with open(path) as f:
        return from_json(f.read(), name=path)


# ------------------------------------------------------------------ CBF subset
_VAR_BOX = {"F": (-math.inf, math.inf), "L+": (0.0, math.inf), "L-": (-math.inf, 0.0), "L=": (0.0, 0.0)}
_CONE = {"Q": SOC, "QR": RSOC, "EXP": EXP}
_ROW = {"L=": ZERO, "L+": NONNEG, "L-": NONNEG, "Q": SOC, "QR": RSOC, "EXP": EXP}
_UNSUPPORTED = {"INT": "integer variables (relaxed upstream, not here; PAPER.md §5.1)",
                "PSDVAR": "PSD variables (SDP cones are out of scope, PAPER.md:492)",
                "PSDCON": "PSD constraints (SDP cones are out of scope, PAPER.md:492)",
                "OBJFCOORD": "PSD objective coordinates", "FCOORD": "PSD constraint coordinates",
                "HCOORD": "PSD constraint coordinates", "DCOORD": "PSD constraint coordinates",
                "POWCONES": "power cones", "POW*CONES": "dual power cones"}


def _merge_dups(m, n, rows, cols, vals):
    """CSR with duplicate (row, col) entries summed (the C ABI needs strictly
    increasing column ids within a row)."""
    rows = np.asarray(rows, np.int64); cols = np.asarray(cols, np.int64)
    key = rows * max(n, 1) + cols
    uk, inv = np.unique(key, return_inverse=True)
    v = np.zeros(uk.shape[0]); np.add.at(v, inv, np.asarray(vals, np.float64))
    return csr_from_coo(m, n, uk // max(n, 1), uk % max(n, 1), v)


def _cbf_lines(text: str):
    for ln, raw in enumerate(text.splitlines(), 1):
        s = raw.strip()
        if s and not s.startswith("#"):
            yield ln, s


def from_cbf(text: str, name: str = "cbf") -> ConicProgram:
    it = iter(_cbf_lines(text))

    def nxt(what):
        try:
            return next(it)
        except StopIteration:
            raise InstanceError(f"{name}: unexpected end of file while reading {what}") from None

    def ints(ln, s, k, what):
        p = s.split()
        if len(p) != k:
            raise InstanceError(f"{name}:{ln}: {what}: expected {k} fields, got {s!r}")
        try:
            return [int(x) for x in p]
        except ValueError:
            raise InstanceError(f"{name}:{ln}: {what}: bad integer in {s!r}") from None

    def cone_list(ln, s, what, table):
        total, k = ints(ln, s, 2, what)
        out = []
        for _ in range(k):
            ln2, s2 = nxt(what)
            p = s2.split()
            if len(p) != 2:
                raise InstanceError(f"{name}:{ln2}: {what}: expected 'CONE dim', got {s2!r}")
            if p[0] not in table:
                raise UnsupportedFeature(f"{name}:{ln2}: unsupported cone {p[0]!r} in {what}")
            out.append((p[0], int(p[1])))
        if sum(d for _, d in out) != total:
            raise InstanceError(f"{name}:{ln}: {what} cone dims sum to {sum(d for _, d in out)}, not {total}")
        return total, out

    nvar = ncon = None
    var_cones = con_cones = None
    sense = 1.0
    obj = {}
    c0 = 0.0
    acoo = ([], [], [])
    bvec = {}
    seen_ver = False
    for ln, rec in it:
        key = rec.split()[0]
        if key in _UNSUPPORTED:
            raise UnsupportedFeature(f"{name}:{ln}: unsupported record {key}: {_UNSUPPORTED[key]}")
        if key == "VER":
            nxt("VER")
            seen_ver = True
        elif key == "OBJSENSE":
            ln2, s = nxt("OBJSENSE")
            if s not in ("MIN", "MAX"):
                raise InstanceError(f"{name}:{ln2}: OBJSENSE must be MIN or MAX, got {s!r}")
            sense = 1.0 if s == "MIN" else -1.0
        elif key == "VAR":
            ln2, s = nxt("VAR")
            nvar, var_cones = cone_list(ln2, s, "VAR", {**_VAR_BOX, **_CONE})
        elif key == "CON":
            ln2, s = nxt("CON")
            ncon, con_cones = cone_list(ln2, s, "CON", {**_ROW, "F": None})
        elif key in ("OBJACOORD", "ACOORD", "BCOORD"):
            ln2, s = nxt(key)
            (cnt,) = ints(ln2, s, 1, key)
            for _ in range(cnt):
                ln3, s3 = nxt(key)
                p = s3.split()
                want = {"OBJACOORD": 2, "ACOORD": 3, "BCOORD": 2}[key]
                if len(p) != want:
                    raise InstanceError(f"{name}:{ln3}: {key}: expected {want} fields, got {s3!r}")
                try:
                    idx = [int(x) for x in p[:-1]]
                    val = float(p[-1])
                except ValueError:
                    raise InstanceError(f"{name}:{ln3}: {key}: bad entry {s3!r}") from None
                if key == "OBJACOORD":
                    obj[idx[0]] = obj.get(idx[0], 0.0) + val
                elif key == "ACOORD":
                    acoo[0].append(idx[0]); acoo[1].append(idx[1]); acoo[2].append(val)
                else:
                    bvec[idx[0]] = bvec.get(idx[0], 0.0) + val
        elif key == "OBJBCOORD":
            ln2, s = nxt("OBJBCOORD")
            c0 = float(s)
        else:
            raise UnsupportedFeature(f"{name}:{ln}: unsupported record {key}")
    if not seen_ver:
        raise InstanceError(f"{name}: missing VER record")
    if not nvar:
        raise InstanceError(f"{name}: empty program (no VAR record or zero variables)")
    if con_cones is None:
        ncon, con_cones = 0, []

    # variable permutation: box coordinates first, then cone blocks in file order
    box_idx, box_l, box_u, cone_idx, pk, pdim = [], [], [], [], [], []
    j = 0
    for cn, d in var_cones:
        ids = list(range(j, j + d))
        if cn in _VAR_BOX:
            lo, hi = _VAR_BOX[cn]
            box_idx += ids; box_l += [lo] * d; box_u += [hi] * d
        else:
            if cn == "EXP":
                if d != 3:
                    raise InstanceError(f"{name}: EXP variable cone must have dim 3, got {d}")
                ids = ids[::-1]                      # (r, s, t) = (x3, x2, x1)
            cone_idx += ids; pk.append(_CONE[cn]); pdim.append(d)
        j += d
    var_perm = np.array(box_idx + cone_idx, dtype=np.int64)       # ours j -> CBF var_perm[j]
    newpos = np.empty(nvar, np.int64)
    newpos[var_perm] = np.arange(nvar)

    # rows: drop F, negate L-, reverse EXP blocks
    row_map, row_sign, rk, rdim = [], [], [], []
    i = 0
    for cn, d in con_cones:
        ids = list(range(i, i + d))
        if cn != "F":
            if cn == "EXP":
                if d != 3:
                    raise InstanceError(f"{name}: EXP constraint cone must have dim 3, got {d}")
                ids = ids[::-1]
            row_map += ids; row_sign += [-1.0 if cn == "L-" else 1.0] * d
            rk.append(_ROW[cn]); rdim.append(d)
        i += d
    m = len(row_map)
    newrow = np.full(max(ncon, 1), -1, np.int64)
    newrow[np.array(row_map, np.int64)] = np.arange(m)
    sign = np.array(row_sign, np.float64)

    ai = np.array(acoo[0], np.int64); aj = np.array(acoo[1], np.int64); av = np.array(acoo[2], np.float64)
    if ai.size and (ai.min() < 0 or ai.max() >= ncon or aj.min() < 0 or aj.max() >= nvar):
        raise InstanceError(f"{name}: ACOORD index out of range")
    keep = newrow[ai] >= 0 if ai.size else np.zeros(0, bool)
    r = newrow[ai[keep]]
    row_ptr, col_idx, vals = _merge_dups(m, nvar, r, newpos[aj[keep]], av[keep] * sign[r])
    h = np.zeros(m)
    for bi, bv in bvec.items():
        if not 0 <= bi < ncon:
            raise InstanceError(f"{name}: BCOORD index {bi} out of range")
        if newrow[bi] >= 0:
            h[newrow[bi]] -= bv * sign[newrow[bi]]               # G x - h = A x + b
    c = np.zeros(nvar)
    for vj, cv in obj.items():
        if not 0 <= vj < nvar:
            raise InstanceError(f"{name}: OBJACOORD index {vj} out of range")
        c[newpos[vj]] += sense * cv
    prog = ConicProgram(m=m, n=nvar, n1=len(box_idx), row_ptr=row_ptr, col_idx=col_idx, vals=vals,
                        c=c, h=h, l=np.array(box_l, np.float64), u=np.array(box_u, np.float64),
                        pk=np.array(pk, np.int32), pdim=np.array(pdim, np.int64),
                        rk=np.array(rk, np.int32), rdim=np.array(rdim, np.int64), name=name)
    prog.var_perm = var_perm
    prog.obj_const = sense * c0
    prog.obj_sign = sense
    validate(prog)
    return prog


def read_cbf(path: str) -> ConicProgram:
    with open(path) as f:
        return from_cbf(f.read(), name=path)


def read_instance(path: str) -> ConicProgram:
    """JSON or CBF by extension."""
    if path.lower().endswith(".cbf"):
        return read_cbf(path)
    return read_json(path)


def to_cbf_solution(prog: ConicProgram, x: np.ndarray) -> np.ndarray:
    """Our x (original space) back in the CBF variable order."""
    out = np.empty(prog.n)
    out[prog.var_perm] = x
    return out
