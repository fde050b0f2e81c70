"""Row sharding of K for 1-8 GPUs.

Rank p owns the contiguous rows [row_begin_p, row_end_p) of G.  Cuts are made
only on row-cone block boundaries (a cone block never straddles ranks, else the
library returns PDCS_ERR_SHARD) and are placed to balance nonzeros.  The primal
side is replicated on every rank.  This module holds index bookkeeping only;
all arithmetic of the method runs in libpdcs.so.
"""
from __future__ import annotations

import numpy as np


def block_boundaries(rdim) -> np.ndarray:
    """Row indices where a row-cone block starts (plus m).  Zero / NonNeg blocks
    are elementwise and may be cut anywhere, so every row inside them is a
    boundary too."""
    return np.concatenate([[0], np.cumsum(np.asarray(rdim, np.int64))])


def cut_points(rk, rdim) -> np.ndarray:
    """All admissible cut rows (sorted, including 0 and m)."""
    rk = np.asarray(rk)
    rdim = np.asarray(rdim, np.int64)
    starts = np.concatenate([[0], np.cumsum(rdim)])
    pts = [starts]
    for b in np.nonzero((rk == 0) | (rk == 1))[0]:          # Zero / NonNeg: any row
        pts.append(np.arange(starts[b], starts[b + 1], dtype=np.int64))
    return np.unique(np.concatenate(pts))


def partition_rows(row_ptr, rk, rdim, world: int):
    """[(row_begin, row_end)] per rank: admissible cuts nearest to equal nnz."""
    row_ptr = np.asarray(row_ptr, np.int64)
    m = row_ptr.shape[0] - 1
    if world <= 1:
        return [(0, m)]
    cuts = cut_points(rk, rdim)
    nnz_at = row_ptr[cuts]
    total = row_ptr[-1]
    bounds = [0]
    for p in range(1, world):
        target = total * p / world
        i = int(np.searchsorted(nnz_at, target))
        cand = [c for c in (i - 1, i) if 0 <= c < len(cuts)]
        best = min(cand, key=lambda c: abs(nnz_at[c] - target))
        bounds.append(max(int(cuts[best]), bounds[-1]))
    bounds.append(m)
    return [(bounds[p], bounds[p + 1]) for p in range(world)]


def shard(prog, row_begin: int, row_end: int):
    """Local CSR (row pointers rebased to 0) and h of rows [row_begin, row_end).
    A program generated rank-locally (instances.ShardedProgram, .rows) already
    holds exactly its rows."""
    if hasattr(prog, "rows"):
        if tuple(prog.rows) != (row_begin, row_end):
            raise ValueError(f"shard {prog.rows} holds other rows than [{row_begin}, {row_end})")
        return dict(row_ptr=np.ascontiguousarray(prog.row_ptr, np.int64), col=prog.col_idx, val=prog.vals,
                    h=np.ascontiguousarray(prog.h))
    rp = np.asarray(prog.row_ptr, np.int64)
    a, b = int(rp[row_begin]), int(rp[row_end])
    return dict(row_ptr=np.ascontiguousarray(rp[row_begin:row_end + 1] - a),
                col=np.ascontiguousarray(prog.col_idx[a:b]),
                val=np.ascontiguousarray(prog.vals[a:b]),
                h=np.ascontiguousarray(prog.h[row_begin:row_end]))
