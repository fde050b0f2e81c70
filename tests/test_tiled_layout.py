"""Host-side tests of the column-tiled SpMV layout builder,
through the host-only diagnostic pdcs_tiled_layout_stats (no GPU needed).

The builder decides which entries are staged through shared-memory tiles,
packs them into zero-padded quads, sorts each segment's rows by length and
permutes entries inside rows to balance shared-memory banks.  None of that may
lose, duplicate or relabel an entry (structure_errors == 0), the result must
not depend on the number of host build threads, and the bank balancing must
lower the modeled wavefront count without going below its lower bound.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from paper_2505_00311_b200 import _lib
from instances import gen_lasso, gen_mpo, gen_fisher


def _csr(prog):
    K = sp.csr_matrix((prog.vals, prog.col_idx, prog.row_ptr), shape=(prog.m, prog.n))
    KT = K.T.tocsr()
    KT.sort_indices()
    return K, KT


def _stats(A, nvec, elem):
    return _lib.pdcs_tiled_layout_stats(A.indptr.astype(np.int64), A.indices.astype(np.int32), nvec, elem)


def _random_csr(rng, rows, cols, row_len):
    ptr = [0]
    idx = []
    for _ in range(rows):
        k = int(rng.integers(row_len[0], row_len[1] + 1))
        c = np.sort(rng.choice(cols, size=min(k, cols), replace=False))
        idx.append(c)
        ptr.append(ptr[-1] + len(c))
    idx = np.concatenate(idx) if idx else np.zeros(0, np.int64)
    return sp.csr_matrix((np.ones(len(idx)), idx, ptr), shape=(rows, cols))


@pytest.mark.parametrize("kb", ["1", "4", "32"])
def test_layout_structure_lasso(monkeypatch, kb):
    monkeypatch.setenv("PDCS_TILE_KB", kb)
    prog = gen_lasso(6000, 700, 0.03, seed=2)
    K, KT = _csr(prog)
    for A, nvec, elem in [(K, prog.n, 2), (KT, prog.m, 1)]:
        st = _stats(A, nvec, elem)
        assert st["nnz"] == A.nnz
        assert st["structure_errors"] == 0
        assert st["quads"] * 4 == st["staged"] + st["pads"]
        assert st["lds_wavefronts"] >= st["lds_wavefront_bound"] - 1e-9


def test_layout_structure_ragged_and_degenerate(monkeypatch):
    """Ragged rows (0 .. 300 entries), empty rows, a single row, a single column."""
    monkeypatch.setenv("PDCS_TILE_KB", "1")
    rng = np.random.default_rng(5)
    cases = [_random_csr(rng, 3000, 900, (0, 300)), _random_csr(rng, 1, 5000, (4000, 4000)),
             _random_csr(rng, 2500, 1, (0, 1)), _random_csr(rng, 1500, 3000, (0, 0))]
    for A in cases:
        for elem, nvec in [(2, A.shape[1]), (1, A.shape[1])]:
            st = _stats(A, nvec, elem)
            assert st["nnz"] == A.nnz and st["structure_errors"] == 0


def test_layout_other_configs(monkeypatch):
    monkeypatch.setenv("PDCS_TILE_KB", "4")
    for prog in [gen_mpo(4, 60, seed=1), gen_fisher(300, 40, 0.2, seed=1)]:
        K, KT = _csr(prog)
        assert _stats(K, prog.n, 2)["structure_errors"] == 0
        assert _stats(KT, prog.m, 1)["structure_errors"] == 0


def test_layout_independent_of_build_threads(monkeypatch):
    monkeypatch.setenv("PDCS_TILE_KB", "2")
    prog = gen_lasso(9000, 500, 0.04, seed=3)
    K, _ = _csr(prog)
    out = []
    for nth in ["1", "3", "8"]:
        monkeypatch.setenv("PDCS_BUILD_THREADS", nth)
        st = _stats(K, prog.n, 2)
        st.pop("build_ms")
        out.append(st)
    assert out[0] == out[1] == out[2]


def test_bank_balancing_lowers_wavefronts(monkeypatch):
    """The model charges each 8-lane (pairs) / 16-lane (doubles) phase the
    largest number of distinct addresses in one bank group (tools/lds_probe.cu
    measured this rule on B200).  Balancing must beat the unbalanced layout and
    come within 30% of the per-phase lower bound."""
    prog = gen_lasso(20000, 10000, 0.01, seed=0)
    K, KT = _csr(prog)
    for A, nvec, elem in [(K, prog.n, 2), (KT, prog.m, 1)]:
        monkeypatch.setenv("PDCS_TILE_BALANCE", "0")
        raw = _stats(A, nvec, elem)
        monkeypatch.setenv("PDCS_TILE_BALANCE", "1")
        bal = _stats(A, nvec, elem)
        assert raw["structure_errors"] == 0 and bal["structure_errors"] == 0
        assert bal["lds_wavefronts"] < 0.85 * raw["lds_wavefronts"], (raw, bal)
        assert bal["lds_wavefronts"] <= 1.3 * bal["lds_wavefront_bound"], bal


def test_parts_mode_build_matches_concatenated(monkeypatch):
    """The solver's builds keep the per-thread parts and upload them at their
    offsets (pdcs_tiled_build_host times that mode); the staged-entry count
    must equal the concatenated layout's for any thread count."""
    prog = gen_lasso(9000, 600, 0.03, seed=5)
    K, KT = _csr(prog)
    for A, nvec, elem in [(K, prog.n, 2), (KT, prog.m, 1)]:
        ref = _stats(A, nvec, elem)
        for th in ("1", "3", "8"):
            monkeypatch.setenv("PDCS_BUILD_THREADS", th)
            b = _lib.pdcs_tiled_build_host(A.indptr.astype(np.int64), A.indices.astype(np.int32),
                                           A.shape[0], nvec, elem)
            assert b["staged"] == ref["staged"] and b["build_ms"] >= b["ranges_ms"] >= 0.0
    with pytest.raises(ValueError):
        _lib.pdcs_tiled_build_host(K.indptr.astype(np.int64), K.indices.astype(np.int32), K.shape[0], 0, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("kb,elem,which", [("1", 2, "K"), ("2", 1, "KT"), ("32", 2, "K"), ("32", 1, "KT"),
                                           ("4", 2, "rand"), ("4", 1, "rand")])
def test_device_balanced_build_is_bit_identical(monkeypatch, kb, elem, which):
    """The solver's deferred build (host structure; shared-memory bank balancing
    and the sliced re-layout on the device, tiled.cuh k_tile_balance /
    k_tile_slice) gives the all-host build's layout entry for entry: column
    ids, value permutation, row pointers, block bases, segment descriptors
    (pdcs_tiled_device_check), with 1 and 5 host build threads."""
    monkeypatch.setenv("PDCS_TILE_KB", kb)
    if which == "rand":
        A = _random_csr(np.random.default_rng(4), 3000, 9000, (1, 300))
        nvec = 9000
    else:
        K, KT = _csr(gen_lasso(3000, 300, 0.2, seed=6))
        A = K if which == "K" else KT
        nvec = A.shape[1]
    for threads in ("1", "5"):
        monkeypatch.setenv("PDCS_BUILD_THREADS", threads)
        r = _lib.pdcs_tiled_device_check(A.indptr.astype(np.int64), A.indices.astype(np.int32), A.shape[0],
                                         nvec, elem)
        assert r["mismatches"] == 0 and r["entries"] > 0, r


def _banded_csr(rng, rows, cols, row_len, band):
    """Rows whose columns cluster in a band (staged tiles) plus a few random
    far columns (direct entries), with empty rows sprinkled in."""
    ptr = [0]
    idx = []
    for r in range(rows):
        k = 0 if r % 97 == 5 else int(rng.integers(row_len[0], row_len[1] + 1))
        lo = (r * 7) % max(1, cols - band)
        near = rng.choice(band, size=min(k, band), replace=False) + lo
        far = rng.choice(cols, size=int(rng.integers(0, 4)), replace=False) if k else np.zeros(0, np.int64)
        c = np.unique(np.concatenate([near, far]).astype(np.int64))
        idx.append(c)
        ptr.append(ptr[-1] + len(c))
    idx = np.concatenate(idx)
    return sp.csr_matrix((np.ones(len(idx)), idx, ptr), shape=(rows, cols))


@pytest.mark.gpu
@pytest.mark.parametrize("kb,elem,which", [("1", 2, "K"), ("2", 1, "KT"), ("32", 2, "K"), ("32", 1, "KT"),
                                           ("4", 2, "rand"), ("4", 1, "rand"), ("2", 2, "band"),
                                           ("1", 1, "band"), ("32", 2, "mpoK"), ("32", 1, "fisherKT")])
def test_device_structure_build_is_bit_identical(monkeypatch, kb, elem, which):
    """The device structure build (build_tiled_device: the (chunk, tile) and
    per-row segment counts, the entries' slots and the bank balancing on the
    device; the host sees counts only) gives the all-host build's layout entry
    for entry: staged and direct column ids and value permutation, row
    pointers, row order, block bases, segment descriptors, work items,
    batches, chunks (pdcs_tiled_devbuild_check).  Ragged last chunks, empty
    rows and chunks with no staged tile are covered."""
    monkeypatch.setenv("PDCS_TILE_KB", kb)
    rng = np.random.default_rng(11)
    if which == "rand":
        A = _random_csr(rng, 3000, 9000, (1, 300)); nvec = 9000
    elif which == "band":
        A = _banded_csr(rng, 2500, 20000, (0, 400), 1500); nvec = 20000
    elif which == "mpoK":
        A, _ = _csr(gen_mpo(4, 200, seed=1)); nvec = A.shape[1]
    elif which == "fisherKT":
        _, A = _csr(gen_fisher(300, 100, 0.2, seed=2)); nvec = A.shape[1]
    else:
        K, KT = _csr(gen_lasso(3000, 300, 0.2, seed=6))
        A = K if which == "K" else KT
        nvec = A.shape[1]
    r = _lib.pdcs_tiled_devbuild_check(A.indptr.astype(np.int64), A.indices.astype(np.int32), A.shape[0],
                                       nvec, elem)
    assert r["mismatches"] == 0 and r["entries"] > 0, r
