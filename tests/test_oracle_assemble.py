"""Pins for oracle.assemble (f1 clique assembly), CPU only.

The oracle's loop is checked against the matrix definition A = sum_p R_p^T Ssym_p R_p
evaluated densely with explicit 0/1 selection matrices R_p (SURVEY.md
§8(f) f1; ledger L12), on cliques that overlap arbitrarily (several cliques per block),
plus the generator's own accumulation, the no-op symmetrisation of symmetric input and the
complex-symmetric (no conjugation) case.
"""
import numpy as np
import pytest

import dd_inputs
from dd_inputs import Problem, block_pattern_from_cliques, dense_expand
import oracle


def random_cliques(nblk, ncl, rng, kmin=1, kmax=5, smax=40, complex_=False):
    sizes = rng.integers(1, smax + 1, nblk).astype(np.int64)
    cliques = []
    for _ in range(ncl):
        k = int(rng.integers(kmin, min(kmax, nblk) + 1))
        cliques.append(sorted(int(x) for x in rng.choice(nblk, k, replace=False)))
    colptr, rowidx = block_pattern_from_cliques(nblk, cliques)
    val_offset, total = dd_inputs._layout(sizes, colptr, rowidx)
    S = []
    for c in cliques:
        m = int(sizes[c].sum())
        M = rng.standard_normal((m, m))
        if complex_:
            M = M + 1j * rng.standard_normal((m, m))
        S.append(M)
    return sizes, colptr, rowidx, val_offset, cliques, S


def dense_definition(sizes, cliques, S, symmetrize):
    n = int(sizes.sum())
    off = np.concatenate([[0], np.cumsum(sizes)])
    A = np.zeros((n, n), dtype=np.result_type(*S))
    for c, Sp in zip(cliques, S):
        idx = np.concatenate([np.arange(off[I], off[I + 1]) for I in c])
        R = np.zeros((len(idx), n))
        R[np.arange(len(idx)), idx] = 1.0                 # R_p: clique DoF -> global DoF
        Ssym = 0.5 * (Sp + Sp.T) if symmetrize else Sp
        A = A + R.T @ Ssym @ R
    return A


@pytest.mark.parametrize("complex_", [False, True])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_matches_dense_definition(complex_, seed):
    rng = np.random.default_rng(seed)
    sizes, colptr, rowidx, vo, cl, S = random_cliques(9, 7, rng, complex_=complex_)
    vals = oracle.assemble(sizes, colptr, rowidx, vo, cl, S, symmetrize=True)
    p = Problem(sizes, colptr, rowidx, vals, vo, [])
    A = dense_expand(p)
    Ad = dense_definition(sizes, cl, S, True)
    assert np.max(np.abs(A - Ad)) <= 1e-14 * np.max(np.abs(Ad))
    assert np.array_equal(A, A.T)                          # complex symmetric, never Hermitian
    # overlap really happened: some block is covered by several cliques
    cover = {}
    for c in cl:
        for a in c:
            for b in c:
                cover[(a, b)] = cover.get((a, b), 0) + 1
    assert max(cover.values()) >= 2


def test_unsymmetrized_lower_blocks():
    """symmetrize=False takes S_p's lower blocks as given (upper ones never read)."""
    rng = np.random.default_rng(5)
    sizes, colptr, rowidx, vo, cl, S = random_cliques(6, 5, rng)
    vals = oracle.assemble(sizes, colptr, rowidx, vo, cl, S, symmetrize=False)
    Ad = dense_definition(sizes, cl, S, False)
    p = Problem(sizes, colptr, rowidx, vals, vo, [])
    off = p.dof_offset
    for (i, j), blk in p.blocks().items():
        ref = Ad[off[i]:off[i + 1], off[j]:off[j + 1]]
        assert np.max(np.abs(blk - ref)) <= 1e-14 * max(1.0, np.max(np.abs(ref)))


def test_symmetric_input_noop():
    rng = np.random.default_rng(7)
    sizes, colptr, rowidx, vo, cl, S = random_cliques(8, 6, rng, complex_=True)
    Ssym = [0.5 * (M + M.T) for M in S]
    a = oracle.assemble(sizes, colptr, rowidx, vo, cl, S, symmetrize=True)
    b = oracle.assemble(sizes, colptr, rowidx, vo, cl, Ssym, symmetrize=False)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name,grid,sizes", [("cfg0", None, None), ("cfg2", (3, 3, 2), 20), ("cfg3", (2, 2, 2), 12)])
def test_generator_accumulation(name, grid, sizes):
    """The seeded generator's own accumulation (dd_inputs) equals the oracle's assembly bit for bit."""
    p = dd_inputs.config(name, grid=grid, sizes=sizes, keep_cliques=True)
    vals = oracle.assemble(p.blk_size, p.colptr, p.rowidx, p.val_offset, [c for _, c in p.cliques], p.clique_S)
    assert np.array_equal(vals, p.values)


def test_uncovered_blocks_zero():
    sizes = np.array([3, 4, 5], dtype=np.int64)
    colptr, rowidx = block_pattern_from_cliques(3, [[0, 2], [1]])
    vo, total = dd_inputs._layout(sizes, colptr, rowidx)
    vals = oracle.assemble(sizes, colptr, rowidx, vo, [[0, 2]], [np.ones((8, 8))])
    p = Problem(sizes, colptr, rowidx, vals, vo, [])
    assert np.all(p.blocks()[(1, 1)] == 0) and np.all(p.blocks()[(2, 0)] == 1)
