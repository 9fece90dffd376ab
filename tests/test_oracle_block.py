"""Pins for oracle.block_ldlt (block LDL^T + solve + refinement), CPU only.

The three checks the north_star names -- brute-force dense LU solves, the
reconstruction ||P A P^T - L D L^T|| / ||A||, Sylvester inertia -- plus the
SPEC.md:522-526 random block-sparse corpus, one-group == dense BK,
block-diagonal == per-block BK, and negation / SPD metamorphics.
"""
import numpy as np
import pytest

import dd_inputs
from dd_inputs import Problem, block_pattern_from_cliques, dense_expand, random_rhs
import oracle
from oracle.bk import bk_factor
from oracle.block_ldlt import dense_factors, global_permutation, residual_berr

TOL_REL = 1e-9      # north_star: solution relative difference
TOL_BERR = 1e-12    # north_star: backward error


def _check_against_dense(p, order, nrhs=3, seed=0, refine=1):
    B = random_rhs(p.n, nrhs, p.is_complex, seed)
    F = oracle.block_factor(p, order)
    X, b0, b1 = oracle.refine_solve(p, F, B, refine)
    Ad = dense_expand(p)
    Xd = np.linalg.solve(Ad, B)                    # LAPACK getrf/getrs (partial-pivot LU)
    rel = (np.abs(X - Xd).max(axis=0) / np.abs(Xd).max(axis=0)).max()
    assert rel <= TOL_REL, rel
    assert b1.max() <= TOL_BERR, b1.max()
    Ld, Dd = dense_factors(F, p.dof_offset)
    gp = global_permutation(F, p.dof_offset)
    rec = np.linalg.norm(Ad[np.ix_(gp, gp)] - Ld @ Dd @ Ld.T) / np.linalg.norm(Ad)
    assert rec <= 1e-12, rec
    if not p.is_complex:
        ev = np.linalg.eigvalsh(Ad)
        assert oracle.inertia(F) == (int((ev > 0).sum()), int((ev < 0).sum()), 0)
    return F


def test_cfg0_all_orders():
    p = dd_inputs.config("cfg0")
    for order in ([0, 1, 2, 3], [3, 2, 1, 0], [1, 2, 0, 3], [2, 0, 3, 1]):
        _check_against_dense(p, order, nrhs=4)


@pytest.mark.parametrize("name,grid,s", [("cfg1", (2, 2, 2), 24), ("cfg1", (3, 2, 2), 16),
                                         ("cfg3", (2, 2, 2), 20), ("cfg2", (3, 3, 2), None)])
def test_scaled_down_configs(name, grid, s):
    kw = {} if s is None else {"sizes": s}
    if name == "cfg2":
        kw = {"sizes": lambda n, rng: rng.integers(4, 30, n)}
    p = dd_inputs.config(name, grid=grid, **kw)
    rng = np.random.default_rng(4)
    _check_against_dense(p, list(rng.permutation(p.nblk)))


def _random_block_problem(rng, cplx):
    """SPEC.md:522 corpus: 2-8 groups, sizes 1-40, 30-100% block density, zero-diagonal blocks."""
    nblk = int(rng.integers(2, 9))
    sizes = rng.integers(1, 41, nblk)
    dens = rng.uniform(0.3, 1.0)
    edges = [(u, v) for u in range(nblk) for v in range(u) if rng.random() < dens]
    colptr, rowidx = block_pattern_from_cliques(nblk, [list(e) for e in edges])
    off = []
    tot = 0
    for j in range(nblk):
        for q in range(colptr[j], colptr[j + 1]):
            off.append(tot)
            tot += int(sizes[rowidx[q]]) * int(sizes[j])
    vals = rng.standard_normal(tot)
    if cplx:
        vals = vals + 1j * rng.standard_normal(tot)
    p = Problem(np.asarray(sizes, dtype=np.int64), colptr, rowidx, vals, np.asarray(off, dtype=np.int64), [])
    if rng.random() < 0.3:  # zero-diagonal diagonal blocks
        for j in range(nblk):
            q = colptr[j]
            blk = p.block(q)
            np.fill_diagonal(blk, 0.0)
    return p


def test_spec_corpus():
    rng = np.random.default_rng(2024)
    done = 0
    for trial in range(200):
        if done == 60:
            break
        p = _random_block_problem(rng, cplx=(trial % 2 == 1))
        if np.linalg.cond(dense_expand(p)) > 1e10:   # exactly/near-singular draw: not a valid case
            continue
        done += 1
        order = list(rng.permutation(p.nblk))
        F = _check_against_dense(p, order, nrhs=2, seed=trial)
        # restriction contract: each in-block permutation stays inside its block
        for k in range(p.nblk):
            assert sorted(F.perm[k]) == list(range(int(p.blk_size[k])))


def test_one_group_equals_dense_bk():
    rng = np.random.default_rng(9)
    A = rng.standard_normal((37, 37))
    A = A + A.T
    p = Problem(np.array([37]), np.array([0, 1]), np.array([0], dtype=np.int32),
                np.asfortranarray(A).ravel(order="F"), np.array([0]), [])
    F = oracle.block_factor(p, [0])
    f = bk_factor(A)
    np.testing.assert_array_equal(F.ipiv[0], f["ipiv"])
    np.testing.assert_array_equal(F.Lkk[0], f["L"])
    np.testing.assert_array_equal(F.d[0], f["d"])


def test_block_diagonal_equals_per_block_bk():
    rng = np.random.default_rng(10)
    sizes = [5, 9, 3]
    vals = []
    mats = []
    for s in sizes:
        A = rng.standard_normal((s, s))
        A = A + A.T
        mats.append(A)
        vals.append(A.ravel(order="F"))
    off = np.concatenate([[0], np.cumsum([s * s for s in sizes])[:-1]])
    p = Problem(np.array(sizes), np.array([0, 1, 2, 3]), np.array([0, 1, 2], dtype=np.int32),
                np.concatenate(vals), off, [])
    F = oracle.block_factor(p, [2, 0, 1])
    for k in range(3):
        f = bk_factor(mats[k])
        np.testing.assert_array_equal(F.ipiv[k], f["ipiv"])
        np.testing.assert_array_equal(F.Lkk[k], f["L"])


def test_negation_and_spd_inertia():
    p = dd_inputs.config("cfg1", grid=(2, 2, 2), sizes=12)
    order = list(range(p.nblk))
    P, Q, Z = oracle.inertia(oracle.block_factor(p, order))
    neg = Problem(p.blk_size, p.colptr, p.rowidx, -p.values, p.val_offset, [])
    assert oracle.inertia(oracle.block_factor(neg, order)) == (Q, P, Z)
    # SPD variant: all d > 0 in the generator recipe -> A = sum G^T D G + 0.1 I is SPD
    rng = np.random.default_rng(0)
    spd = Problem(p.blk_size, p.colptr, p.rowidx, p.values.copy(), p.val_offset, [])
    Ad = dense_expand(p)
    ev = np.linalg.eigvalsh(Ad)
    shift = -ev.min() + 1.0
    for j in range(p.nblk):  # add shift*I to diagonal blocks
        np.fill_diagonal(spd.block(int(p.colptr[j])), np.diag(p.block(int(p.colptr[j]))) + shift)
    assert oracle.inertia(oracle.block_factor(spd, order)) == (p.n, 0, 0)


def test_refinement_policy():
    """refine_tol: a step is skipped iff max berr <= tol; refine_steps=0 returns the plain solve."""
    p = dd_inputs.config("cfg0")
    F = oracle.block_factor(p, [0, 1, 2, 3])
    B = random_rhs(p.n, 2, False, 1)
    X0, b0, b1 = oracle.refine_solve(p, F, B, 0)
    assert np.array_equal(b0, b1)
    X1, c0, c1 = oracle.refine_solve(p, F, B, 1, refine_tol=1.0)
    assert np.array_equal(X0, X1)
    np.testing.assert_allclose(residual_berr(p, X0, B), b0)
