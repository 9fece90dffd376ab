"""Round-2 pins of the oracle functions every GPU parity assertion leans on (CPU only).

Each check compares an oracle function with something other than itself:
  * norm_inf_A / matvec_blocks / residual_berr  -- the dense expansion of the block matrix
    (numpy abs-row-sum, dense matmul), i.e. the north_star definition
    ||A x - b||_inf / (||A||_inf ||x||_inf) written out on the full n x n matrix;
  * flops_solve_per_rhs / flops_factor           -- hand counts on configs[0] (a 4-cycle of
    32-DoF interfaces: struct sizes 2, 2, 1, 0 in ANY order);
  * the IDAMAX smallest-index tie rule (reading L3) -- LAPACK dsytrf on integer blocks full of
    exact ties (dd_inputs.tie_block), where every value is a short dyadic rational;
  * static perturbation (reading L4, opt-in)     -- reconstruction P (A + delta e_m e_m^T) P^T =
    L D L^T and the dense solve of the perturbed matrix;
  * zero / non-finite pivots (readings L4, L4b)  -- hand-derived first DoF in ELIMINATION order;
  * max_abs_L                                    -- a matrix built as L0 D0 L0^T whose BK
    factorization needs no interchange, so L = L0 exactly.
"""
import numpy as np
import pytest
import scipy.linalg.lapack as lapack

import dd_inputs
from dd_inputs import Problem, block_pattern_from_cliques, dense_expand, random_rhs
import oracle
from oracle.bk import bk_factor, d_matrix
from oracle.block_ldlt import (dense_factors, flops_factor, flops_solve_per_rhs, global_permutation, matvec_blocks,
                               max_abs_L, norm_inf_A, residual_berr, symbolic)


def _problems():
    yield dd_inputs.config("cfg0")
    yield dd_inputs.config("cfg1", grid=(2, 2, 2), sizes=12)
    yield dd_inputs.config("cfg2", grid=(3, 3, 2), sizes=lambda n, r: r.integers(3, 20, n))
    yield dd_inputs.config("cfg3", grid=(2, 2, 2), sizes=10)


@pytest.mark.parametrize("idx", range(4))
def test_norm_matvec_berr_against_dense(idx):
    p = list(_problems())[idx]
    Ad = dense_expand(p)
    # ||A||_inf = max absolute row sum of the full symmetric matrix (modulus for complex)
    assert norm_inf_A(p) == pytest.approx(float(np.abs(Ad).sum(axis=1).max()), rel=1e-14)
    X = random_rhs(p.n, 5, p.is_complex, idx)
    np.testing.assert_allclose(matvec_blocks(p, X), Ad @ X, rtol=1e-12, atol=1e-12 * np.abs(Ad @ X).max())
    B = random_rhs(p.n, 5, p.is_complex, idx + 10)
    want = np.abs(B - Ad @ X).max(axis=0) / (np.abs(Ad).sum(axis=1).max() * np.abs(X).max(axis=0))
    np.testing.assert_allclose(residual_berr(p, X, B), want, rtol=1e-12)
    # a double-counted diagonal block would change ||A||: the symmetric lower/upper split matters
    if p.nblk > 1:
        assert norm_inf_A(p) < float(np.abs(Ad).sum(axis=1).max()) * (1 + 1e-12)


def test_flop_counts_cfg0_hand():
    """configs[0]: 4 interfaces of 32 DoFs on a 4-cycle.  Any order eliminates vertices with
    |struct| = 2, 2, 1, 0, so sum r = 32 * (2 + 2 + 1) = 160 and
      solve  = 2 * (4 * 32^2 + 2 * 32 * 160)              = 28,672 per RHS
      factor = 4 * 32^3/3 + 160 * 32^2 + (64^2 * 2 + 32^2) * 32 = 502,444.67."""
    p = dd_inputs.config("cfg0")
    for order in ([0, 1, 2, 3], [3, 1, 0, 2], [2, 0, 3, 1]):
        sym = symbolic(p.nblk, p.colptr, p.rowidx, order)
        assert flops_solve_per_rhs(p.blk_size, sym) == 28672.0
        assert flops_factor(p.blk_size, sym) == pytest.approx(4 * 32 ** 3 / 3 + 160 * 1024 + (2 * 64 ** 2 + 32 ** 2) * 32)
        assert flops_solve_per_rhs(p.blk_size, sym, mu=4) == 4 * 28672.0


def _ties_in_first_columns(A):
    n = A.shape[0]
    cnt = 0
    for j in range(n - 1):
        c = np.abs(A[j + 1:, j])
        m = c.max()
        cnt += int(m > 0 and (c == m).sum() >= 2)
    return cnt


@pytest.mark.parametrize("s", [9, 96, 300, 1031])
def test_idamax_ties_match_lapack(s):
    """Reading L3: ties in the pivot search go to the smallest index (IDAMAX).  On tie_block the
    arithmetic is exact, so LAPACK dsytrf's ipiv is THE answer, bit for bit."""
    A = dd_inputs.tie_block(s, seed=s)
    assert _ties_in_first_columns(A) >= s // 12
    f = bk_factor(A)
    lu, ipiv, info = lapack.dsytrf(A, lower=1)
    assert info == 0 and f["info"] == 0
    np.testing.assert_array_equal(f["ipiv"], ipiv)
    assert f["n2x2"] > 0 and (f["perm"] != np.arange(s)).any()
    # exact arithmetic: every multiplier and pivot is a multiple of 1/64
    assert np.all(np.mod(f["L"] * 64, 1) == 0) and np.all(np.mod(f["d"] * 64, 1) == 0)
    np.testing.assert_array_equal(f["d"], np.diag(lu))


def _zero_dof_problem(rng, zero_dofs, sizes=(7, 5, 9, 6), cplx=False):
    """Dense-coupled 4-interface problem whose listed global DoFs have an all-zero row/column."""
    nblk = len(sizes)
    cliques = [list(range(nblk))]
    colptr, rowidx = block_pattern_from_cliques(nblk, cliques)
    n = int(sum(sizes))
    G = rng.standard_normal((n, n))
    A = G + G.T
    if cplx:
        H = rng.standard_normal((n, n))
        A = A + 1j * (H + H.T)
    for m in zero_dofs:
        A[m, :] = 0
        A[:, m] = 0
    off = np.concatenate([[0], np.cumsum(sizes)])
    vals, voff, tot = [], [], 0
    for j in range(nblk):
        for q in range(colptr[j], colptr[j + 1]):
            i = int(rowidx[q])
            blk = A[off[i]:off[i + 1], off[j]:off[j + 1]]
            voff.append(tot)
            vals.append(np.asfortranarray(blk).ravel(order="F"))
            tot += blk.size
    return Problem(np.asarray(sizes, dtype=np.int64), colptr, rowidx, np.concatenate(vals),
                   np.asarray(voff, dtype=np.int64), []), A


@pytest.mark.parametrize("cplx", [False, True])
def test_static_perturbation(cplx):
    """Reading L4 (opt-in): an exactly-zero pivot column gets d = tau * ||A||_inf.  The factor is
    then an exact BK factorization of A + delta * sum_m e_m e_m^T over the zero DoFs m."""
    rng = np.random.default_rng(3 + cplx)
    zero = [3, 15]
    p, A = _zero_dof_problem(rng, zero, cplx=cplx)
    order = [2, 0, 3, 1]
    F0 = oracle.block_factor(p, order)
    assert F0.info != 0 and F0.nperturbed == 0
    tau = 1e-3
    F = oracle.block_factor(p, order, perturb_tau=tau)
    delta = tau * float(np.abs(A).sum(axis=1).max())
    assert F.info == 0 and F.nperturbed == len(zero) and F.nonfinite == 0
    Ap = A.copy()
    for m in zero:
        Ap[m, m] = delta
    off = p.dof_offset
    Ld, Dd = dense_factors(F, off)
    gp = global_permutation(F, off)
    rec = np.linalg.norm(Ap[np.ix_(gp, gp)] - Ld @ Dd @ Ld.T) / np.linalg.norm(Ap)
    assert rec <= 1e-13, rec
    B = random_rhs(p.n, 3, cplx, 1)
    from oracle.block_ldlt import block_solve
    X = block_solve(F, B, off)
    Xd = np.linalg.solve(Ap, B)
    assert (np.abs(X - Xd).max(0) / np.abs(Xd).max(0)).max() <= 1e-9


def test_first_zero_pivot_in_elimination_order():
    """Reading L4: info = 1 + ORIGINAL DoF of the first zero pivot in ELIMINATION order (block
    order pi, then column order inside the block) -- LAPACK INFO generalised to blocks."""
    rng = np.random.default_rng(8)
    sizes = (7, 5, 9, 6)
    off = np.concatenate([[0], np.cumsum(sizes)])
    zero = [int(off[1]) + 2, int(off[3]) + 4]           # one zero DoF in block 1, one in block 3
    p, _ = _zero_dof_problem(rng, zero, sizes)
    assert oracle.block_factor(p, [0, 1, 2, 3]).info == zero[0] + 1
    assert oracle.block_factor(p, [3, 2, 1, 0]).info == zero[1] + 1   # block 3 is eliminated first
    assert oracle.block_factor(p, [2, 3, 0, 1]).info == zero[1] + 1


def test_nonfinite_pivot_first_column():
    """Reading L4b: a NaN (or Inf) in the pivot column is a non-finite pivot at that column."""
    rng = np.random.default_rng(9)
    p, A = _zero_dof_problem(rng, [], sizes=(6, 5, 7))
    order = [1, 2, 0]
    off = p.dof_offset
    for bad in (np.nan, np.inf):
        q = dd_inputs.Problem(p.blk_size, p.colptr, p.rowidx, p.values.copy(), p.val_offset, [])
        blk = q.block(int(q.colptr[1]))           # diagonal block of interface 1 (eliminated first)
        blk[3, 0] = bad                           # column 0, row 3 (lower triangle)
        F = oracle.block_factor(q, order)
        assert F.info == int(off[1]) + 0 + 1 and F.nonfinite >= 1
        # and in the diagonal entry itself (LAPACK's DISNAN(absakk) branch)
        q2 = dd_inputs.Problem(p.blk_size, p.colptr, p.rowidx, p.values.copy(), p.val_offset, [])
        q2.block(int(q2.colptr[1]))[0, 0] = bad
        F2 = oracle.block_factor(q2, order)
        assert F2.info == int(off[1]) + 1 and F2.nonfinite >= 1


@pytest.mark.parametrize("cplx", [False, True])
def test_max_abs_L_no_pivoting(cplx):
    """A = L0 D0 L0^T with CABS1(L0) <= 1.4 and |D0| >= 1 makes every BK step a 1x1 pivot without
    interchange (|a_kk| = |d_k| >= alpha * 1.4 |d_k| >= alpha * colmax), so the block factor in
    natural order reproduces L0 and max_abs_L must equal max |L0|."""
    rng = np.random.default_rng(12 + cplx)
    sizes = (6, 9, 5)
    n = sum(sizes)
    re = 1.1 if cplx else 1.4             # complex pivoting measures CABS1 = |Re| + |Im| <= 1.4
    L0 = np.tril(rng.uniform(-re, re, (n, n)), -1) + np.eye(n)
    if cplx:
        L0 = L0 + 1j * np.tril(rng.uniform(-0.3, 0.3, (n, n)), -1)
    d0 = rng.choice([-1.0, 1.0], n) * rng.uniform(1.0, 2.0, n)
    A = L0 @ np.diag(d0) @ L0.T
    colptr, rowidx = block_pattern_from_cliques(3, [[0, 1, 2]])
    off = np.concatenate([[0], np.cumsum(sizes)])
    vals, voff, tot = [], [], 0
    for j in range(3):
        for q in range(colptr[j], colptr[j + 1]):
            i = int(rowidx[q])
            blk = A[off[i]:off[i + 1], off[j]:off[j + 1]]
            voff.append(tot)
            vals.append(np.asfortranarray(blk).ravel(order="F"))
            tot += blk.size
    p = Problem(np.asarray(sizes, dtype=np.int64), colptr, rowidx, np.concatenate(vals), np.asarray(voff), [])
    F = oracle.block_factor(p, [0, 1, 2])
    assert all((F.perm[k] == np.arange(sizes[k])).all() for k in range(3))
    assert max_abs_L(F) == pytest.approx(float(np.abs(L0).max()), rel=1e-10)
