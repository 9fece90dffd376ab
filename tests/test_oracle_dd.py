"""Pins for oracle.dd (f3 subdomain elimination, f2 primal recovery), CPU only.

Independent references: scipy's direct sparse solve of the GLOBAL arrowhead matrix (all primal
and dual unknowns at once, no decomposition), the dense Schur complement of the global matrix
onto the dual DoFs (numpy LAPACK solve), and special cases (decoupled subdomains, zero data,
a manufactured solution).  The block-layout generator is pinned against the sparse model too.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spl

from dd_inputs import dense_expand
from dd_inputs.fem import arrowhead, arrowhead_rhs, fem_dd, schur_block_problem
import oracle.dd as odd


@pytest.mark.parametrize("cplx", [False, True])
def test_pipeline_equals_global_sparse_solve(cplx):
    m = fem_dd(2, 2, 2, 6, complex_=cplx, seed=1, nrhs=3)
    xs, xb = odd.dd_solve(m)
    X = spl.spsolve(arrowhead(m).tocsc(), arrowhead_rhs(m))
    got = np.concatenate(xs + [xb])
    rel = np.abs(got - X).max(0) / np.abs(X).max(0)
    assert rel.max() <= 1e-10, rel.max()


@pytest.mark.parametrize("cplx", [False, True])
def test_schur_sum_equals_dense_schur_complement(cplx):
    m = fem_dd(3, 2, 1, 5, complex_=cplx, seed=2)
    A = arrowhead(m).toarray()
    nprim = m.nsub * m.a ** 3
    App, Apb, Abb = A[:nprim, :nprim], A[:nprim, nprim:], A[nprim:, nprim:]
    Sd = Abb - Apb.T @ np.linalg.solve(App, Apb)          # plain transpose: complex symmetric
    Sa = odd.aux_matrix(m)
    assert np.abs(Sa - Sd).max() <= 1e-11 * np.abs(Sd).max()
    for p in range(m.nsub):
        S = odd.schur_contribution(m, p)
        assert np.abs(S - S.T).max() <= 1e-13 * np.abs(S).max()


def test_decoupled_and_zero_cases():
    m = fem_dd(2, 1, 1, 5, seed=3)
    for p in range(m.nsub):                                # C_p = 0 -> S_p = A_bb,p
        m.C[p] = m.C[p] * 0.0
    S = odd.schur_contribution(m, 0)
    assert np.array_equal(S, np.diag(np.full(S.shape[0], 0.05)))
    xb = np.zeros((m.n_dual, 2))
    F = [np.zeros_like(f[:, :2]) for f in m.f]
    assert np.all(odd.recover(m, 0, xb, F) == 0)          # zero data -> zero primal


def test_manufactured_solution():
    m = fem_dd(2, 2, 1, 6, seed=4, nrhs=2)
    A = arrowhead(m)
    rng = np.random.default_rng(0)
    X0 = rng.standard_normal((A.shape[0], 2))
    B = A @ X0
    n_p = m.a ** 3
    m.f = [B[p * n_p:(p + 1) * n_p] for p in range(m.nsub)]
    m.bb = B[m.nsub * n_p:]
    xs, xb = odd.dd_solve(m)
    got = np.concatenate(xs + [xb])
    assert np.abs(got - X0).max() <= 1e-10 * np.abs(X0).max()


@pytest.mark.parametrize("cplx", [False, True])
def test_block_layout_reproduces_arrowhead(cplx):
    """dd_inputs.fem.schur_block_problem: the block-sparse input of the partial factorization is
    the arrowhead matrix with one copy of the dual DoFs per subdomain (copies sum back to A)."""
    m = fem_dd(2, 2, 1, 6, complex_=cplx, seed=5)
    prob, ns, tgt, grp, auxs, info = schur_block_problem(m, leaf=16)
    D = dense_expand(prob)
    n_p = m.a ** 3
    rows = np.concatenate([p * n_p + info["node_perm"] for p in range(m.nsub)] +
                          [m.nsub * n_p + tgt[k] * m.s_dual + np.arange(m.s_dual) for k in range(ns)])
    R = np.zeros((arrowhead(m).shape[0], D.shape[0]))
    R[rows, np.arange(len(rows))] = 1
    assert np.array_equal(R @ D @ R.T, arrowhead(m).toarray())
    # kept blocks are the last ids, grouped by subdomain, with their interface targets
    assert ns == sum(len(x) for x in m.sub_ifaces)
    assert list(grp) == sorted(grp)
