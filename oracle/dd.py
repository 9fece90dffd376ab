"""Subdomain elimination (f3) and primal recovery (f2) -- oracle (TEST INFRASTRUCTURE ONLY).

PAPER.md:27 (§II): the arrowhead system [K C; C^T A_bb] "is then reduced in size by eliminating
via many independent sparse direct factorizations the primal DoFs"; "the solution of
all or a subset of primal unknowns are recovered in an embarrassingly parallel manner via many
smaller size sparse forward backward substitutions".  Both results have plain definitions, and
this oracle is those definitions written out (one subdomain at a time, in ascending p), with the
sparse direct solve K_p^{-1} as a single library step (scipy SuperLU, `splu`, natural column
order -- an LU, i.e. a different algorithm from the library's restricted-BK LDL^T):

  S_p     = A_bb,p - C_p^T K_p^{-1} C_p                    (dense m_p x m_p Schur contribution)
  g       = b_b - sum_p R_p^T C_p^T K_p^{-1} f_p            (condensed right-hand side)
  A_aux   = sum_p R_p^T S_p R_p                             (the auxiliary matrix, f1)
  x_p     = K_p^{-1} (f_p - C_p R_p x_b)                    (primal recovery)

R_p selects p's interfaces' dual DoFs from the global dual vector.  Inputs are a
dd_inputs.fem.FEMDD model.  Pins (tests/test_oracle_dd.py, -m "not gpu"): the whole pipeline
against scipy's direct sparse solve of the global arrowhead matrix; sum_p S_p against the dense
Schur complement of the global matrix; symmetry; decoupled and zero special cases; a
manufactured solution.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse.linalg as spl

from dd_inputs.fem import abb_share


def _lu(K):
    return spl.splu(K.tocsc(), permc_spec="NATURAL")


def dual_rows(m, p):
    """Global dual DoFs of p's interfaces, concatenated in ascending interface id (R_p)."""
    if not m.sub_ifaces[p]:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate([m.dual_offset(I) + np.arange(m.s_dual) for I in m.sub_ifaces[p]])


def schur_contribution(m, p, lu=None):
    """S_p = A_bb,p - C_p^T K_p^{-1} C_p (dense, m_p x m_p)."""
    lu = lu or _lu(m.K[p])
    C = m.C[p].toarray()
    W = lu.solve(C) if C.shape[1] else np.zeros_like(C)
    return np.diag(abb_share(m, p)) - C.T @ W


def condense(m, F=None, bb=None):
    """g = b_b - sum_p R_p^T C_p^T K_p^{-1} f_p (multi-column)."""
    F = m.f if F is None else F
    g = np.array(m.bb if bb is None else bb, dtype=np.result_type(m.bb, m.K[0].dtype))
    for p in range(m.nsub):
        if not m.sub_ifaces[p]:
            continue
        z = _lu(m.K[p]).solve(np.asarray(F[p], dtype=g.dtype))
        g[dual_rows(m, p)] -= m.C[p].T @ z
    return g


def aux_matrix(m, S=None):
    """Dense auxiliary matrix sum_p R_p^T S_p R_p."""
    n = m.n_dual
    A = np.zeros((n, n), dtype=np.complex128 if m.complex_ else np.float64)
    for p in range(m.nsub):
        r = dual_rows(m, p)
        Sp = schur_contribution(m, p) if S is None else S[p]
        A[np.ix_(r, r)] += Sp
    return A


def recover(m, p, xb, F=None):
    """x_p = K_p^{-1} (f_p - C_p R_p x_b)."""
    f = (m.f if F is None else F)[p]
    rhs = np.asarray(f, dtype=np.result_type(f, xb, m.K[p].dtype)) - m.C[p] @ xb[dual_rows(m, p)]
    return _lu(m.K[p]).solve(rhs)


def dd_solve(m):
    """The whole direct DD solve: condense, dense auxiliary solve, recover.  Returns (x_p list, x_b)."""
    g = condense(m)
    xb = np.linalg.solve(aux_matrix(m), g)
    return [recover(m, p, xb) for p in range(m.nsub)], xb
