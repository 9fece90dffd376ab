"""Block LDL^T of the auxiliary matrix + multi-RHS solve -- oracle (test infrastructure).

PAPER.md:29 (§II APPROACH): the auxiliary matrix is "symmetric ... block-wise
sparse (sparse collection of dense blocks)"; it "is LDL^T factorized via a very
fast symbolic factorization step [on the] attributed clique graph of the
block-wise sparse matrix, followed by a custom block LDL^T with restricted
Bunch-Kaufman pivoting"; then "the auxiliary problem" is solved by forward /
backward substitution for many excitations.

Step by step:
  O1 symbolic: elimination game on the block graph in the given block order pi:
     eliminating k makes its current neighbours struct(k) a clique (L14).
  O3 for k in pi:
     a. in-block restricted BK of the updated A_kk          (oracle.bk, L1-L5)
     b. panel: for i in struct(k): A_ik <- A_ik P_k^T; W_ik = A_ik L_kk^{-T};
        L_ik = W_ik D_k^{-1}
     c. update: for i, j in struct(k):  A_ij <- A_ij - W_ik L_jk^T
  O4 inertia from D (real only; Sylvester)
  O5 solve: y = P b; forward L; D^{-1}; backward L^T; x = P^T y
  O6 refinement: r = b - A x on the ORIGINAL blocks, x += solve(r)  (L7)

Blocks are stored in dictionaries keyed by original interface ids (i, k) with
i after k in elimination order, each dense s_i x s_k.  Library primitives used
as single steps: numpy matmul (@) and scipy.linalg.solve_triangular.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple

import numpy as np
from scipy.linalg import solve_triangular

from .bk import bk_factor, apply_dinv, solve_d, inertia_of_d


# ------------------------------------------------------------------ O1 symbolic
def symbolic(nblk: int, colptr, rowidx, order: Sequence[int]):
    """Elimination game on the block graph ("symbolic factorization step
    ... clique graph"; SPEC.md:460,488 clique-completion rule).

    Returns dict with
      pos[k]       elimination position of block k
      struct[k]    list of blocks adjacent to k when it is eliminated, sorted by position
      fill         set of (i, j) pairs (original ids, unordered as (max,min) by id) created
      parent[k]    elimination-tree parent = earliest-eliminated member of struct(k), or -1
      level[k]     height in the elimination tree (leaves 0)
    """
    order = [int(x) for x in order]
    assert sorted(order) == list(range(nblk)), "order must be a permutation"
    pos = np.empty(nblk, dtype=np.int64)
    pos[order] = np.arange(nblk)
    adj: List[set] = [set() for _ in range(nblk)]
    orig = set()
    for j in range(nblk):
        for p in range(int(colptr[j]), int(colptr[j + 1])):
            i = int(rowidx[p])
            if i != j:
                adj[i].add(j)
                adj[j].add(i)
                orig.add((max(i, j), min(i, j)))
    eliminated = np.zeros(nblk, dtype=bool)
    struct: List[List[int]] = [[] for _ in range(nblk)]
    fill = set()
    for k in order:
        nb = [v for v in adj[k] if not eliminated[v]]
        nb.sort(key=lambda v: pos[v])
        struct[k] = nb
        for a in range(len(nb)):
            for b in range(a + 1, len(nb)):
                u, v = nb[a], nb[b]
                if v not in adj[u]:
                    adj[u].add(v)
                    adj[v].add(u)
                    fill.add((max(u, v), min(u, v)))
        eliminated[k] = True
    parent = np.full(nblk, -1, dtype=np.int64)
    for k in range(nblk):
        if struct[k]:
            parent[k] = struct[k][0]
    level = np.zeros(nblk, dtype=np.int64)
    for k in order:  # children are eliminated before parents
        if parent[k] >= 0:
            level[parent[k]] = max(level[parent[k]], level[k] + 1)
    return dict(pos=pos, struct=struct, fill=fill, orig=orig, parent=parent, level=level, order=order)


def flops_factor(sizes, sym, mu=1) -> float:
    """Algorithmic factor flops mu * sum_k (s^3/3 + r s^2 + r^2 s)."""
    tot = 0.0
    for k in range(len(sizes)):
        s = float(sizes[k])
        r = float(sum(sizes[i] for i in sym["struct"][k]))
        tot += s ** 3 / 3.0 + r * s * s + r * r * s
    return mu * tot


def flops_solve_per_rhs(sizes, sym, mu=1) -> float:
    """mu * 2 * sum_k (s^2 + 2 r s)."""
    tot = 0.0
    for k in range(len(sizes)):
        s = float(sizes[k])
        r = float(sum(sizes[i] for i in sym["struct"][k]))
        tot += 2.0 * (s * s + 2.0 * r * s)
    return mu * tot


# ------------------------------------------------------------------ O2-O3 numeric
@dataclasses.dataclass
class OracleFactor:
    sizes: np.ndarray
    sym: dict
    Lkk: Dict[int, np.ndarray]
    L: Dict[Tuple[int, int], np.ndarray]      # (i, k) -> L_ik, i in struct(k)
    d: Dict[int, np.ndarray]
    e: Dict[int, np.ndarray]
    ipiv: Dict[int, np.ndarray]
    perm: Dict[int, np.ndarray]
    info: int                                  # 0 or 1 + first zero-pivot global DoF (orig numbering)
    n2x2: int
    nonfinite: int = 0                         # pivot columns with non-finite decision values (L4b)
    nperturbed: int = 0                        # statically perturbed zero pivots (L4 opt-in)


def _lower_blocks(prob_blocks, sym):
    """O2: dense storage for every filled block, oriented (later, earlier) in elimination order."""
    pos = sym["pos"]
    A: Dict[Tuple[int, int], np.ndarray] = {}
    dtype = next(iter(prob_blocks.values())).dtype
    sizes = {}
    for (i, j), blk in prob_blocks.items():
        sizes[i], sizes[j] = blk.shape
    for (i, j), blk in prob_blocks.items():
        if i == j:
            A[(i, i)] = np.array(blk, dtype=dtype)
        elif pos[i] > pos[j]:
            A[(i, j)] = np.array(blk, dtype=dtype)
        else:
            A[(j, i)] = np.array(blk.T, dtype=dtype)
    for (u, v) in sym["fill"]:
        a, b = (u, v) if pos[u] > pos[v] else (v, u)
        A[(a, b)] = np.zeros((sizes[a], sizes[b]), dtype=dtype)
    return A


def block_factor(prob, order, perturb_tau=0.0) -> OracleFactor:
    """Right-looking block LDL^T with restricted BK (O3 a-c).

    perturb_tau > 0 (reading L4, opt-in): an exactly-zero pivot column gets
    the 1x1 pivot d = perturb_tau * ||A||_inf instead of reporting a zero pivot.
    `info` is the FIRST zero / non-finite pivot in elimination order (block order pi, then the
    column order inside the block), as LAPACK's INFO is for one block."""
    delta = perturb_tau * norm_inf_A(prob) if perturb_tau > 0 else 0.0
    sym = symbolic(prob.nblk, prob.colptr, prob.rowidx, order)
    A = _lower_blocks(prob.blocks(), sym)
    sizes = np.asarray(prob.blk_size)
    off = prob.dof_offset
    Lkk, L, d, e, ipiv, perm = {}, {}, {}, {}, {}, {}
    info = 0
    n2x2 = nonfinite = nperturbed = 0
    for k in sym["order"]:
        # a. in-block restricted Bunch-Kaufman on the updated diagonal block
        f = bk_factor(A[(k, k)], perturb_delta=delta)
        Lkk[k], d[k], e[k], ipiv[k], perm[k] = f["L"], f["d"], f["e"], f["ipiv"], f["perm"]
        n2x2 += f["n2x2"]
        nonfinite += f["nonfinite"]
        nperturbed += f["nperturbed"]
        if f["info"] and not info:
            info = int(off[k]) + int(perm[k][f["info"] - 1]) + 1
        # b. panel: column permutation, triangular solve, D scaling
        W = {}
        for i in sym["struct"][k]:
            Ahat = A[(i, k)][:, perm[k]]
            W[i] = solve_triangular(Lkk[k], Ahat.T, lower=True, unit_diagonal=True, check_finite=False).T  # Ahat Lkk^{-T}
            L[(i, k)] = apply_dinv(W[i], d[k], e[k], ipiv[k])
        # c. Schur update of every target pair in struct(k)
        st = sym["struct"][k]
        for a, i in enumerate(st):
            for j in st[:a + 1]:
                A[(i, j)] -= W[i] @ L[(j, k)].T
        A[(k, k)] = None  # consumed
        for i in st:
            A[(i, k)] = None
    return OracleFactor(sizes, sym, Lkk, L, d, e, ipiv, perm, info, n2x2, nonfinite, nperturbed)


def max_abs_L(F: OracleFactor) -> float:
    """max |L_ij| over the whole unit-lower factor (diagonal ones included; modulus for complex):
    the element-growth diagnostic of the restricted BK factorization (SURVEY.md §8(b) max_abs_L)."""
    m = 1.0
    for k in F.sym["order"]:
        m = max(m, float(np.abs(F.Lkk[k]).max()) if F.Lkk[k].size else 1.0)
        for i in F.sym["struct"][k]:
            if F.L[(i, k)].size:
                m = max(m, float(np.abs(F.L[(i, k)]).max()))
    return m


# ------------------------------------------------------------------ O4 inertia
def inertia(F: OracleFactor):
    p = q = z = 0
    for k in F.sym["order"]:
        a, b, c = inertia_of_d(F.d[k], F.e[k], F.ipiv[k])
        p, q, z = p + a, q + b, z + c
    return p, q, z


# ------------------------------------------------------------------ O5 solve
def block_solve(F: OracleFactor, B, off):
    """X = A^{-1} B via P, L, D, L^T, P^T ("forward backward substitution")."""
    # Rows of L_ik are in block i's ORIGINAL local order (perm_i is only chosen when
    # i itself is eliminated), so the running vector of a not-yet-eliminated block
    # stays in original order; perm_k is applied at k's diagonal solve and undone
    # after k's backward solve.
    B = np.asarray(B)
    dtype = np.result_type(B, next(iter(F.d.values())))
    y = {k: np.array(B[off[k]:off[k + 1]], dtype=dtype) for k in F.sym["order"]}
    z = {}
    for k in F.sym["order"]:                        # forward: L
        z[k] = solve_triangular(F.Lkk[k], y[k][F.perm[k]], lower=True, unit_diagonal=True, check_finite=False)
        for i in F.sym["struct"][k]:
            y[i] = y[i] - F.L[(i, k)] @ z[k]
    for k in F.sym["order"]:                        # D
        z[k] = solve_d(z[k], F.d[k], F.e[k], F.ipiv[k])
    x = {}
    for k in reversed(F.sym["order"]):              # backward: L^T
        for i in F.sym["struct"][k]:
            z[k] = z[k] - F.L[(i, k)].T @ x[i]
        zk = solve_triangular(F.Lkk[k].T, z[k], lower=False, unit_diagonal=True, check_finite=False)
        x[k] = np.empty_like(zk)
        x[k][F.perm[k]] = zk
    X = np.empty(B.shape, dtype=dtype)
    for k in F.sym["order"]:
        X[off[k]:off[k + 1]] = x[k]
    return X


def matvec_blocks(prob, X):
    """A X with the full symmetric A given by its lower blocks (lower triangle of diagonal blocks)."""
    off = prob.dof_offset
    Y = np.zeros(X.shape, dtype=np.result_type(prob.values, X))
    for (i, j), blk in prob.blocks().items():
        if i == j:
            S = np.tril(blk) + np.tril(blk, -1).T
            Y[off[i]:off[i + 1]] += S @ X[off[i]:off[i + 1]]
        else:
            Y[off[i]:off[i + 1]] += blk @ X[off[j]:off[j + 1]]
            Y[off[j]:off[j + 1]] += blk.T @ X[off[i]:off[i + 1]]
    return Y


def norm_inf_A(prob):
    """||A||_inf: max absolute row sum of the full symmetric A (modulus for complex)."""
    off = prob.dof_offset
    rs = np.zeros(prob.n)
    for (i, j), blk in prob.blocks().items():
        if i == j:
            S = np.tril(blk) + np.tril(blk, -1).T
            rs[off[i]:off[i + 1]] += np.abs(S).sum(axis=1)
        else:
            rs[off[i]:off[i + 1]] += np.abs(blk).sum(axis=1)
            rs[off[j]:off[j + 1]] += np.abs(blk).sum(axis=0)
    return float(rs.max())


def residual_berr(prob, X, B, normA=None):
    """Per-column backward error ||A x_j - b_j||_inf / (||A||_inf ||x_j||_inf) (north_star, L6)."""
    if normA is None:
        normA = norm_inf_A(prob)
    R = B - matvec_blocks(prob, X)
    num = np.abs(R).max(axis=0)
    den = normA * np.abs(X).max(axis=0)
    return num / np.where(den == 0, 1.0, den)


def refine_solve(prob, F: OracleFactor, B, refine_steps=1, refine_tol=0.0):
    """O6: x = solve(b); repeat refine_steps times: r = b - A x; x += solve(r).

    The step is skipped when max_j berr_j <= refine_tol (refine_tol = 0 always
    refines), the same policy dd_aux_solve applies (reading L7).
    Returns (X, berr_before, berr_after).
    """
    off = prob.dof_offset
    X = block_solve(F, B, off)
    normA = norm_inf_A(prob)
    berr0 = residual_berr(prob, X, B, normA)
    berr = berr0
    for _ in range(refine_steps):
        if refine_tol > 0 and berr.max() <= refine_tol:
            break
        R = B - matvec_blocks(prob, X)
        X = X + block_solve(F, R, off)
        berr = residual_berr(prob, X, B, normA)
    return X, berr0, berr


def global_permutation(F: OracleFactor, off):
    """Global P with (P A P^T)[a, b] = A[gp[a], gp[b]] (block order then in-block perm)."""
    gp = []
    for k in F.sym["order"]:
        gp.extend(int(off[k]) + F.perm[k])
    return np.asarray(gp)


def dense_factors(F: OracleFactor, off):
    """Dense L (unit lower) and D of P A P^T = L D L^T, in elimination-position order."""
    order = F.sym["order"]
    sizes = F.sizes
    poff = np.concatenate([[0], np.cumsum([sizes[k] for k in order])])
    pidx = {k: t for t, k in enumerate(order)}
    n = int(poff[-1])
    dtype = next(iter(F.Lkk.values())).dtype
    Ld = np.zeros((n, n), dtype=dtype)
    Dd = np.zeros((n, n), dtype=dtype)
    from .bk import d_matrix
    for k in order:
        a = pidx[k]
        Ld[poff[a]:poff[a + 1], poff[a]:poff[a + 1]] = F.Lkk[k]
        Dd[poff[a]:poff[a + 1], poff[a]:poff[a + 1]] = d_matrix(F.d[k], F.e[k], F.ipiv[k])
        for i in F.sym["struct"][k]:
            b = pidx[i]
            # L_ik rows are in block i's original order; P puts them in perm_i order
            Ld[poff[b]:poff[b + 1], poff[a]:poff[a + 1]] = F.L[(i, k)][F.perm[i]]
    return Ld, Dd
