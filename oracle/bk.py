"""Dense Bunch-Kaufman LDL^T of ONE diagonal block -- oracle (test infrastructure).

PAPER.md:29 (§II): "a custom block LDL^T with restricted Bunch-Kaufman pivoting
[BUNCH1977]".  Reading L1: the pivot search (colmax, rowmax) never
leaves the diagonal block of one interface, so this function is applied to each
updated diagonal block A_kk in isolation.  The decision rule is Bunch & Kaufman's
partial pivoting with alpha = (1+sqrt(17))/8, in the exact order of LAPACK
xSYTF2 (lower), so LAPACK ?sytrf is an independent pin of every decision:

  for column k (0-based) of the remaining block:
    absakk = |a_kk|;  (imax, colmax) = argmax_{i>k} |a_ik|  (first index on ties)
    if max(absakk, colmax) == 0:  zero pivot, 1x1, no elimination      (L4)
    elif absakk >= alpha*colmax:  1x1, no swap
    else: rowmax = max_{j in [k,n), j != imax} |a_{imax,j}|  (symmetric access)
          if absakk >= alpha*colmax*(colmax/rowmax):  1x1, no swap
          elif |a_{imax,imax}| >= alpha*rowmax:        1x1, swap k <-> imax
          else:                                        2x2, swap k+1 <-> imax
    symmetric interchange of the trailing block AND of the rows of the
    already-computed L columns (explicit form, reading L5);
    rank-1 / rank-2 update of the trailing block.

|.| is abs for real and CABS1 = |Re|+|Im| for complex (LAPACK zsytf2; reading L2).
Complex matrices are complex *symmetric*: plain transposes, no conjugation.

Output (P A P^T = L D L^T, (P A P^T)[i, j] = A[perm[i], perm[j]]):
  L    unit lower triangular (s x s)
  d    diagonal of D;  e[k] = D[k+1, k] for the first column of a 2x2 pivot, else 0
  ipiv LAPACK convention (1-based): ipiv[k] = kp+1 for a 1x1 pivot, and
       ipiv[k] = ipiv[k+1] = -(kp+1) for a 2x2 pivot
  perm composite permutation
  info 0, or 1 + first column with a zero or non-finite pivot (LAPACK INFO)
  nonfinite  number of pivot columns whose decision quantities (absakk, colmax,
       or rowmax when it is evaluated) were not finite (reading L4b)
  nperturbed number of exactly-zero pivot columns given d = perturb_delta
       (opt-in static perturbation, reading L4)

Failure readings (L4, L4b): LAPACK's xSYTF2 treats
max(absakk, colmax) == 0 or DISNAN(absakk) as a zero pivot (INFO = k, no
elimination).  This oracle extends the non-finite test to colmax and rowmax
(NaN or Inf anywhere in the pivot column or the imax row), where LAPACK's
IDAMAX would silently skip a NaN; on finite input the rule is LAPACK's exactly.
With perturb_delta > 0 an exactly-zero pivot column is instead given the 1x1
pivot d = +perturb_delta ("perturbation fallback ... flagged")
and does not set info.
"""
from __future__ import annotations

import math

import numpy as np

ALPHA = (1.0 + math.sqrt(17.0)) / 8.0


def cabs1(z):
    """|Re| + |Im| (LAPACK CABS1) for complex; abs for real (reading L2)."""
    if np.iscomplexobj(z):
        return np.abs(np.real(z)) + np.abs(np.imag(z))
    return np.abs(z)


def _argmax_first(v):
    """Index of the first maximum (IDAMAX / IZAMAX tie rule, reading L3)."""
    return int(np.argmax(v))  # numpy returns the first occurrence


def _rel_gap(x, y):
    """Relative distance of the two sides of a pivot-test comparison (diagnostic only)."""
    den = max(abs(x), abs(y))
    return abs(x - y) / den if den > 0 else 0.0


def bk_factor(A, perturb_delta=0.0, margins=None):
    """Restricted Bunch-Kaufman LDL^T of one symmetric block; lower triangle read.

    margins (optional list, diagnostic only -- it changes no decision): receives, per pivot
    step, (k, m) with m the smallest relative gap between the two sides of every comparison the
    step evaluated (the alpha tests, and the largest vs second-largest |a_ik| that fixes imax).
    A decision another correct implementation may legitimately take the other way under a
    different rounding order is one with a tiny m (DESIGN.md "near-tie" reading of L3)."""
    A = np.asarray(A)
    n = A.shape[0]
    a = np.tril(A).astype(np.complex128 if np.iscomplexobj(A) else np.float64)  # working copy, lower used
    ipiv = np.zeros(n, dtype=np.int64)
    perm = np.arange(n)
    info = 0
    n2x2 = 0
    nonfinite = 0
    nperturbed = 0

    def sym(i, j):  # a(i, j) of the symmetric working matrix from its lower triangle
        return a[i, j] if i >= j else a[j, i]

    k = 0
    while k < n:
        kstep = 1
        absakk = float(cabs1(a[k, k]))
        if k + 1 < n:
            col = cabs1(a[k + 1:, k])
            imax = k + 1 + _argmax_first(col)
            colmax = float(col[imax - k - 1])
        else:
            imax, colmax = k, 0.0
        bad = not (math.isfinite(absakk) and math.isfinite(colmax))
        if not bad and max(absakk, colmax) == 0.0 and perturb_delta > 0.0:
            a[k, k] = perturb_delta          # static perturbation (L4 opt-in): 1x1 pivot, no swap
            absakk = float(cabs1(a[k, k]))
            nperturbed += 1
        elif bad or max(absakk, colmax) == 0.0:
            nonfinite += int(bad)
            if info == 0:
                info = k + 1
            kp = k
            ipiv[k] = kp + 1
            k += 1
            continue
        gaps = []
        if margins is not None and k + 1 < n and col.size > 1:
            top2 = np.partition(col, col.size - 2)[-2:]
            gaps.append(_rel_gap(float(top2[1]), float(top2[0])))
        if margins is not None:
            gaps.append(_rel_gap(absakk, ALPHA * colmax))
        if absakk >= ALPHA * colmax:
            kp = k
        else:
            # rowmax over row imax of the trailing block, excluding the diagonal entry
            rowvals = np.array([cabs1(sym(imax, j)) for j in range(k, n) if j != imax])
            rowmax = float(np.max(rowvals))      # np.max propagates NaN (L4b)
            if not math.isfinite(rowmax):
                nonfinite += 1
                if info == 0:
                    info = k + 1
                ipiv[k] = k + 1
                k += 1
                continue
            if margins is not None:
                gaps.append(_rel_gap(absakk, ALPHA * colmax * (colmax / rowmax)))
                gaps.append(_rel_gap(float(cabs1(a[imax, imax])), ALPHA * rowmax))
            if absakk >= ALPHA * colmax * (colmax / rowmax):
                kp = k
            elif float(cabs1(a[imax, imax])) >= ALPHA * rowmax:
                kp = imax
            else:
                kp = imax
                kstep = 2
        if margins is not None:
            margins.append((k, min(gaps) if gaps else 1.0))
        kk = k + kstep - 1
        if kp != kk:
            # symmetric interchange of indices kk < kp, lower-triangle storage:
            #   column parts below kp
            a[kp + 1:, [kk, kp]] = a[kp + 1:, [kp, kk]]
            #   column kk between the two  <->  row kp between the two
            mid = np.arange(kk + 1, kp)
            t = a[mid, kk].copy()
            a[mid, kk] = a[kp, mid]
            a[kp, mid] = t
            #   diagonal entries
            a[kk, kk], a[kp, kp] = a[kp, kp], a[kk, kk]
            #   rows kk, kp in every column left of kk: the trailing block's column k
            #   (2x2 case) and -- explicit form, reading L5 -- all computed L columns
            a[[kk, kp], :kk] = a[[kp, kk], :kk]
            perm[[kk, kp]] = perm[[kp, kk]]
        if kstep == 1:
            d11 = a[k, k]
            x = a[k + 1:, k].copy()
            l = x / d11
            # trailing rank-1 update  A22 <- A22 - x x^T / d11
            a[k + 1:, k + 1:] -= np.tril(np.outer(l, x))
            a[k + 1:, k] = l
            ipiv[k] = kp + 1
        else:
            D = np.array([[a[k, k], a[k + 1, k]], [a[k + 1, k], a[k + 1, k + 1]]])
            X = a[k + 2:, k:k + 2].copy()          # (n-k-2) x 2 block column
            Dinv = np.linalg.inv(D)                 # 2x2 closed form inverse (library primitive)
            Lc = X @ Dinv
            # trailing rank-2 update  A22 <- A22 - X D^{-1} X^T
            a[k + 2:, k + 2:] -= np.tril(Lc @ X.T)
            a[k + 2:, k:k + 2] = Lc
            ipiv[k] = ipiv[k + 1] = -(kp + 1)
            n2x2 += 1
        k += kstep

    d = np.diag(a).copy()
    e = np.zeros(n, dtype=a.dtype)
    L = np.tril(a, -1) + np.eye(n, dtype=a.dtype)
    k = 0
    while k < n:
        if ipiv[k] < 0:
            e[k] = a[k + 1, k]
            L[k + 1, k] = 0.0
            k += 2
        else:
            k += 1
    return dict(L=L, d=d, e=e, ipiv=ipiv, perm=perm, info=info, n2x2=n2x2, nonfinite=nonfinite,
                nperturbed=nperturbed)


def d_matrix(d, e, ipiv):
    """Block-diagonal D (1x1 / 2x2) from (d, e, ipiv)."""
    n = len(d)
    D = np.diag(d).astype(np.result_type(d, e))
    k = 0
    while k < n:
        if ipiv[k] < 0:
            D[k + 1, k] = D[k, k + 1] = e[k]
            k += 2
        else:
            k += 1
    return D


def apply_dinv(W, d, e, ipiv):
    """W D^{-1} column-pair-wise (1x1 divide, 2x2 closed-form inverse).

    A zero 1x1 pivot (info > 0, LAPACK semantics) leaves the column as is: its
    column below the pivot is exactly zero in the block, and the caller reports
    the matrix singular (reading L4).
    """
    W = np.asarray(W)
    L = np.empty_like(W)
    n = len(d)
    k = 0
    while k < n:
        if ipiv[k] < 0:
            a, b, c = d[k], e[k], d[k + 1]
            det = a * c - b * b
            L[:, k] = (c * W[:, k] - b * W[:, k + 1]) / det
            L[:, k + 1] = (a * W[:, k + 1] - b * W[:, k]) / det
            k += 2
        else:
            L[:, k] = W[:, k] / d[k] if d[k] != 0 else W[:, k]
            k += 1
    return L


def solve_d(y, d, e, ipiv):
    """y <- D^{-1} y (rows), D block diagonal 1x1 / 2x2."""
    return apply_dinv(np.asarray(y).T, d, e, ipiv).T


def inertia_of_d(d, e, ipiv):
    """(n+, n-, n0) of a real D: 1x1 by sign; 2x2 by det<0 -> (+1,-1), else by trace sign.

    Sylvester's law of inertia makes this the inertia of the factored matrix
    (north_star: "identical inertia for real-symmetric cases").
    """
    npos = nneg = nzero = 0
    n = len(d)
    k = 0
    while k < n:
        if ipiv[k] < 0:
            a, b, c = float(np.real(d[k])), float(np.real(e[k])), float(np.real(d[k + 1]))
            det = a * c - b * b
            if det < 0:
                npos += 1
                nneg += 1
            elif det > 0:
                if a + c > 0:
                    npos += 2
                else:
                    nneg += 2
            else:
                tr = a + c
                nzero += 1
                if tr > 0:
                    npos += 1
                elif tr < 0:
                    nneg += 1
                else:
                    nzero += 1
            k += 2
        else:
            v = float(np.real(d[k]))
            if v > 0:
                npos += 1
            elif v < 0:
                nneg += 1
            else:
                nzero += 1
            k += 1
    return npos, nneg, nzero
