"""Clique assembly of the auxiliary matrix -- oracle (TEST INFRASTRUCTURE ONLY).

PAPER.md:27 (§II): the primal unknowns of every subdomain are eliminated, which leaves a
dense contribution of that subdomain over the dual DoFs of the interfaces it touches;
PAPER.md:29: the auxiliary matrix assembled from them is "symmetric ... block-wise sparse
(sparse collection of dense blocks)", one dense clique per subdomain.  The plain definition
(ledger L12 for the symmetric part):

    A_IJ = sum over cliques p (ascending) with I, J in p of  Ssym_p[rows of I, cols of J],
    Ssym_p = (S_p + S_p^T) / 2   (symmetrize) or S_p,         for every lower block I >= J,

written as the obvious loop; blocks no clique covers stay zero.  Complex matrices are
complex SYMMETRIC: plain transpose, never conjugated.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np


def assemble(blk_size, colptr, rowidx, val_offset, cliques: Sequence[Sequence[int]], S_list, symmetrize=True):
    """Values of every lower block (caller layout: block at CSC position q is column-major
    s_row x s_col at val_offset[q]) from the cliques' dense matrices S_list[p] (DoFs = the
    clique's members concatenated in the listed order)."""
    blk_size = np.asarray(blk_size, dtype=np.int64)
    nblk = len(blk_size)
    pos = {}
    total = 0
    for j in range(nblk):
        for q in range(int(colptr[j]), int(colptr[j + 1])):
            i = int(rowidx[q])
            pos[(i, j)] = q
            total = max(total, int(val_offset[q]) + int(blk_size[i]) * int(blk_size[j]))
    cplx = any(np.iscomplexobj(S) for S in S_list)
    values = np.zeros(total, dtype=np.complex128 if cplx else np.float64)
    for p, members in enumerate(cliques):
        S = np.asarray(S_list[p])
        if symmetrize:
            S = 0.5 * (S + S.T)
        offs = np.concatenate([[0], np.cumsum([blk_size[I] for I in members])])
        for a, I in enumerate(members):
            for b, J in enumerate(members):
                if I < J:
                    continue
                q = pos[(int(I), int(J))]
                si, sj = int(blk_size[I]), int(blk_size[J])
                dst = values[val_offset[q]:val_offset[q] + si * sj].reshape(sj, si).T
                dst += S[offs[a]:offs[a + 1], offs[b]:offs[b + 1]]
    return values
