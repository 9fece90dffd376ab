"""Seeded FEM-like domain-decomposition model for the rows f2/f3.

PAPER.md:27 (§II): the decomposed BVP, discretised "in terms of primal degrees-of-freedom (DoFs)
in domain volumes and dual DoF on domain interfaces leads to a large sparse arrowhead matrix that
is then reduced in size by eliminating via many independent sparse direct factorizations the
primal DoFs"; afterwards "the solution of all or a subset of primal unknowns are
recovered ... via many smaller size sparse forward backward substitutions".  The paper's mixed/
hybrid formulation (its refs [moshfegh2016, 2017]) is not in PAPER.md, so this module builds a
synthetic arrowhead system with that structure (f2/f3):

    [ K_1            C_1 ] [x_1]   [f_1]
    [      ...       ... ] [...] = [...]            A_bb = sum_p A_bb,p
    [           K_P  C_P ] [x_P]   [f_P]
    [ C_1^T ... C_P^T A_bb] [x_b]   [b_b]

* A box grid of nx*ny*nz subdomains (ids p = x + nx*(y + ny*z)), each an a*a*a grid of primal
  nodes.  K_p is a 7-point "Helmholtz-like" operator: a graph Laplacian with random edge weights
  U(0.5, 1.5) minus kappa^2 * diag(m), m ~ U(0.5, 1.5), kappa^2 = 0.1 -- symmetric indefinite,
  like a CEM operator above its lowest resonances; complex: kappa^2 (1 + 0.05i) (a lossy medium,
  complex SYMMETRIC).
* Interfaces = face-adjacent subdomain pairs {p < q} (ids sorted, as dd_inputs.grid_interfaces),
  each carrying (a-2)^2 dual DoFs, one per face-interior node of the shared face (edge and corner
  nodes carry none, so no cross points).  C_p maps the face nodes of p to the dual DoFs, with
  sign +1 on the lower subdomain of the pair and -1 on the upper (a FETI-style jump).
* A_bb,p = (sigma_b / 2) I on every dual DoF of p's interfaces (sigma_b = 0.1, complex
  0.1 + 0.05i), so A_bb = sigma_b I.
* f ~ N(0,1) per primal DoF, b_b ~ N(0,1) per dual DoF (complex: re and im).

Only data construction lives here (no factorization, no solve): the sparse K_p / C_p, and the
same system laid out as the library's block-sparse input for the partial factorization -- the
primal nodes of each subdomain grouped into blocks by a geometric nested dissection of its box
(the ordering input, the role MeTiS plays in the paper), followed by one kept
(Schur) block per (subdomain, interface) pair.  All random draws use numpy default_rng(seed).
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import numpy as np
import scipy.sparse as sp

from . import Problem, grid_interfaces

KAPPA2 = 0.1
SIGMA_B = 0.1


def _nid(i, j, k, a):
    return i + a * (j + a * k)


def box_nd(a: int, leaf: int = 64):
    """Geometric nested dissection of an a^3 node box: recursively cut the longest side at its
    middle plane; leaves have <= leaf nodes.  Returns the blocks (arrays of local node ids) in
    postorder (both halves, then their separator)."""
    out: List[np.ndarray] = []

    def rec(lo, hi):
        dims = [hi[d] - lo[d] for d in range(3)]
        n = dims[0] * dims[1] * dims[2]
        if n == 0:
            return
        d = int(np.argmax(dims))
        if n <= leaf or dims[d] < 3:
            ii, jj, kk = np.meshgrid(np.arange(lo[0], hi[0]), np.arange(lo[1], hi[1]), np.arange(lo[2], hi[2]),
                                     indexing="ij")
            out.append(np.sort(_nid(ii, jj, kk, a).ravel()))
            return
        mid = (lo[d] + hi[d]) // 2
        h1 = list(hi)
        h1[d] = mid
        l2 = list(lo)
        l2[d] = mid + 1
        rec(lo, h1)
        rec(l2, hi)
        ls, hs = list(lo), list(hi)
        ls[d], hs[d] = mid, mid + 1
        rec(ls, hs)

    rec([0, 0, 0], [a, a, a])
    return out


def _laplacian_pattern(a):
    """Edges (i < j) of the 7-point stencil on the a^3 box."""
    e = []
    idx = np.arange(a ** 3).reshape(a, a, a).transpose(2, 1, 0)  # idx[i, j, k] = i + a(j + a k)
    e.append(np.stack([idx[:-1, :, :].ravel(), idx[1:, :, :].ravel()], 1))
    e.append(np.stack([idx[:, :-1, :].ravel(), idx[:, 1:, :].ravel()], 1))
    e.append(np.stack([idx[:, :, :-1].ravel(), idx[:, :, 1:].ravel()], 1))
    return np.concatenate(e)


def _face_nodes(a, axis, side):
    """Face-interior nodes of one face of the box, in a fixed order (the dual DoF order)."""
    r = np.arange(1, a - 1)
    u, v = np.meshgrid(r, r, indexing="ij")
    c = np.full(u.shape, 0 if side == 0 else a - 1)
    if axis == 0:
        ijk = (c, u, v)
    elif axis == 1:
        ijk = (u, c, v)
    else:
        ijk = (u, v, c)
    return _nid(ijk[0], ijk[1], ijk[2], a).ravel()


@dataclasses.dataclass
class FEMDD:
    grid: Tuple[int, int, int]
    a: int
    complex_: bool
    pairs: List[Tuple[int, int]]          # interfaces (p, q), p < q
    sub_ifaces: List[List[int]]            # interfaces of each subdomain, ascending
    K: List[sp.csr_matrix]                 # K_p (n_p x n_p)
    C: List[sp.csr_matrix]                 # C_p (n_p x m_p), columns = p's interfaces' duals concatenated
    Abb_diag: np.ndarray                   # sum_p A_bb,p diagonal, per global dual DoF
    f: List[np.ndarray]                    # primal right-hand sides (n_p x nrhs)
    bb: np.ndarray                         # dual right-hand sides (n_b x nrhs)
    s_dual: int                            # dual DoFs per interface

    @property
    def nsub(self):
        return len(self.K)

    @property
    def n_dual(self):
        return len(self.pairs) * self.s_dual

    def dual_offset(self, I):
        return I * self.s_dual


def fem_dd(nx, ny, nz, a, *, complex_=False, seed=0, nrhs=4) -> FEMDD:
    """Draw the model (module doc).  Per subdomain p ascending: edge weights, masses, then the
    right-hand sides f_p; finally b_b."""
    assert a >= 4
    rng = np.random.default_rng([seed, 2002, 5019])
    pairs = grid_interfaces(nx, ny, nz)
    nsub = nx * ny * nz
    sub_if: List[List[int]] = [[] for _ in range(nsub)]
    for I, (p, q) in enumerate(pairs):
        sub_if[p].append(I)
        sub_if[q].append(I)
    edges = _laplacian_pattern(a)
    n_p = a ** 3
    sd = (a - 2) ** 2
    dt = np.complex128 if complex_ else np.float64
    k2 = KAPPA2 * ((1 + 0.05j) if complex_ else 1.0)
    Ks, Cs, fs = [], [], []
    for p in range(nsub):
        w = rng.uniform(0.5, 1.5, len(edges))
        m = rng.uniform(0.5, 1.5, n_p)
        diag = np.zeros(n_p)
        np.add.at(diag, edges[:, 0], w)
        np.add.at(diag, edges[:, 1], w)
        rows = np.concatenate([edges[:, 0], edges[:, 1], np.arange(n_p)])
        cols = np.concatenate([edges[:, 1], edges[:, 0], np.arange(n_p)])
        vals = np.concatenate([-w, -w, diag - k2 * m]).astype(dt)
        Ks.append(sp.csr_matrix((vals, (rows, cols)), shape=(n_p, n_p)))
        x, y, z = p % nx, (p // nx) % ny, p // (nx * ny)
        cr, cc, cv = [], [], []
        for t, I in enumerate(sub_if[p]):
            P, Q = pairs[I]
            other = Q if P == p else P
            ox, oy, oz = other % nx, (other // nx) % ny, other // (nx * ny)
            axis = 0 if ox != x else (1 if oy != y else 2)
            side = 1 if (ox > x or oy > y or oz > z) else 0
            nodes = _face_nodes(a, axis, side)
            cr.append(nodes)
            cc.append(t * sd + np.arange(sd))
            cv.append(np.full(sd, 1.0 if P == p else -1.0))
        mp = sd * len(sub_if[p])
        if mp:
            Cs.append(sp.csr_matrix((np.concatenate(cv).astype(dt), (np.concatenate(cr), np.concatenate(cc))),
                                    shape=(n_p, mp)))
        else:
            Cs.append(sp.csr_matrix((n_p, 0), dtype=dt))
        F = rng.standard_normal((n_p, nrhs))
        if complex_:
            F = F + 1j * rng.standard_normal((n_p, nrhs))
        fs.append(np.asfortranarray(F))
    nb = len(pairs) * sd
    bb = rng.standard_normal((nb, nrhs))
    if complex_:
        bb = bb + 1j * rng.standard_normal((nb, nrhs))
    sigma = (SIGMA_B + 0.05j) if complex_ else SIGMA_B
    return FEMDD((nx, ny, nz), a, complex_, pairs, sub_if, Ks, Cs, np.full(nb, sigma, dtype=dt), fs,
                 np.asfortranarray(bb), sd)


def abb_share(m: FEMDD, p: int) -> np.ndarray:
    """Diagonal of A_bb,p over p's dual DoFs (half of sigma_b on each side of an interface)."""
    sigma = (SIGMA_B + 0.05j) if m.complex_ else SIGMA_B
    return np.full(len(m.sub_ifaces[p]) * m.s_dual, sigma / 2, dtype=np.complex128 if m.complex_ else np.float64)


def arrowhead(m: FEMDD) -> sp.csr_matrix:
    """The global sparse arrowhead matrix [K C; C^T A_bb] (primal of p ascending, then duals)."""
    nsub = m.nsub
    n_p = m.a ** 3
    blocks = [[None] * (nsub + 1) for _ in range(nsub + 1)]
    nb = m.n_dual
    for p in range(nsub):
        blocks[p][p] = m.K[p]
        # C_p columns -> global dual columns
        cols = np.concatenate([m.dual_offset(I) + np.arange(m.s_dual) for I in m.sub_ifaces[p]]) \
            if m.sub_ifaces[p] else np.zeros(0, dtype=np.int64)
        Cg = sp.csr_matrix((m.C[p].shape[0], nb), dtype=m.K[p].dtype)
        if len(cols):
            coo = m.C[p].tocoo()
            Cg = sp.csr_matrix((coo.data, (coo.row, cols[coo.col])), shape=(n_p, nb))
        blocks[p][nsub] = Cg
        blocks[nsub][p] = Cg.T.tocsr()
    blocks[nsub][nsub] = sp.diags(m.Abb_diag)
    return sp.bmat(blocks, format="csr")


def arrowhead_rhs(m: FEMDD) -> np.ndarray:
    return np.concatenate(m.f + [m.bb])


def schur_block_problem(m: FEMDD, leaf: int = 64):
    """The system laid out for the library's partial (Schur-mode) block LDL^T (include/dd_aux.h
    dd_aux_analyze_partial): returns (prob, n_schur, schur_target, schur_group, aux_sizes, info).

    Block ids: for p ascending, the box-ND blocks of subdomain p (postorder); then the kept blocks,
    one per (p, interface I of p), p ascending then I ascending.  schur_target[k] = I,
    schur_group[k] = p for kept block k (0-based among the kept).  prob.values holds every
    structurally nonzero block densely (column-major; diagonal blocks full), the kept diagonal
    blocks are A_bb,p, the kept-primal blocks are C_p^T restricted to the block's nodes.
    info["sub_dof"][p] = (first DoF of p's primal blocks, n_p) in the handle's DoF numbering, and
    info["kept_dof"][k] = first DoF of kept block k."""
    a = m.a
    n_p = a ** 3
    nds = box_nd(a, leaf)
    nblk_p = len(nds)
    node_blk = np.empty(n_p, dtype=np.int64)
    node_loc = np.empty(n_p, dtype=np.int64)
    for b, nodes in enumerate(nds):
        node_blk[nodes] = b
        node_loc[nodes] = np.arange(len(nodes))
    sizes_p = np.array([len(x) for x in nds], dtype=np.int64)
    edges = _laplacian_pattern(a)
    bpairs = set()
    for u, v in edges:
        bu, bv = node_blk[u], node_blk[v]
        if bu != bv:
            bpairs.add((max(bu, bv), min(bu, bv)))
    nsub = m.nsub
    kept = [(p, I) for p in range(nsub) for I in m.sub_ifaces[p]]
    n_schur = len(kept)
    nblk = nsub * nblk_p + n_schur
    sizes = np.concatenate([np.tile(sizes_p, nsub), np.full(n_schur, m.s_dual, dtype=np.int64)])
    cols: List[set] = [set([j]) for j in range(nblk)]
    for p in range(nsub):
        base = p * nblk_p
        for (bi, bj) in bpairs:
            cols[base + bj].add(base + bi)
    # kept (p, I): coupled to every primal block holding one of the face nodes of I
    kid = {}
    for k, (p, I) in enumerate(kept):
        kid[(p, I)] = nsub * nblk_p + k
    face = {}
    for k, (p, I) in enumerate(kept):
        t = m.sub_ifaces[p].index(I)
        coo = m.C[p][:, t * m.s_dual:(t + 1) * m.s_dual].tocoo()
        o = np.argsort(coo.col)
        face[k] = (coo.row[o], coo.data[o])   # node and sign of dual DoF d = 0..s_dual-1
        for b in np.unique(node_blk[coo.row]):
            cols[p * nblk_p + int(b)].add(kid[(p, I)])
    colptr = np.zeros(nblk + 1, dtype=np.int64)
    rowidx = []
    for j in range(nblk):
        r = sorted(cols[j])
        rowidx.extend(r)
        colptr[j + 1] = colptr[j] + len(r)
    rowidx = np.asarray(rowidx, dtype=np.int32)
    pos = {}
    val_offset = np.zeros(len(rowidx), dtype=np.int64)
    tot = 0
    for j in range(nblk):
        for q in range(colptr[j], colptr[j + 1]):
            i = int(rowidx[q])
            pos[(i, j)] = q
            val_offset[q] = tot
            tot += int(sizes[i]) * int(sizes[j])
    dt = np.complex128 if m.complex_ else np.float64
    vals = np.zeros(tot, dtype=dt)
    for p in range(nsub):
        base = p * nblk_p
        qtab = np.full((nblk_p, nblk_p), -1, dtype=np.int64)
        for bj in range(nblk_p):
            for q in range(colptr[base + bj], colptr[base + bj + 1]):
                bi = int(rowidx[q]) - base
                if bi < nblk_p:
                    qtab[bi, bj] = q
        coo = m.K[p].tocoo()
        r, c, v = coo.row, coo.col, coo.data
        br, bc = node_blk[r], node_blk[c]
        # each entry once, in the lower block (bi > bj) or the lower part of a diagonal block
        sel = (br > bc) | ((br == bc) & (node_loc[r] >= node_loc[c]))
        q = qtab[br[sel], bc[sel]]
        assert (q >= 0).all()
        dest = val_offset[q] + node_loc[r[sel]] + node_loc[c[sel]] * sizes_p[br[sel]]
        vals[dest] = v[sel]
        sh = abb_share(m, p)
        d = np.arange(m.s_dual)
        for t, I in enumerate(m.sub_ifaces[p]):
            kk = kid[(p, I)]
            qd = pos[(kk, kk)]
            vals[val_offset[qd] + d + d * m.s_dual] = sh[t * m.s_dual + d]
            nodes, sign = face[kk - nsub * nblk_p]
            for b in np.unique(node_blk[nodes]):
                selb = node_blk[nodes] == b
                qb = pos[(kk, base + int(b))]
                vals[val_offset[qb] + d[selb] + node_loc[nodes[selb]] * m.s_dual] = sign[selb]
    prob = Problem(sizes, colptr, rowidx, vals, val_offset, [], "fem-dd")
    schur_target = np.asarray([I for (_, I) in kept], dtype=np.int32)
    schur_group = np.asarray([p for (p, _) in kept], dtype=np.int32)
    aux_sizes = np.full(len(m.pairs), m.s_dual, dtype=np.int64)
    off = prob.dof_offset
    info = {"nblk_per_sub": nblk_p, "sub_dof": [(int(off[p * nblk_p]), n_p) for p in range(nsub)],
            "kept_dof": [int(off[nsub * nblk_p + k]) for k in range(n_schur)],
            "node_perm": np.concatenate([nds[b] for b in range(nblk_p)])}
    return prob, n_schur, schur_target, schur_group, aux_sizes, info
