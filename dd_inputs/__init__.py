"""Seeded synthetic inputs shaped like the paper's 3D DD auxiliary matrices.

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle (`oracle/`).  It holds no arithmetic of the method (no factorization, no
solve): it only draws random numbers and builds the input matrix the paper's
pipeline would hand to the auxiliary-problem solver.

What is synthesised (BASELINE.json `configs[0..4]`, DESIGN.md
"Input recipe"):

* A box grid of nx*ny*nz subdomains; an *interface* is an unordered pair {p<q}
  of touching subdomains (face pairs; for config 2 also edge/corner pairs),
  subdomain id p = x + nx*(y + ny*z), interface ids sorted by (p, q)
  (SURVEY.md ledger L13).  Interface I carries s_I dual DoFs.
* Each subdomain p contributes one dense symmetric clique
  S_p = G^T diag(d) G + sigma*I over the concatenated DoFs of the interfaces it
  touches (ascending interface id), G square N(0,1) (ledger L11),
  d = +-U(0.5, 2) (complex: + i*U(0, 0.1)), sigma = 0.1 (complex 0.1+0.05i),
  plain transpose (complex *symmetric*, never Hermitian), then symmetrised
  (S + S^T)/2 (ledger L12) and accumulated additively into the lower blocks.
  This is the "sparse collection of dense blocks" of PAPER.md:29 (§II): one
  dense clique per subdomain, as the primal elimination of PAPER.md:27 would
  produce.
* Right-hand sides B (n x nrhs) with N(0,1) entries (complex: re and im).

Two random back-ends with the same recipe:
  backend="numpy": numpy.random.default_rng(seed) (PCG64), draw order per
      subdomain ascending: G (re, then im), sign, mag, (im_d); then B.
  backend="torch": a torch.Generator on the target device (used only for the
      full-size bench configs where numpy would take minutes); same recipe,
      different stream of numbers.  Both sides of any parity comparison always
      receive the very same bytes.
"""
from __future__ import annotations

import dataclasses
import itertools
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

__all__ = ["Problem", "grid_interfaces", "build_problem", "build_clique_buffer", "config", "config_cliques",
           "CONFIGS", "random_rhs",
           "dense_expand", "block_pattern_from_cliques", "tie_block", "single_block_problem"]


@dataclasses.dataclass
class Problem:
    """Block-sparse symmetric matrix in the C-ABI input format.

    blk_size[nblk]      int64, interface sizes s_I
    colptr[nblk+1]      int64, block-CSC column pointers of the LOWER pattern
    rowidx[nnzb]        int32, row block ids (sorted, >= column, diagonal first)
    values              1-D float64 / complex128: all blocks concatenated, block p
                        (CSC position) is column-major s_row x s_col at val_offset[p]
    val_offset[nnzb]    int64 element offsets
    cliques             list of (subdomain id, interface ids) -- provenance only
    """
    blk_size: np.ndarray
    colptr: np.ndarray
    rowidx: np.ndarray
    values: np.ndarray
    val_offset: np.ndarray
    cliques: List[Tuple[int, List[int]]]
    name: str = ""

    @property
    def nblk(self) -> int:
        return int(self.blk_size.shape[0])

    @property
    def n(self) -> int:
        return int(self.blk_size.sum())

    @property
    def nnzb(self) -> int:
        return int(self.rowidx.shape[0])

    @property
    def is_complex(self) -> bool:
        if self.values is None:  # clique form before assembly (build_clique_buffer)
            return bool(getattr(self, "complex_", False))
        if isinstance(self.values, np.ndarray):
            return np.iscomplexobj(self.values)
        return bool(self.values.is_complex())  # torch tensor (device-resident values)

    @property
    def dof_offset(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.blk_size)]).astype(np.int64)

    def block(self, p: int) -> np.ndarray:
        """Block at CSC position p as an (s_row, s_col) view (column-major storage)."""
        j = int(np.searchsorted(self.colptr, p, side="right") - 1)
        i = int(self.rowidx[p])
        si, sj = int(self.blk_size[i]), int(self.blk_size[j])
        off = int(self.val_offset[p])
        return self.values[off:off + si * sj].reshape(sj, si).T

    def blocks(self) -> Dict[Tuple[int, int], np.ndarray]:
        out = {}
        for j in range(self.nblk):
            for p in range(int(self.colptr[j]), int(self.colptr[j + 1])):
                out[(int(self.rowidx[p]), j)] = self.block(p)
        return out


# --------------------------------------------------------------------------- topology
def _sid(x, y, z, nx, ny):
    return x + nx * (y + ny * z)


def grid_interfaces(nx: int, ny: int, nz: int) -> List[Tuple[int, int]]:
    """Face-adjacent subdomain pairs (p<q), sorted by (p, q) (ledger L13)."""
    pairs = []
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                p = _sid(x, y, z, nx, ny)
                if x + 1 < nx:
                    pairs.append((p, _sid(x + 1, y, z, nx, ny)))
                if y + 1 < ny:
                    pairs.append((p, _sid(x, y + 1, z, nx, ny)))
                if z + 1 < nz:
                    pairs.append((p, _sid(x, y, z + 1, nx, ny)))
    return sorted(pairs)


def _edge_corner_pairs(nx, ny, nz):
    out = []
    for z, y, x in itertools.product(range(nz), range(ny), range(nx)):
        p = _sid(x, y, z, nx, ny)
        for dx, dy, dz in itertools.product((-1, 0, 1), repeat=3):
            if abs(dx) + abs(dy) + abs(dz) < 2:
                continue
            X, Y, Z = x + dx, y + dy, z + dz
            if 0 <= X < nx and 0 <= Y < ny and 0 <= Z < nz:
                q = _sid(X, Y, Z, nx, ny)
                if p < q:
                    out.append((p, q))
    return sorted(out)


def unstructured_interfaces(nx, ny, nz, rng: np.random.Generator, drop=0.3, dmin=4, dmax=14):
    """Config 2 topology, reading L9.

    Drop 30% of face pairs at random; each subdomain draws a target degree
    t_p ~ U{dmin..dmax}; shuffled edge/corner pairs are added while both ends are
    below target; then a fix-up pass adds pairs (faces first) until every
    subdomain touches >= dmin interfaces.
    """
    nsub = nx * ny * nz
    faces = grid_interfaces(nx, ny, nz)
    keep = rng.random(len(faces)) >= drop
    pairs = {f for f, k in zip(faces, keep) if k}
    target = rng.integers(dmin, dmax + 1, nsub)
    deg = np.zeros(nsub, dtype=np.int64)
    for p, q in pairs:
        deg[p] += 1
        deg[q] += 1
    cand = _edge_corner_pairs(nx, ny, nz)
    order = rng.permutation(len(cand))
    for t in order:
        p, q = cand[t]
        if deg[p] < target[p] and deg[q] < target[q] and deg[p] < dmax and deg[q] < dmax:
            pairs.add((p, q))
            deg[p] += 1
            deg[q] += 1
    # fix-up: every subdomain touches >= dmin interfaces
    allc = [f for f in faces if f not in pairs] + [c for c in cand if c not in pairs]
    for p in range(nsub):
        for (a, b) in allc:
            if deg[p] >= dmin:
                break
            if p in (a, b) and (a, b) not in pairs and deg[a] < dmax and deg[b] < dmax:
                pairs.add((a, b))
                deg[a] += 1
                deg[b] += 1
    return sorted(pairs)


def block_pattern_from_cliques(nblk: int, cliques: Sequence[Sequence[int]]):
    """Lower block pattern = diagonal + union of clique pairs (block-CSC)."""
    cols: List[set] = [{j} for j in range(nblk)]
    for members in cliques:
        ms = sorted(members)
        for a in range(len(ms)):
            for b in range(a + 1, len(ms)):
                cols[ms[a]].add(ms[b])
    colptr = np.zeros(nblk + 1, dtype=np.int64)
    rows = []
    for j in range(nblk):
        r = sorted(cols[j])
        rows.extend(r)
        colptr[j + 1] = colptr[j] + len(r)
    return colptr, np.asarray(rows, dtype=np.int32)


# --------------------------------------------------------------------------- values
def _layout(blk_size, colptr, rowidx):
    nnzb = len(rowidx)
    off = np.zeros(nnzb, dtype=np.int64)
    tot = 0
    for j in range(len(blk_size)):
        for p in range(int(colptr[j]), int(colptr[j + 1])):
            off[p] = tot
            tot += int(blk_size[rowidx[p]]) * int(blk_size[j])
    return off, tot


def _topology(nx, ny, nz, sizes_fn, rng, topology):
    """Interfaces, sizes, cliques, lower block pattern and value layout (no values)."""
    if topology == "faces":
        pairs = grid_interfaces(nx, ny, nz)
    else:
        pairs = unstructured_interfaces(nx, ny, nz, rng)
    nblk = len(pairs)
    blk_size = np.asarray(sizes_fn(nblk, rng), dtype=np.int64)
    nsub = nx * ny * nz
    touch: List[List[int]] = [[] for _ in range(nsub)]
    for I, (p, q) in enumerate(pairs):
        touch[p].append(I)
        touch[q].append(I)
    cliques = [(p, sorted(touch[p])) for p in range(nsub) if touch[p]]
    colptr, rowidx = block_pattern_from_cliques(nblk, [c for _, c in cliques])
    val_offset, total = _layout(blk_size, colptr, rowidx)
    return pairs, blk_size, cliques, colptr, rowidx, val_offset, total


def _clique_draw(m, complex_, rng=None, gen=None, device="cpu"):
    """One subdomain's raw dense contribution S_p = G^T diag(d) G + sigma*I (before the
    symmetrisation of ledger L12); numpy (rng) or torch (gen) draws, recipe in the module doc."""
    sigma = (0.1 + 0.05j) if complex_ else 0.1
    if rng is not None:
        G = rng.standard_normal((m, m))
        if complex_:
            G = G + 1j * rng.standard_normal((m, m))
        sign = 2.0 * rng.integers(0, 2, m) - 1.0
        mag = rng.uniform(0.5, 2.0, m)
        d = sign * mag
        if complex_:
            d = d + 1j * rng.uniform(0.0, 0.1, m)
        S = G.T @ (d[:, None] * G)
        return S + sigma * np.eye(m)
    import torch
    tdt = torch.complex128 if complex_ else torch.float64
    G = torch.randn(m, m, generator=gen, device=device, dtype=torch.float64)
    if complex_:
        G = torch.complex(G, torch.randn(m, m, generator=gen, device=device, dtype=torch.float64))
    sign = 2.0 * torch.randint(0, 2, (m,), generator=gen, device=device).double() - 1.0
    mag = 0.5 + 1.5 * torch.rand(m, generator=gen, device=device, dtype=torch.float64)
    d = (sign * mag).to(tdt)
    if complex_:
        d = d + 1j * (0.1 * torch.rand(m, generator=gen, device=device, dtype=torch.float64))
    S = G.transpose(0, 1) @ (d[:, None] * G)
    return S + sigma * torch.eye(m, dtype=tdt, device=device)


def build_problem(nx, ny, nz, sizes_fn, *, complex_=False, seed=0, topology="faces",
                  backend="numpy", device="cpu", name="", keep_cliques=False) -> Problem:
    """Build the auxiliary matrix of a grid DD model (recipe in the module doc).

    sizes_fn(n_interfaces, rng) -> int array of interface sizes.
    backend "numpy" draws with default_rng(seed); "torch" with a torch.Generator
    on `device` (values then stay on that device as a torch tensor).
    keep_cliques (numpy only): also keep the raw per-clique matrices S_p in
    prob.clique_S (list, clique order), the input of the f1 assembly.
    """
    rng = np.random.default_rng(seed)
    pairs, blk_size, cliques, colptr, rowidx, val_offset, total = _topology(nx, ny, nz, sizes_fn, rng, topology)
    nblk = len(pairs)
    dtype = np.complex128 if complex_ else np.float64
    if backend == "torch":
        import torch
        values = torch.zeros(total, dtype=torch.complex128 if complex_ else torch.float64, device=device)
        gen = torch.Generator(device=device)
        gen.manual_seed(seed)
    else:
        values = np.zeros(total, dtype=dtype)
    pos = {}
    for j in range(nblk):
        for p in range(int(colptr[j]), int(colptr[j + 1])):
            pos[(int(rowidx[p]), j)] = p
    kept = []
    for p_sub, members in cliques:
        m = int(sum(blk_size[I] for I in members))
        if backend == "numpy":
            S = _clique_draw(m, complex_, rng=rng)
            if keep_cliques:
                kept.append(S)
            S = 0.5 * (S + S.T)
        else:
            import torch
            S = _clique_draw(m, complex_, gen=gen, device=device)
            S = 0.5 * (S + S.transpose(0, 1))
        offs = np.concatenate([[0], np.cumsum([blk_size[I] for I in members])])
        if backend == "torch":
            # one scatter per clique: destination offset of every (row, col) of S whose block
            # (I, J) has I >= J (a clique never repeats an interface, so indices are unique)
            import torch
            rows, cols = [], []
            for a, I in enumerate(members):
                for b, J in enumerate(members):
                    if I < J:
                        continue
                    si, sj = int(blk_size[I]), int(blk_size[J])
                    base = int(val_offset[pos[(I, J)]])
                    r = np.arange(si)
                    c = np.arange(sj)
                    rows.append((offs[a] + r[:, None] + 0 * c[None, :]).ravel())
                    cols.append((offs[b] + c[None, :] + 0 * r[:, None]).ravel())
                    rows[-1] = np.stack([rows[-1], (base + r[:, None] + c[None, :] * si).ravel()])
            src_r = np.concatenate([x[0] for x in rows])
            dst = np.concatenate([x[1] for x in rows])
            src_c = np.concatenate(cols)
            sr = torch.from_numpy(src_r).to(S.device)
            sc = torch.from_numpy(src_c).to(S.device)
            values.index_add_(0, torch.from_numpy(dst).to(S.device), S[sr, sc])
            continue
        for a, I in enumerate(members):
            for b, J in enumerate(members):
                if I < J:
                    continue
                blk = S[offs[a]:offs[a + 1], offs[b]:offs[b + 1]]
                pp = pos[(I, J)]
                si, sj = int(blk_size[I]), int(blk_size[J])
                dst = values[val_offset[pp]:val_offset[pp] + si * sj].reshape(sj, si).T
                dst += blk
    prob = Problem(blk_size, colptr, rowidx, values, val_offset, cliques, name)
    prob.pairs = pairs
    prob.grid = (nx, ny, nz)
    if keep_cliques:
        prob.clique_S = kept
    return prob


def build_clique_buffer(nx, ny, nz, sizes_fn, *, complex_=False, seed=0, topology="faces", device="cuda",
                        name=""):
    """Clique form of the same workload for the f1 assembly bench (torch draws on `device`).

    Returns (prob, S, S_offset): prob carries the pattern and value layout (values=None);
    S is one 1-D device tensor holding every raw S_p column-major (ld = m_p) at element
    offset S_offset[p], clique order.  The draws are those of build_problem(backend="torch"),
    so assembling with symmetrisation reproduces its values.
    """
    import torch
    rng = np.random.default_rng(seed)
    pairs, blk_size, cliques, colptr, rowidx, val_offset, total = _topology(nx, ny, nz, sizes_fn, rng, topology)
    ms = [int(sum(blk_size[I] for I in members)) for _, members in cliques]
    S_offset = np.concatenate([[0], np.cumsum([m * m for m in ms])]).astype(np.int64)
    tdt = torch.complex128 if complex_ else torch.float64
    S = torch.empty(int(S_offset[-1]), dtype=tdt, device=device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    for q, m in enumerate(ms):
        Sp = _clique_draw(m, complex_, gen=gen, device=device)
        # column-major m x m == row-major transpose
        S[int(S_offset[q]):int(S_offset[q]) + m * m].copy_(Sp.transpose(0, 1).reshape(-1))
        del Sp
    prob = Problem(blk_size, colptr, rowidx, None, val_offset, cliques, name)
    prob.pairs = pairs
    prob.grid = (nx, ny, nz)
    prob.total = total
    prob.complex_ = bool(complex_)
    return prob, S, S_offset[:-1]


def corner_interfaces(prob: Problem, sub_grid) -> List[int]:
    """Interfaces whose two subdomains both lie in the corner sub-grid [0,gx)x[0,gy)x[0,gz)."""
    nx, ny, _ = prob.grid
    gx, gy, gz = sub_grid

    def inside(p):
        x, y, z = p % nx, (p // nx) % ny, p // (nx * ny)
        return x < gx and y < gy and z < gz

    return [I for I, (p, q) in enumerate(prob.pairs) if inside(p) and inside(q)]


def subproblem(prob: Problem, keep) -> Problem:
    """Principal sub-matrix on the interface subset `keep` (renumbered ascending), host numpy values.

    Used only to carve a BOUNDED sample of a large workload for the CPU oracle timing
    (bench.py cpu_baseline); pure data movement.
    """
    keep = sorted(int(k) for k in keep)
    new = {old: i for i, old in enumerate(keep)}
    blocks = []
    for j in keep:
        for p in range(int(prob.colptr[j]), int(prob.colptr[j + 1])):
            i = int(prob.rowidx[p])
            if i in new:
                blocks.append((new[j], new[i], p))
    blocks.sort()
    nb = len(keep)
    sizes = np.asarray([prob.blk_size[k] for k in keep], dtype=np.int64)
    colptr = np.zeros(nb + 1, dtype=np.int64)
    rowidx = np.zeros(len(blocks), dtype=np.int32)
    offs = np.zeros(len(blocks), dtype=np.int64)
    chunks = []
    tot = 0
    for q, (jn, in_, p) in enumerate(blocks):
        colptr[jn + 1] += 1
        rowidx[q] = in_
        offs[q] = tot
        ln = int(prob.blk_size[prob.rowidx[p]]) * int(prob.blk_size[keep[jn]])
        seg = prob.values[int(prob.val_offset[p]):int(prob.val_offset[p]) + ln]
        chunks.append(seg if isinstance(seg, np.ndarray) else seg.cpu().numpy())
        tot += ln
    colptr = np.cumsum(colptr)
    vals = np.concatenate(chunks) if chunks else np.zeros(0)
    return Problem(sizes, colptr, rowidx, vals, offs, [], prob.name + "-sample")


def random_rhs(n: int, nrhs: int, complex_: bool, seed: int) -> np.ndarray:
    """N(0,1) right-hand sides, (n, nrhs) Fortran-ordered (column-major)."""
    rng = np.random.default_rng([seed, 7919])
    B = rng.standard_normal((n, nrhs))
    if complex_:
        B = B + 1j * rng.standard_normal((n, nrhs))
    return np.asfortranarray(B)


def dense_expand(prob: Problem) -> np.ndarray:
    """The full symmetric n x n matrix the blocks define (A^T = A, no conjugation).

    Only the lower triangle of each diagonal block is used, as the C ABI states.
    """
    n = prob.n
    off = prob.dof_offset
    A = np.zeros((n, n), dtype=prob.values.dtype)
    for (i, j), blk in prob.blocks().items():
        if i == j:
            lo = np.tril(blk)
            A[off[i]:off[i + 1], off[j]:off[j + 1]] = lo + np.tril(blk, -1).T
        else:
            A[off[i]:off[i + 1], off[j]:off[j + 1]] = blk
            A[off[j]:off[j + 1], off[i]:off[i + 1]] = blk.T
    return A


def tie_block(s: int, seed: int = 0) -> np.ndarray:
    """Integer-valued symmetric s x s block with many exact IDAMAX ties (reading L3 tests).

    The block is a random interleaving of small decoupled groups whose local matrices are
        T1 = [[0, s1, s2], [s1, 0, 0], [s2, 0, c]]                  c in {+-1, +-2, +-4}
        T2 = [[1, 2 s1, 2 s2], [2 s1, 4, 0], [2 s2, 0, c]]          c in {+-1, +-2, +-4}
        T0 = [[c]]                                                    (filler, c = +-1)
    with random signs s1, s2 = +-1.  The first column of T1 / T2 has two entries of equal
    magnitude (a tie the smallest-index rule must break), and every entry is a small integer
    chosen so that the pivots that occur are +-1, +-2, +-4 or the 2x2 [[0, x], [x, y]] with
    x = +-1, +-2: every value a Bunch-Kaufman factorization produces is then a short dyadic
    rational, i.e. exact in binary64 in any evaluation order.  Pure data construction.
    """
    rng = np.random.default_rng([seed, 4242])
    A = np.zeros((s, s))
    posn = rng.permutation(s)
    q = 0
    while q < s:
        left = s - q
        kind = 0 if left < 3 else int(rng.integers(0, 3))
        if kind == 0:
            p0 = int(posn[q])
            A[p0, p0] = float(rng.choice([-1.0, 1.0]))
            q += 1
            continue
        loc = np.sort(posn[q:q + 3])
        q += 3
        s1, s2 = (float(v) for v in rng.choice([-1.0, 1.0], 2))
        c = float(rng.choice([-4.0, -2.0, -1.0, 1.0, 2.0, 4.0]))
        if kind == 1:
            M = np.array([[0.0, s1, s2], [s1, 0.0, 0.0], [s2, 0.0, c]])
        else:
            M = np.array([[1.0, 2 * s1, 2 * s2], [2 * s1, 4.0, 0.0], [2 * s2, 0.0, c]])
        A[np.ix_(loc, loc)] = M
    return A


def single_block_problem(A: np.ndarray) -> Problem:
    """One interface whose diagonal block is the dense symmetric A (C-ABI input layout)."""
    A = np.asarray(A)
    n = A.shape[0]
    return Problem(np.array([n], dtype=np.int64), np.array([0, 1], dtype=np.int64), np.array([0], dtype=np.int32),
                   np.asfortranarray(A).ravel(order="F"), np.array([0], dtype=np.int64), [])


# --------------------------------------------------------------------------- configs
def _const(s):
    return lambda n, rng: np.full(n, s, dtype=np.int64)


def _uniform(lo, hi):
    return lambda n, rng: rng.integers(lo, hi + 1, n)


# name -> (grid, sizes, complex, topology, nrhs, order)   (BASELINE.json configs[i])
CONFIGS = {
    "cfg0": dict(grid=(2, 2, 1), sizes=_const(32), complex_=False, topology="faces", nrhs=4, order="auto"),
    "cfg1": dict(grid=(4, 4, 4), sizes=_const(256), complex_=False, topology="faces", nrhs=64, order="nd"),
    "cfg2": dict(grid=(6, 6, 6), sizes=_uniform(128, 1024), complex_=False, topology="unstructured", nrhs=256,
                 order="auto"),
    "cfg3": dict(grid=(8, 8, 4), sizes=_const(512), complex_=True, topology="faces", nrhs=1000, order="auto"),
    "cfg3alt": dict(grid=(3, 6, 10), sizes=_const(512), complex_=True, topology="faces", nrhs=1000, order="auto"),
    "cfg4": dict(grid=(8, 8, 4), sizes=_const(512), complex_=True, topology="faces", nrhs=1000, order="auto",
                 batches=10),
}


def config(name: str, *, seed: int = 0, backend: str = "numpy", device: str = "cpu",
           grid: Optional[Tuple[int, int, int]] = None, sizes=None, keep_cliques=False) -> Problem:
    """Problem for a named BASELINE config; `grid`/`sizes` override for scaled-down variants."""
    c = CONFIGS[name]
    g = grid or c["grid"]
    sz = c["sizes"] if sizes is None else (sizes if callable(sizes) else _const(int(sizes)))
    return build_problem(*g, sz, complex_=c["complex_"], seed=seed, topology=c["topology"],
                         backend=backend, device=device, name=name, keep_cliques=keep_cliques)


def config_cliques(name: str, *, seed: int = 0, device: str = "cuda"):
    """Clique form (prob without values, S buffer, S offsets) of a named config (torch draws)."""
    c = CONFIGS[name]
    return build_clique_buffer(*c["grid"], c["sizes"], complex_=c["complex_"], seed=seed, topology=c["topology"],
                               device=device, name=name)
