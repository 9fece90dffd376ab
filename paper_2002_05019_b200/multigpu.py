"""f4: multi-GPU factorization of the auxiliary matrix by subtree-to-GPU mapping.

PAPER.md:8,31,79: the method's "parallel and GPU processing prospects" -- it "attempts to maximize
the concurrency in sparse matrix computations".  SURVEY.md §8(e): independent elimination-tree
subtrees map one per GPU with no communication; their contributions to the shared top separators
must then be summed (one reduce) and the top part factored.  This module is that schedule, built
from the library's own calls (no arithmetic here -- host integer planning and torch.distributed
plumbing only):

  plan (every rank, host, identical):  the global symbolic (dd_aux_analyze, host only) gives the
      block elimination order, the elimination tree and struct(k); a top set T of separators is
      peeled off the forest from the roots down until the remaining subtrees can be dealt onto
      the ranks with a balanced flop count (LPT).  T is ancestor-closed, so every subtree's
      outside neighbours lie in T and form the clique struct(root).
  factor (rank r):  the blocks of its subtrees + the T blocks of their structs, laid out as a
      Schur-mode problem (dd_aux_analyze_partial: the T blocks are kept, zero-valued) -> one
      partial factorization of all its subtrees at once (they are independent: the level
      scheduler batches them) -> dd_aux_schur_export: the dense update S_tau = -sum_{k in tau}
      W L^T of every subtree tau on struct(root tau).
  reduce:  the S_tau of all ranks go to rank 0 (NCCL point-to-point), where dd_aux_assemble_acc
      adds them onto the top matrix's own blocks; rank 0 factors the top matrix (dd_aux_factor).
  solve:  every rank condenses its subtrees' right-hand sides onto T (dd_aux_condense) -> NCCL
      reduce to rank 0 -> top solve (dd_aux_solve, with refinement against the top matrix) ->
      broadcast x_T -> every rank recovers its subtrees' unknowns (dd_aux_recover).

Mathematically this is the same block LDL^T as the one-GPU factorization (same order, same
restricted pivots per block); only the summation order of the top separators' updates differs.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional

import numpy as np

from . import (DD_OK, DD_ORDER_AUTO, DD_ORDER_NATURAL, DD_REAL64, AuxSolver, SchurSolver, cliques_to_csr,
               dd_aux_analyze, dd_aux_assemble_acc, dd_aux_assemble_work_bytes, dd_aux_default_options,
               dd_aux_destroy, dd_aux_get_etree, dd_aux_get_order, dd_aux_get_struct, dd_aux_residual,
               dd_aux_solve_work_bytes)


@dataclasses.dataclass
class PartPlan:
    """Rank-local Schur-mode problem: local block l < n_elim is global block elim[l]; local block
    n_elim + q is top block kept[q] (T-local id)."""
    elim: np.ndarray            # global ids, elimination order
    kept: np.ndarray            # T-local ids, ascending
    groups: List[int]           # subtree index of each kept entry's group is per (subtree, member)
    schur_target: np.ndarray    # [n_schur] T-local id
    schur_group: np.ndarray     # [n_schur] subtree id
    blk_size: np.ndarray
    colptr: np.ndarray
    rowidx: np.ndarray
    src: List[tuple]            # per local stored block: (global CSC position or -1 = zero, transpose?)
    val_offset: np.ndarray
    nvals: int
    flops: float


@dataclasses.dataclass
class Plan:
    nparts: int
    order: np.ndarray           # global elimination order
    top: np.ndarray             # T: global ids in elimination order (T-local id = index)
    top_pos: Dict[int, int]
    roots: List[int]            # subtree roots (global ids)
    owner: Dict[int, int]       # subtree root -> part
    parts: List[PartPlan]
    top_sizes: np.ndarray
    top_colptr: np.ndarray
    top_rowidx: np.ndarray
    top_src: List[tuple]
    top_val_offset: np.ndarray
    top_nvals: int
    cliques: List[List[int]]    # per subtree (in order of `roots`): struct(root) as T-local ids
    flops_parts: List[float]
    flops_top: float


def _lower_csc(nb, pairs):
    cols = [set([j]) for j in range(nb)]
    for (i, j) in pairs:
        a, b = (i, j) if i >= j else (j, i)
        cols[b].add(a)
    colptr = np.zeros(nb + 1, dtype=np.int64)
    rows = []
    for j in range(nb):
        r = sorted(cols[j])
        rows.extend(r)
        colptr[j + 1] = colptr[j] + len(r)
    return colptr, np.asarray(rows, dtype=np.int32)


def plan_subtrees(blk_size, colptr, rowidx, nparts, *, order_opt=DD_ORDER_AUTO, balance=1.10,
                  max_top_frac=0.6) -> Plan:
    """Host planning, deterministic (every rank computes the same plan)."""
    blk_size = np.asarray(blk_size, dtype=np.int64)
    colptr = np.asarray(colptr, dtype=np.int64)
    rowidx = np.asarray(rowidx, dtype=np.int32)
    N = len(blk_size)
    h = dd_aux_analyze(blk_size, colptr, rowidx, DD_REAL64, dd_aux_default_options(order_opt, 0))
    order = dd_aux_get_order(h).astype(np.int64)
    parent, level, _ = dd_aux_get_etree(h)
    st_ptr, st_blk = dd_aux_get_struct(h)
    dd_aux_destroy(h)
    pos = np.empty(N, dtype=np.int64)
    pos[order] = np.arange(N)
    s = blk_size.astype(np.float64)
    r = np.array([s[st_blk[st_ptr[k]:st_ptr[k + 1]]].sum() for k in range(N)])
    fl = s ** 3 / 3 + r * s * s + r * r * s
    sub = fl.copy()
    children: List[List[int]] = [[] for _ in range(N)]
    for k in order:                      # children before parents
        p = int(parent[k])
        if p >= 0:
            sub[p] += sub[k]
            children[p].append(int(k))
    total = float(fl.sum())
    roots = sorted([int(k) for k in range(N) if parent[k] < 0], key=lambda k: pos[k])
    top: List[int] = []
    top_fl = 0.0

    def lpt(rs):
        loads = [0.0] * nparts
        own = {}
        for k in sorted(rs, key=lambda k: (-sub[k], pos[k])):
            q = int(np.argmin(loads))
            loads[q] += sub[k]
            own[k] = q
        return loads, own

    while roots:
        loads, own = lpt(roots)
        if max(loads) <= balance * (total - top_fl) / nparts and len(roots) >= nparts:
            break
        k = max(roots, key=lambda k: (sub[k], -pos[k]))
        if top_fl + fl[k] > max_top_frac * total and len(roots) >= nparts:
            break
        roots.remove(k)
        top.append(k)
        top_fl += fl[k]
        roots.extend(children[k])
    # a subtree whose root has no outside neighbours (a whole connected component) has nothing to
    # condense onto T: its root joins T too, so every part's kept set is non-empty
    while True:
        lone = [k for k in roots if st_ptr[k + 1] == st_ptr[k]]
        if not lone:
            break
        for k in lone:
            roots.remove(k)
            top.append(k)
            top_fl += fl[k]
            roots.extend(children[k])
    loads, own = lpt(roots)
    top = sorted(top, key=lambda k: pos[k])
    top_pos = {k: i for i, k in enumerate(top)}
    in_top = np.zeros(N, dtype=bool)
    in_top[top] = True
    # every subtree's nodes
    owner_node = np.full(N, -1, dtype=np.int64)
    sub_of = np.full(N, -1, dtype=np.int64)
    for si, rt in enumerate(roots):
        stack = [rt]
        while stack:
            k = stack.pop()
            owner_node[k] = own[rt]
            sub_of[k] = si
            stack.extend(children[k])
    assert np.all(in_top | (owner_node >= 0))
    cliques = []
    for rt in roots:
        stt = st_blk[st_ptr[rt]:st_ptr[rt + 1]]
        assert np.all(in_top[stt]), "T must be ancestor-closed"
        cliques.append(sorted(top_pos[int(u)] for u in stt))
    # stored global blocks by (row, col) with row >= col
    gpos = {}
    for j in range(N):
        for q in range(colptr[j], colptr[j + 1]):
            gpos[(int(rowidx[q]), j)] = q
    parts = []
    for prt in range(nparts):
        # elim: the nodes of this rank's subtrees (global elimination order); kept: one COPY of
        # struct(root tau) per subtree tau (like a subdomain's dual copies), group = tau
        elim = np.array([k for k in order if owner_node[k] == prt and not in_top[k]], dtype=np.int64)
        my_subs = [si for si, rt in enumerate(roots) if own[rt] == prt]
        ne = len(elim)
        loc = {int(k): l for l, k in enumerate(elim)}
        kloc, tgt, grp = {}, [], []
        for si in my_subs:
            for t in cliques[si]:
                kloc[(si, t)] = ne + len(tgt)
                tgt.append(t)
                grp.append(si)
        nb = ne + len(tgt)
        sizes = np.concatenate([blk_size[elim], blk_size[[top[t] for t in tgt]]]).astype(np.int64)
        pairs, srcmap = [], {}
        for (gi, gj), q in gpos.items():
            if gi == gj or (in_top[gi] and in_top[gj]):
                continue
            if owner_node[gi] != prt and owner_node[gj] != prt:
                continue
            if in_top[gi]:
                li, lj = kloc[(int(sub_of[gj]), top_pos[gi])], loc[gj]
            elif in_top[gj]:
                li, lj = loc[gi], kloc[(int(sub_of[gi]), top_pos[gj])]
            else:
                li, lj = loc[gi], loc[gj]
            pairs.append((li, lj))
            srcmap[(max(li, lj), min(li, lj))] = (q, (li < lj))  # stored (gi, gj) = (li, lj) block
        cp, ri = _lower_csc(nb, pairs)
        src, voff, tot = [], np.zeros(len(ri), dtype=np.int64), 0
        for j in range(nb):
            for q in range(cp[j], cp[j + 1]):
                i = int(ri[q])
                if i == j:
                    src.append((gpos[(int(elim[j]), int(elim[j]))], False) if j < ne else (-1, False))
                else:
                    src.append(srcmap[(i, j)])
                voff[q] = tot
                tot += int(sizes[i]) * int(sizes[j])
        parts.append(PartPlan(elim, np.asarray(tgt, dtype=np.int64), my_subs, np.asarray(tgt, dtype=np.int32),
                              np.asarray(grp, dtype=np.int32), sizes, cp, ri, src, voff, tot, float(loads[prt])))
    # top matrix: original T-T blocks + the clique pairs of every subtree struct
    nt = len(top)
    tpairs = []
    for (gi, gj), q in gpos.items():
        if gi != gj and in_top[gi] and in_top[gj]:
            tpairs.append((top_pos[gi], top_pos[gj]))
    for c in cliques:
        for a in range(len(c)):
            for b in range(a):
                tpairs.append((c[a], c[b]))
    tcp, tri = _lower_csc(nt, tpairs)
    tsrc, tvo, ttot = [], np.zeros(len(tri), dtype=np.int64), 0
    tsizes = blk_size[top].astype(np.int64)
    for j in range(nt):
        for q in range(tcp[j], tcp[j + 1]):
            i = int(tri[q])
            gi, gj = top[i], top[j]
            key = (gi, gj) if gi >= gj else (gj, gi)
            tsrc.append((gpos[key], gi < gj) if key in gpos else (-1, False))
            tvo[q] = ttot
            ttot += int(tsizes[i]) * int(tsizes[j])
    return Plan(nparts, order, np.asarray(top, dtype=np.int64), top_pos, roots, own, parts, tsizes, tcp, tri, tsrc,
                tvo, ttot, cliques, [p.flops for p in parts], top_fl)


def gather_values(vals, val_offset, blk_size, colptr, rowidx, src, out_offset, out_sizes, out_colptr, out_rowidx,
                  nvals):
    """Data movement only: build a sub-problem's value buffer (device) from the global one."""
    import torch
    out = torch.zeros(max(nvals, 1), dtype=vals.dtype, device=vals.device)
    gj_of = np.repeat(np.arange(len(blk_size)), np.diff(colptr))
    nb = len(out_sizes)
    for j in range(nb):
        for q in range(out_colptr[j], out_colptr[j + 1]):
            gq, tr = src[q]
            if gq < 0:
                continue
            gi, gj = int(rowidx[gq]), int(gj_of[gq])
            si, sj = int(blk_size[gi]), int(blk_size[gj])
            blk = vals[int(val_offset[gq]):int(val_offset[gq]) + si * sj].view(sj, si).t()  # (si x sj)
            if tr:
                blk = blk.t()
            ri, cj = blk.shape
            o = int(out_offset[q])
            out[o:o + ri * cj].view(cj, ri).copy_(blk.t())
    return out


class MultiGPUFactor:
    """Subtree-mapped factorization + distributed solve.  With `dist` = torch.distributed (NCCL, one
    process per GPU) the parts run on their own GPUs; with dist=None all parts run one after the
    other in this process (single-GPU emulation of the same schedule: no rank waits on another)."""

    def __init__(self, blk_size, colptr, rowidx, nparts, complex_=False, rank=0, dist=None, device="cuda",
                 order_opt=DD_ORDER_AUTO):
        self.plan = plan_subtrees(blk_size, colptr, rowidx, nparts, order_opt=order_opt)
        self.bs = np.asarray(blk_size, dtype=np.int64)
        self.colptr = np.asarray(colptr, dtype=np.int64)
        self.rowidx = np.asarray(rowidx, dtype=np.int32)
        self.cplx = bool(complex_)
        self.rank, self.dist, self.device = rank, dist, device
        self.nparts = nparts
        mine = range(nparts) if dist is None else [rank]
        self.parts = {}
        for prt in mine:
            pp = self.plan.parts[prt]
            if len(pp.elim) == 0:  # more ranks than subtrees: this part has nothing to factor
                continue
            ss = SchurSolver(pp.blk_size, pp.colptr, pp.rowidx, pp.schur_target, pp.schur_group, self.plan.top_sizes,
                             complex_=complex_, order=DD_ORDER_NATURAL, device=device)
            ss._auxs = self.plan.top_sizes
            self.parts[prt] = ss
        self.top = None
        if dist is None or rank == 0:
            self.top = AuxSolver(self.plan.top_sizes, self.plan.top_colptr, self.plan.top_rowidx, complex_=complex_,
                                 order=DD_ORDER_NATURAL, device=device, refine_steps=1)
        self.dof = np.concatenate([[0], np.cumsum(self.bs)]).astype(np.int64)

    # -------------------------------------------------------------------------------- factor
    def factor(self, d_vals, val_offset):
        import torch
        P = self.plan
        exports = {}
        self.timings = {"parts_ms": {}, "export_bytes": {}}
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        for prt, ss in self.parts.items():
            pp = P.parts[prt]
            pv = gather_values(d_vals, val_offset, self.bs, self.colptr, self.rowidx, pp.src, pp.val_offset,
                               pp.blk_size, pp.colptr, pp.rowidx, pp.nvals)
            e0, e1 = ev(), ev()
            e0.record()
            rc, _ = ss.factor(pv, pp.val_offset)
            if rc != DD_OK:
                raise RuntimeError(f"part {prt}: partial factorization rc={rc}")
            ss._pv = pv
            dS, Soff = ss.export()
            e1.record()
            torch.cuda.synchronize()
            self.timings["parts_ms"][prt] = e0.elapsed_time(e1)
            self.timings["export_bytes"][prt] = dS.numel() * dS.element_size()
            exports[prt] = (dS, Soff, ss.cliques())
        if self.dist is not None:       # NCCL point-to-point: every rank's S buffer to rank 0
            if self.rank != 0:
                dS = exports[self.rank][0] if self.rank in exports else torch.zeros(0, dtype=torch.complex128 if
                                                                                     self.cplx else torch.float64,
                                                                                     device=self.device)
                self.dist.send(torch.tensor([dS.numel()], dtype=torch.int64, device=dS.device), dst=0)
                if dS.numel():
                    self.dist.send(dS, dst=0)
            else:
                for src in range(1, self.nparts):
                    n = torch.zeros(1, dtype=torch.int64, device=self.device)
                    self.dist.recv(n, src=src)
                    buf = torch.empty(int(n.item()), dtype=torch.complex128 if self.cplx else torch.float64,
                                      device=self.device)
                    if buf.numel():
                        self.dist.recv(buf, src=src)
                    else:
                        continue
                    cl = [P.cliques[si] for si in P.parts[src].groups]
                    ms = [int(P.top_sizes[c].sum()) for c in cl]
                    soff = np.concatenate([[0], np.cumsum([m * m for m in ms])[:-1]]).astype(np.int64)
                    exports[src] = (buf, soff, cl)
        if self.top is None:
            return DD_OK
        tv = gather_values(d_vals, val_offset, self.bs, self.colptr, self.rowidx, P.top_src, P.top_val_offset,
                           P.top_sizes, P.top_colptr, P.top_rowidx, P.top_nvals)
        self._tv_orig = tv.clone()  # the top blocks' own values (global refinement residual)
        e0, e1 = ev(), ev()
        e0.record()
        for prt in sorted(exports):
            dS, Soff, cl = exports[prt]
            if not cl:
                continue
            ptr, blk = cliques_to_csr(cl)
            w = torch.empty(max(256, dd_aux_assemble_work_bytes(self.top.h, ptr, blk)), dtype=torch.uint8,
                            device=self.device)
            dd_aux_assemble_acc(self.top.h, ptr, blk, dS, Soff, P.top_val_offset, tv, w)
            torch.cuda.synchronize()
        self._tv = tv
        rc, fi = self.top.factor(tv, P.top_val_offset)
        e1.record()
        torch.cuda.synchronize()
        self.timings["top_ms"] = e0.elapsed_time(e1)  # assemble_acc of every part's S + top factor
        return rc

    # -------------------------------------------------------------------------------- solve
    def _rows(self, prt):
        pp = self.plan.parts[prt]
        ne = len(pp.elim)
        rows = np.concatenate([np.arange(self.dof[g], self.dof[g + 1]) for g in pp.elim]) if ne else \
            np.zeros(0, dtype=np.int64)
        return rows, int(pp.blk_size[:ne].sum()), int(pp.blk_size[ne:].sum())

    def _local(self, prt, B):
        """The part's n_loc x nrhs right-hand side: its subtrees' rows of B, then zero kept rows."""
        import torch
        rows, ne, nk = self._rows(prt)
        top = B.index_select(0, torch.from_numpy(rows).to(B.device))
        kept = torch.zeros((nk, B.shape[1]), dtype=B.dtype, device=B.device)
        return torch.cat([top, kept], 0).t().contiguous().t()

    def _dd_solve(self, Bparts, bT):
        """Condense -> reduce -> top solve -> broadcast -> recover.  Returns (x_T, {part: X_loc})."""
        import torch
        P = self.plan
        nrhs = next(iter(Bparts.values())).shape[1]
        dt = next(iter(Bparts.values())).dtype
        dev = next(iter(Bparts.values())).device
        G = torch.zeros((nrhs, self._ntd), dtype=dt, device=dev).t()
        for prt, ss in self.parts.items():
            ss.condense_(Bparts[prt], G)
        if self.dist is not None:
            self.dist.reduce(G, dst=0)
        if self.top is not None:
            G += bT
            self.top.solve_(G)
        if self.dist is not None:
            Gc = G.t().contiguous()
            self.dist.broadcast(Gc, src=0)
            G = Gc.t()
        Xl = {prt: ss.recover(Bparts[prt], G) for prt, ss in self.parts.items()}
        return G, Xl

    def solve(self, B, refine_steps=1):
        """B: global n x nrhs CUDA tensor (column-major) on every rank.  The DD solve, then
        refine_steps steps of global iterative refinement r = b - A x (the residual of every part's
        original blocks and of the top's original blocks, dd_aux_residual), x += solve(r).  Returns
        X on rank 0 (dist) or here (emulation); None on other ranks."""
        import torch
        P = self.plan
        self._tdof = np.concatenate([[0], np.cumsum(P.top_sizes)]).astype(np.int64)
        self._ntd = int(self._tdof[-1])
        trows = torch.from_numpy(np.concatenate([np.arange(self.dof[g], self.dof[g + 1]) for g in P.top])).to(B.device)
        bT = B.index_select(0, trows).t().contiguous().t() if self.top is not None else None
        Bp = {prt: self._local(prt, B) for prt in self.parts}
        xT, Xl = self._dd_solve(Bp, bT)
        for _ in range(refine_steps):
            # residual pieces: every part's rows (its kept rows collect -A_{T,part} x_part per copy)
            Rp, RT = {}, torch.zeros_like(xT)
            for prt, ss in self.parts.items():
                rows, ne, nk = self._rows(prt)
                pp = self.plan.parts[prt]
                kidx = np.concatenate([np.arange(self._tdof[t], self._tdof[t + 1]) for t in pp.schur_target]) if nk \
                    else np.zeros(0, dtype=np.int64)
                kept = xT.index_select(0, torch.from_numpy(kidx).to(B.device))
                Xloc = torch.cat([Xl[prt][:ne], kept], 0).t().contiguous().t()
                R = torch.empty_like(Xloc)
                w = ss._work(dd_aux_solve_work_bytes(ss.h, Xloc.shape[1]))
                dd_aux_residual(ss.h, ss.factor_buf, ss._pv, Bp[prt], Xloc, R, w)
                RT.index_add_(0, torch.from_numpy(kidx).to(B.device), R[ne:])  # sum over the T copies
                Rp[prt] = torch.cat([R[:ne], torch.zeros_like(R[ne:])], 0).t().contiguous().t()
            if self.dist is not None:
                self.dist.reduce(RT, dst=0)
            rT = None
            if self.top is not None:
                Rt = torch.empty_like(xT)
                w = self.top._work(dd_aux_solve_work_bytes(self.top.h, xT.shape[1]))
                dd_aux_residual(self.top.h, self.top.factor_buf, self._tv_orig, bT, xT, Rt, w)
                rT = Rt + RT
            dT, dXl = self._dd_solve(Rp, rT)
            xT = xT + dT
            for prt in Xl:
                Xl[prt] = Xl[prt] + dXl[prt]
        # gather X (rank 0)
        X = torch.zeros_like(B.t()).t() if (self.dist is None or self.rank == 0) else None
        for prt in Xl:
            rows, ne, nk = self._rows(prt)
            if X is not None:
                X.index_copy_(0, torch.from_numpy(rows).to(B.device), Xl[prt][:ne])
            else:
                self.dist.send(Xl[prt][:ne].t().contiguous(), dst=0)
        if self.dist is not None and self.rank == 0:
            for src in range(1, self.nparts):
                if len(self.plan.parts[src].elim) == 0:
                    continue
                rows, ne, nk = self._rows(src)
                buf = torch.empty((B.shape[1], len(rows)), dtype=B.dtype, device=B.device)
                self.dist.recv(buf, src=src)
                X.index_copy_(0, torch.from_numpy(rows).to(B.device), buf.t())
        if X is not None:
            X.index_copy_(0, trows, xT)
        return X
