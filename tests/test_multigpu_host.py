"""f4 host logic (CPU): the subtree-to-GPU plan and the gather/reduce protocol.

The plan (paper_2002_05019_b200.multigpu.plan_subtrees) is checked structurally (T ancestor-
closed, every other block in exactly one part, no block coupling two parts, cliques = structs)
and numerically with plain dense linear algebra on CPU: each part's Schur contribution
S_tau = -A_{K,tau} A_{tau,tau}^{-1} A_{tau,K} (the plain definition, numpy solve) assembled onto
the top blocks' own values must equal the dense Schur complement of the whole matrix onto T.  A
world-size-2 gloo run exercises the same send/recv protocol MultiGPUFactor uses over NCCL.
"""
import os

import numpy as np
import pytest
import torch

import dd_inputs
from dd_inputs import dense_expand
import paper_2002_05019_b200 as dd
from paper_2002_05019_b200.multigpu import gather_values, plan_subtrees


def _prob(name="cfg1", grid=(3, 3, 2), sizes=12):
    return dd_inputs.config(name, grid=grid, sizes=sizes)


def _part_dense(p, pp):
    """Dense symmetric matrix of a part's Schur-mode problem (values gathered like the library)."""
    vals = torch.from_numpy(p.values)
    v = gather_values(vals, p.val_offset, p.blk_size, p.colptr, p.rowidx, pp.src, pp.val_offset, pp.blk_size,
                      pp.colptr, pp.rowidx, pp.nvals).numpy()
    q = dd_inputs.Problem(pp.blk_size, pp.colptr, pp.rowidx, v, pp.val_offset, [])
    return dense_expand(q)


def _top_dense(p, plan):
    vals = torch.from_numpy(p.values)
    v = gather_values(vals, p.val_offset, p.blk_size, p.colptr, p.rowidx, plan.top_src, plan.top_val_offset,
                      plan.top_sizes, plan.top_colptr, plan.top_rowidx, plan.top_nvals).numpy()
    q = dd_inputs.Problem(plan.top_sizes, plan.top_colptr, plan.top_rowidx, v, plan.top_val_offset, [])
    return dense_expand(q)


def _schur_groups(p, pp, plan):
    """Per group (subtree) of the part: dense S over its clique (T-local block order)."""
    D = _part_dense(p, pp)
    ne = int(pp.blk_size[:len(pp.elim)].sum())
    S = -D[ne:, :ne] @ np.linalg.solve(D[:ne, :ne], D[:ne, ne:])
    out = []
    off = np.concatenate([[0], np.cumsum(pp.blk_size[len(pp.elim):])])
    for si in pp.groups:
        idx = [q for q in range(len(pp.schur_group)) if pp.schur_group[q] == si]
        rows = np.concatenate([np.arange(off[q], off[q + 1]) for q in idx])
        out.append((plan.cliques[si], S[np.ix_(rows, rows)]))
    return out


@pytest.mark.parametrize("nparts", [2, 3, 4])
def test_plan_structure_and_schur_sum(nparts):
    p = _prob()
    plan = plan_subtrees(p.blk_size, p.colptr, p.rowidx, nparts)
    N = p.nblk
    top = set(int(k) for k in plan.top)
    seen = {}
    for prt, pp in enumerate(plan.parts):
        for k in pp.elim:
            assert int(k) not in top and int(k) not in seen
            seen[int(k)] = prt
    assert len(seen) + len(top) == N
    # no original block couples two parts
    for j in range(N):
        for q in range(p.colptr[j], p.colptr[j + 1]):
            i = int(p.rowidx[q])
            if i in seen and j in seen:
                assert seen[i] == seen[j]
    # T is ancestor-closed
    h = dd.dd_aux_analyze(p.blk_size, p.colptr, p.rowidx)
    parent, _, _ = dd.dd_aux_get_etree(h)
    dd.dd_aux_destroy(h)
    for k in top:
        assert parent[k] < 0 or int(parent[k]) in top
    # numerics: top values + sum of the parts' Schur contributions == dense Schur complement onto T
    A = dense_expand(p)
    off = p.dof_offset
    trows = np.concatenate([np.arange(off[k], off[k + 1]) for k in plan.top])
    rest = np.setdiff1d(np.arange(p.n), trows)
    Sref = A[np.ix_(trows, trows)] - A[np.ix_(trows, rest)] @ np.linalg.solve(A[np.ix_(rest, rest)],
                                                                            A[np.ix_(rest, trows)])
    T = _top_dense(p, plan)
    tdof = np.concatenate([[0], np.cumsum(plan.top_sizes)])
    for pp in plan.parts:
        for cl, S in _schur_groups(p, pp, plan):
            r = np.concatenate([np.arange(tdof[t], tdof[t + 1]) for t in cl])
            T[np.ix_(r, r)] += S
    assert np.abs(T - Sref).max() <= 1e-10 * np.abs(Sref).max()
    assert max(plan.flops_parts) <= 1.6 * sum(plan.flops_parts) / nparts


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = _prob()
    plan = plan_subtrees(p.blk_size, p.colptr, p.rowidx, world)
    groups = _schur_groups(p, plan.parts[rank], plan)
    # the MultiGPUFactor protocol: one flat buffer of the part's group matrices (column-major)
    buf = torch.from_numpy(np.concatenate([S.ravel(order="F") for _, S in groups]) if groups else np.zeros(0))
    if rank != 0:
        dist.send(torch.tensor([buf.numel()], dtype=torch.int64), dst=0)
        dist.send(buf, dst=0)
        q.put((rank, None))
    else:
        T = _top_dense(p, plan)
        tdof = np.concatenate([[0], np.cumsum(plan.top_sizes)])
        allg = {0: groups}
        for src in range(1, world):
            n = torch.zeros(1, dtype=torch.int64)
            dist.recv(n, src=src)
            b = torch.empty(int(n.item()), dtype=torch.float64)
            dist.recv(b, src=src)
            cl = [plan.cliques[si] for si in plan.parts[src].groups]
            ms = [int(plan.top_sizes[c].sum()) for c in cl]
            o, gl = 0, []
            for c, m in zip(cl, ms):
                gl.append((c, b[o:o + m * m].numpy().reshape(m, m, order="F")))
                o += m * m
            allg[src] = gl
        for src in range(world):
            for cl, S in allg[src]:
                r = np.concatenate([np.arange(tdof[t], tdof[t + 1]) for t in cl])
                T[np.ix_(r, r)] += S
        A = dense_expand(p)
        off = p.dof_offset
        tr = np.concatenate([np.arange(off[k], off[k + 1]) for k in plan.top])
        rest = np.setdiff1d(np.arange(p.n), tr)
        Sref = A[np.ix_(tr, tr)] - A[np.ix_(tr, rest)] @ np.linalg.solve(A[np.ix_(rest, rest)], A[np.ix_(rest, tr)])
        q.put((0, float(np.abs(T - Sref).max() / np.abs(Sref).max())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reduce_protocol():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    assert res[0] is not None and res[0] <= 1e-10, res


def test_plan_random_patterns_and_validate():
    """plan_subtrees on random block graphs and orders: every non-top block in exactly one part, T
    ancestor-closed, every part's Schur-mode handle passes the library's table validation."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        nblk = int(rng.integers(6, 40))
        sizes = rng.integers(1, 30, nblk)
        edges = [[u, v] for u in range(nblk) for v in range(u) if rng.random() < rng.uniform(0.05, 0.4)]
        cp, ri = dd_inputs.block_pattern_from_cliques(nblk, edges)
        nparts = int(rng.integers(2, 5))
        plan = plan_subtrees(sizes, cp, ri, nparts)
        owned = np.concatenate([pp.elim for pp in plan.parts] + [plan.top])
        assert sorted(owned.tolist()) == list(range(nblk))
        for pp in plan.parts:
            if len(pp.elim) == 0:
                continue
            assert len(pp.schur_target) > 0   # every subtree condenses onto T (lone components join T)
            h = dd.dd_aux_analyze_partial(pp.blk_size, pp.colptr, pp.rowidx, pp.schur_target, pp.schur_group,
                                          plan.top_sizes, dd.DD_REAL64, dd.dd_aux_default_options(dd.DD_ORDER_NATURAL))
            dd.dd_aux_validate(h)
            dd.dd_aux_destroy(h)
        if len(plan.top):
            h = dd.dd_aux_analyze(plan.top_sizes, plan.top_colptr, plan.top_rowidx)
            dd.dd_aux_validate(h)
            dd.dd_aux_destroy(h)
