"""Pins for oracle.symbolic (clique-graph elimination game), CPU only.

Independent reference: the fill-path theorem (Rose, Tarjan & Lueker 1976): in
the filled graph, {u, v} is an edge iff the original graph has a path from u to
v whose interior vertices are all eliminated before both u and v.  That is a
reachability computation, not the elimination game, so a wrong clique rule
fails it.  Plus SPEC.md:486-489 hand cases and elimination-tree properties.
"""
import numpy as np
import pytest

import dd_inputs
from dd_inputs import block_pattern_from_cliques
from oracle.block_ldlt import symbolic, flops_factor


def _fill_path(nblk, edges, order):
    pos = np.empty(nblk, dtype=int)
    pos[list(order)] = np.arange(nblk)
    adj = [set() for _ in range(nblk)]
    for u, v in edges:
        adj[u].add(v)
        adj[v].add(u)
    filled = set()
    for u in range(nblk):
        # DFS from u through vertices eliminated before u; record reachable later vertices
        lim = pos[u]
        seen = {u}
        stack = [u]
        while stack:
            x = stack.pop()
            for y in adj[x]:
                if y in seen:
                    continue
                seen.add(y)
                if pos[y] < lim:
                    stack.append(y)
                elif y != u:
                    # path interior all before u; need interior before y as well: pos[y] > pos[u] here
                    filled.add((max(u, y), min(u, y)))
    return filled


def _pattern(nblk, edges):
    cols = [[j] for j in range(nblk)]
    for u, v in edges:
        i, j = max(u, v), min(u, v)
        if i not in cols[j]:
            cols[j].append(i)
    colptr = [0]
    rows = []
    for j in range(nblk):
        r = sorted(cols[j])
        rows += r
        colptr.append(len(rows))
    return np.array(colptr), np.array(rows, dtype=np.int32)


def test_fill_matches_fill_path_theorem():
    rng = np.random.default_rng(0)
    for trial in range(60):
        nblk = int(rng.integers(2, 25))
        dens = rng.uniform(0.05, 0.6)
        edges = [(u, v) for u in range(nblk) for v in range(u) if rng.random() < dens]
        colptr, rowidx = _pattern(nblk, edges)
        order = rng.permutation(nblk)
        sym = symbolic(nblk, colptr, rowidx, order)
        filled = _fill_path(nblk, edges, order)
        assert filled == sym["fill"] | sym["orig"]


def test_spec_hand_cases():
    # block-diagonal: zero fill, any order
    colptr, rowidx = _pattern(5, [])
    assert symbolic(5, colptr, rowidx, [4, 2, 0, 1, 3])["fill"] == set()
    # path g1-g2-g3: eliminating the middle first fills (g1,g3)
    colptr, rowidx = _pattern(3, [(0, 1), (1, 2)])
    assert symbolic(3, colptr, rowidx, [1, 0, 2])["fill"] == {(2, 0)}
    assert symbolic(3, colptr, rowidx, [0, 1, 2])["fill"] == set()


def test_cfg0_four_cycle():
    """Config 0 (2x2x1 grid) is a 4-cycle of interfaces: any order gives exactly one fill block
    (4 diagonal + 4 original + 1 fill = 9 lower blocks)."""
    p = dd_inputs.config("cfg0")
    assert p.nblk == 4 and p.n == 128 and p.nnzb == 8
    rng = np.random.default_rng(1)
    for _ in range(10):
        order = rng.permutation(4)
        sym = symbolic(4, p.colptr, p.rowidx, order)
        assert len(sym["fill"]) == 1
        # hand count for s = 32: r = 64, 64, 32, 0 along any order of a 4-cycle
        s = 32.0
        hand = 4 * s ** 3 / 3 + (64 + 64 + 32) * s * s + (64 ** 2 + 64 ** 2 + 32 ** 2) * s
        assert flops_factor(p.blk_size, sym) == pytest.approx(hand, rel=1e-15)


def test_etree_levels_are_independent():
    """Nodes of one level are never ancestor/descendant of each other and every
    struct member is an ancestor (so level-batched execution is race-free)."""
    p = dd_inputs.config("cfg1", grid=(3, 3, 3), sizes=8)
    rng = np.random.default_rng(2)
    order = rng.permutation(p.nblk)
    sym = symbolic(p.nblk, p.colptr, p.rowidx, order)
    par = sym["parent"]

    def ancestors(k):
        out = set()
        while par[k] >= 0:
            k = int(par[k])
            out.add(k)
        return out

    anc = [ancestors(k) for k in range(p.nblk)]
    for k in range(p.nblk):
        assert set(sym["struct"][k]) <= anc[k]
        for j in anc[k]:
            assert sym["level"][j] > sym["level"][k]


def test_generator_topology():
    """Interface counts of the BASELINE grids (ledger L10: 8x8x4 has 640 face pairs)."""
    assert len(dd_inputs.grid_interfaces(4, 4, 4)) == 144
    assert len(dd_inputs.grid_interfaces(8, 8, 4)) == 640
    assert len(dd_inputs.grid_interfaces(3, 6, 10)) == 432
    rng = np.random.default_rng(0)
    pairs = dd_inputs.unstructured_interfaces(6, 6, 6, rng)
    deg = np.zeros(216, dtype=int)
    for a, b in pairs:
        deg[a] += 1
        deg[b] += 1
    assert deg.min() >= 4 and deg.max() <= 14
