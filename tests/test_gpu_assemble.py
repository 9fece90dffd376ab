"""GPU parity of the f1 clique assembly (dd_aux_assemble) against oracle.assemble.

The sum is evaluated in the same order with correctly rounded additions on both sides, so
the comparison is BIT-EXACT (include/dd_aux.h).  Cases: the config-0
grid, scaled-down configs 2 (unstructured, ragged sizes) and 3 (complex), random cliques
that overlap (several contributors per block) with sizes 1..70 (ragged 32-column chunks),
with and without the symmetric part, an empty clique list, and assembly -> factor -> solve
end to end against the oracle.
"""
import numpy as np
import pytest

import dd_inputs
import oracle
from dd_inputs import Problem
from tests._gpu import rel_diff, to_dev_colmajor
from tests.test_oracle_assemble import random_cliques

pytestmark = pytest.mark.gpu


def _gpu_assemble(sizes, colptr, rowidx, vo, cliques, S, symmetrize, complex_):
    import torch
    import paper_2002_05019_b200 as dd
    s = dd.AuxSolver(sizes, colptr, rowidx, complex_=complex_)
    offs = np.concatenate([[0], np.cumsum([M.size for M in S])]).astype(np.int64)
    flat = np.concatenate([np.asarray(M).T.ravel() for M in S]) if S else np.zeros(1)  # column-major
    tdt = torch.complex128 if complex_ else torch.float64
    dS = torch.from_numpy(flat.astype(np.complex128 if complex_ else np.float64)).to("cuda")
    total = max(int(vo[q]) + int(sizes[rowidx[q]]) * int(sizes[np.searchsorted(colptr, q, "right") - 1])
                for q in range(len(rowidx)))
    d_vals = torch.full((total,), float("nan"), dtype=tdt, device="cuda")  # every element must be written
    s.assemble(cliques, dS, offs[:-1], vo, d_vals=d_vals, symmetrize=symmetrize)
    torch.cuda.synchronize()
    return s, d_vals


@pytest.mark.parametrize("name,grid,sizes", [("cfg0", None, None),
                                             ("cfg2", (3, 3, 2), lambda n, r: r.integers(1, 70, n)),
                                             ("cfg3", (2, 2, 2), 37)])
@pytest.mark.parametrize("symmetrize", [True, False])
def test_assemble_configs_bitexact(name, grid, sizes, symmetrize):
    p = dd_inputs.config(name, grid=grid, sizes=sizes, keep_cliques=True)
    cl = [c for _, c in p.cliques]
    ref = oracle.assemble(p.blk_size, p.colptr, p.rowidx, p.val_offset, cl, p.clique_S, symmetrize)
    s, d_vals = _gpu_assemble(p.blk_size, p.colptr, p.rowidx, p.val_offset, cl, p.clique_S, symmetrize, p.is_complex)
    got = d_vals.cpu().numpy()
    s.close()
    assert np.array_equal(got, ref)
    if symmetrize:
        assert np.array_equal(got, p.values)  # the generator's own accumulation


@pytest.mark.parametrize("complex_", [False, True])
@pytest.mark.parametrize("seed", [0, 1])
def test_assemble_overlapping_cliques_bitexact(complex_, seed):
    rng = np.random.default_rng(100 + seed)
    sizes, colptr, rowidx, vo, cl, S = random_cliques(10, 9, rng, smax=70, complex_=complex_)
    for sym in (True, False):
        ref = oracle.assemble(sizes, colptr, rowidx, vo, cl, S, sym)
        s, d_vals = _gpu_assemble(sizes, colptr, rowidx, vo, cl, S, sym, complex_)
        got = d_vals.cpu().numpy()
        s.close()
        assert np.array_equal(got, ref)


def test_assemble_empty_clique_list_writes_zeros():
    rng = np.random.default_rng(3)
    sizes, colptr, rowidx, vo, cl, S = random_cliques(5, 4, rng)
    s, d_vals = _gpu_assemble(sizes, colptr, rowidx, vo, [], [], True, False)
    got = d_vals.cpu().numpy()
    s.close()
    assert np.all(got == 0)


@pytest.mark.parametrize("name,grid,sizes", [("cfg1", (3, 3, 2), 48), ("cfg3", (2, 2, 2), 40)])
def test_assemble_then_factor_solve(name, grid, sizes):
    """Clique form in, solution out: assemble on the device, factor, solve; oracle on the same matrix."""
    import torch
    p = dd_inputs.config(name, grid=grid, sizes=sizes, keep_cliques=True)
    cl = [c for _, c in p.cliques]
    s, d_vals = _gpu_assemble(p.blk_size, p.colptr, p.rowidx, p.val_offset, cl, p.clique_S, True, p.is_complex)
    rc, finfo = s.factor(d_vals, p.val_offset)
    B = dd_inputs.random_rhs(p.n, 3, p.is_complex, 0)
    Bd = to_dev_colmajor(B, torch)
    s.solve_(Bd)
    torch.cuda.synchronize()
    X = Bd.cpu().numpy()
    F = oracle.block_factor(p, list(s.order()))
    Xo, _, _ = oracle.refine_solve(p, F, B, 1)
    s.close()
    assert rel_diff(X, Xo) <= 1e-9
    assert oracle.residual_berr(p, X, B).max() <= 1e-12
    if not p.is_complex:
        assert (finfo["npos"], finfo["nneg"], finfo["nzero"]) == oracle.inertia(F)
