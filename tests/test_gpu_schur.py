"""f3 subdomain elimination + f2 primal recovery on the GPU (Schur-mode partial factorization)
against oracle.dd and against scipy's direct solve of the global arrowhead matrix.

PAPER.md:27 (§II): "eliminating via many independent sparse direct factorizations the primal
DoFs"; primal unknowns "recovered ... via many smaller size sparse forward backward
substitutions".  Tolerances: Schur complements / condensed right-hand sides element-wise within
1e-10 of the largest entry (one unrefined partial factorization vs SuperLU); the recovered and
full solutions within the north_star's 1e-9 relative difference, and the global backward error
||A x - b||_inf / (||A||_inf ||x||_inf) <= 1e-12.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spl

import dd_inputs
from dd_inputs.fem import arrowhead, arrowhead_rhs, fem_dd, schur_block_problem
import oracle.dd as odd

from tests._gpu import to_dev_colmajor

pytestmark = pytest.mark.gpu


def _setup(m, leaf):
    import torch
    import paper_2002_05019_b200 as dd
    prob, ns, tgt, grp, auxs, info = schur_block_problem(m, leaf=leaf)
    ss = dd.SchurSolver(prob.blk_size, prob.colptr, prob.rowidx, tgt, grp, auxs, complex_=m.complex_)
    ss._auxs = auxs
    vals = torch.from_numpy(prob.values).cuda()
    rc, fi = ss.factor(vals, prob.val_offset)
    assert rc == dd.DD_OK, rc
    return prob, ss, info, auxs


def _handle_F(m, prob, info):
    """Primal right-hand sides in the handle's DoF numbering (kept rows zero)."""
    F = np.zeros((prob.n, m.f[0].shape[1]), dtype=np.result_type(m.f[0], m.K[0].dtype))
    for p in range(m.nsub):
        s0, n_p = info["sub_dof"][p]
        F[s0:s0 + n_p] = m.f[p][info["node_perm"]]
    return np.asfortranarray(F)


def _primal_from_handle(m, X, info):
    out = []
    for p in range(m.nsub):
        s0, n_p = info["sub_dof"][p]
        x = np.empty((n_p, X.shape[1]), dtype=X.dtype)
        x[info["node_perm"]] = X[s0:s0 + n_p]
        out.append(x)
    return out


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("grid,a,leaf", [((2, 2, 1), 6, 16), ((2, 2, 2), 9, 40)])
def test_schur_export_and_condense(cplx, grid, a, leaf):
    import torch
    m = fem_dd(*grid, a, complex_=cplx, seed=7, nrhs=3)
    prob, ss, info, auxs = _setup(m, leaf)
    dS, Soff = ss.export()
    torch.cuda.synchronize()
    S = dS.cpu().numpy()
    cl = ss.cliques()
    assert cl == [m.sub_ifaces[p] for p in range(m.nsub) if m.sub_ifaces[p]]
    for g, p in enumerate([p for p in range(m.nsub) if m.sub_ifaces[p]]):
        mp = len(cl[g]) * m.s_dual
        Sg = S[Soff[g]:Soff[g] + mp * mp].reshape(mp, mp).T
        So = odd.schur_contribution(m, p)
        assert np.array_equal(Sg, Sg.T)                      # exported symmetric (no conjugation)
        assert np.abs(Sg - So).max() <= 1e-10 * np.abs(So).max(), (p, np.abs(Sg - So).max())
    F = _handle_F(m, prob, info)
    G = to_dev_colmajor(m.bb, torch)
    ss.condense_(to_dev_colmajor(F, torch), G)
    torch.cuda.synchronize()
    Go = odd.condense(m)
    assert np.abs(G.cpu().numpy() - Go).max() <= 1e-10 * np.abs(Go).max()


@pytest.mark.parametrize("cplx", [False, True])
def test_recover_against_oracle(cplx):
    import torch
    m = fem_dd(2, 2, 2, 8, complex_=cplx, seed=8, nrhs=5)
    prob, ss, info, auxs = _setup(m, 32)
    rng = np.random.default_rng(1)
    xb = rng.standard_normal((m.n_dual, 5)) + (1j * rng.standard_normal((m.n_dual, 5)) if cplx else 0)
    F = _handle_F(m, prob, info)
    X = ss.recover(to_dev_colmajor(F, torch), to_dev_colmajor(xb, torch))
    torch.cuda.synchronize()
    xs = _primal_from_handle(m, X.cpu().numpy(), info)
    for p in range(m.nsub):
        xo = odd.recover(m, p, xb)
        rel = np.abs(xs[p] - xo).max(0) / np.abs(xo).max(0)
        assert rel.max() <= 1e-9, (p, rel.max())


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("grid,a,leaf", [((2, 2, 2), 8, 32), ((3, 3, 2), 12, 64)])
def test_full_dd_pipeline_on_gpu(cplx, grid, a, leaf):
    """f3 -> f1 -> aux factor/solve -> f2, every step in the library, against the global solve."""
    import torch
    import paper_2002_05019_b200 as dd
    m = fem_dd(*grid, a, complex_=cplx, seed=9, nrhs=4)
    prob, ss, info, auxs = _setup(m, leaf)
    dS, Soff = ss.export()
    cl = ss.cliques()
    colptr, rowidx = dd_inputs.block_pattern_from_cliques(len(auxs), cl)
    aux_off, _ = dd_inputs._layout(auxs, colptr, rowidx)
    aux = dd.AuxSolver(auxs, colptr, rowidx, complex_=cplx)
    avals = aux.assemble(cl, dS, Soff, aux_off, symmetrize=False)
    rc, _ = aux.factor(avals, aux_off)
    assert rc == dd.DD_OK
    F = to_dev_colmajor(_handle_F(m, prob, info), torch)
    G = to_dev_colmajor(m.bb, torch)
    ss.condense_(F, G)                       # G = b_b - sum_p C_p^T K_p^-1 f_p
    aux.solve_(G)                            # x_b
    X = ss.recover(F, G)                     # x_p
    torch.cuda.synchronize()
    xs = _primal_from_handle(m, X.cpu().numpy(), info)
    xb = G.cpu().numpy()
    got = np.concatenate(xs + [xb])
    A = arrowhead(m)
    b = arrowhead_rhs(m)
    Xd = spl.spsolve(A.tocsc(), b)
    rel = np.abs(got - Xd).max(0) / np.abs(Xd).max(0)
    assert rel.max() <= 1e-9, rel.max()
    nA = float(abs(A).sum(axis=1).max())
    berr = np.abs(A @ got - b).max(0) / (nA * np.abs(got).max(0))
    print(f"grid {grid} a={a}: n={A.shape[0]} rel diff {rel.max():.2e} berr {berr.max():.2e}")
    assert berr.max() <= 1e-12, berr.max()
    aux.close()
    ss.close()


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_schur_mode_random_patterns_one_group(cplx, seed):
    """Schur mode on random block-sparse matrices (sizes 1-40, kept blocks of different sizes, kept
    blocks coupled to each other and to everything): with ONE group the export is the whole Schur
    complement onto the kept blocks, D_kk - D_ke D_ee^{-1} D_ek (the plain definition, numpy)."""
    import torch
    import paper_2002_05019_b200 as dd
    from dd_inputs import Problem, block_pattern_from_cliques, dense_expand
    rng = np.random.default_rng(100 + seed + 10 * cplx)
    nblk = int(rng.integers(5, 12))
    ns = int(rng.integers(1, 4))
    sizes = rng.integers(1, 41, nblk)
    edges = [[u, v] for u in range(nblk) for v in range(u) if rng.random() < 0.5]
    colptr, rowidx = block_pattern_from_cliques(nblk, edges)
    off, tot = [], 0
    for j in range(nblk):
        for q in range(colptr[j], colptr[j + 1]):
            off.append(tot)
            tot += int(sizes[rowidx[q]]) * int(sizes[j])
    vals = rng.standard_normal(tot) + (1j * rng.standard_normal(tot) if cplx else 0)
    p = Problem(np.asarray(sizes, dtype=np.int64), colptr, rowidx, vals, np.asarray(off, dtype=np.int64), [])
    tgt = np.arange(ns, dtype=np.int32)
    grp = np.zeros(ns, dtype=np.int32)
    auxs = np.asarray(sizes[nblk - ns:], dtype=np.int64)
    ss = dd.SchurSolver(p.blk_size, p.colptr, p.rowidx, tgt, grp, auxs, complex_=cplx, order=dd.DD_ORDER_AUTO)
    ss._auxs = auxs
    rc, _ = ss.factor(torch.from_numpy(p.values).cuda(), p.val_offset)
    assert rc == dd.DD_OK
    dd.dd_aux_validate(ss.h)
    dS, Soff = ss.export()
    torch.cuda.synchronize()
    m = int(auxs.sum())
    S = dS.cpu().numpy()[:m * m].reshape(m, m).T
    D = dense_expand(p)
    ne = int(sizes[:nblk - ns].sum())
    Sref = D[ne:, ne:] - D[ne:, :ne] @ np.linalg.solve(D[:ne, :ne], D[:ne, ne:])
    # forward error of a Schur complement ~ u * cond(D_ee) * |D|: allow 1e-12 * cond * max|D| (~4500 u)
    assert np.abs(S - Sref).max() <= 1e-12 * np.linalg.cond(D[:ne, :ne]) * np.abs(D).max()


def test_residual_and_backward_error_apis():
    """dd_aux_residual / dd_aux_backward_error against the oracle's block matvec and berr."""
    import torch
    import paper_2002_05019_b200 as dd
    from dd_inputs import random_rhs
    from oracle.block_ldlt import matvec_blocks, residual_berr
    for name, grid, sz in (("cfg1", (2, 2, 2), 50), ("cfg3", (2, 2, 2), 30)):
        p = dd_inputs.config(name, grid=grid, sizes=sz)
        s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=p.is_complex)
        vals = torch.from_numpy(p.values).cuda()
        s.factor(vals, p.val_offset)
        B = random_rhs(p.n, 5, p.is_complex, 1)
        X = random_rhs(p.n, 5, p.is_complex, 2)
        Bd, Xd = to_dev_colmajor(B, torch), to_dev_colmajor(X, torch)
        R = torch.empty_like(Bd.t().contiguous()).t()
        w = s._work(dd.dd_aux_solve_work_bytes(s.h, 5))
        dd.dd_aux_residual(s.h, s.factor_buf, vals, Bd, Xd, R, w)
        torch.cuda.synchronize()
        Rref = B - matvec_blocks(p, X)
        assert np.abs(R.cpu().numpy() - Rref).max() <= 1e-12 * np.abs(Rref).max()
        be = dd.dd_aux_backward_error(s.h, s.factor_buf, vals, Bd, Xd, w)
        np.testing.assert_allclose(be, residual_berr(p, X, B), rtol=1e-10)
        s.close()
