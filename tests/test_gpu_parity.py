"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Tolerances are the north_star's (BASELINE.json):
  solution relative difference <= 1e-9 (per column, inf-norm, max over columns)
  backward error ||A x - b||_inf / (||A||_inf ||x||_inf) <= 1e-12
  identical inertia for real cases.
Pivot decisions (ipiv) are unique up to near-ties; on isolated blocks they must equal the
oracle (which equals LAPACK ?sytrf).
"""
import numpy as np
import pytest

import dd_inputs
from dd_inputs import Problem, block_pattern_from_cliques, random_rhs
import oracle
from oracle.block_ldlt import residual_berr
from oracle.bk import bk_factor

from tests._gpu import run_gpu, rel_diff

pytestmark = pytest.mark.gpu

TOL_REL = 1e-9
TOL_BERR = 1e-12


def _parity(p, nrhs=3, seed=0, order=None, refine=1, check_inertia=True):
    import paper_2002_05019_b200 as dd
    B = random_rhs(p.n, nrhs, p.is_complex, seed)
    X, finfo, s = run_gpu(p, B, order=order, refine=refine, keep=True)
    perm = s.order()
    s.close()
    F = oracle.block_factor(p, list(perm))
    Xo, _, bo = oracle.refine_solve(p, F, B, refine)
    berr = residual_berr(p, X, B)
    assert berr.max() <= TOL_BERR, berr.max()
    assert bo.max() <= TOL_BERR
    rd = rel_diff(X, Xo)
    assert rd <= TOL_REL, rd
    if check_inertia and not p.is_complex:
        assert (finfo["npos"], finfo["nneg"], finfo["nzero"]) == oracle.inertia(F)
    assert finfo["n2x2"] >= 0
    return X, finfo


def test_cfg0():
    p = dd_inputs.config("cfg0")
    _parity(p, nrhs=4)


@pytest.mark.parametrize("perm", [[0, 1, 2, 3], [3, 2, 1, 0], [1, 2, 0, 3]])
def test_cfg0_user_orders(perm):
    import paper_2002_05019_b200 as dd
    p = dd_inputs.config("cfg0")
    B = random_rhs(p.n, 4, False, 1)
    X, finfo, _ = run_gpu(p, B, user_order=perm)
    F = oracle.block_factor(p, perm)
    Xo, _, _ = oracle.refine_solve(p, F, B, 1)
    assert rel_diff(X, Xo) <= TOL_REL
    assert (finfo["npos"], finfo["nneg"], finfo["nzero"]) == oracle.inertia(F)


@pytest.mark.parametrize("name,grid,sizes", [
    ("cfg1", (2, 2, 2), 96),                                   # several K1 panels, one K3 tile
    ("cfg1", (3, 3, 2), 150),                                  # ragged tiles (150 = 128 + 22)
    ("cfg2", (3, 3, 3), lambda n, r: r.integers(60, 300, n)),  # unstructured-like, odd sizes
    ("cfg3", (2, 2, 2), 80),                                   # complex symmetric
    ("cfg3", (3, 2, 2), 130),                                  # complex, ragged
])
def test_scaled_configs(name, grid, sizes):
    p = dd_inputs.config(name, grid=grid, sizes=sizes)
    _parity(p, nrhs=70)  # 70 rhs: two rhs tiles, ragged


def _random_block_problem(rng, cplx):
    nblk = int(rng.integers(2, 9))
    sizes = rng.integers(1, 41, nblk)
    dens = rng.uniform(0.3, 1.0)
    edges = [(u, v) for u in range(nblk) for v in range(u) if rng.random() < dens]
    colptr, rowidx = block_pattern_from_cliques(nblk, [list(e) for e in edges])
    off, tot = [], 0
    for j in range(nblk):
        for q in range(colptr[j], colptr[j + 1]):
            off.append(tot)
            tot += int(sizes[rowidx[q]]) * int(sizes[j])
    vals = rng.standard_normal(tot)
    if cplx:
        vals = vals + 1j * rng.standard_normal(tot)
    p = Problem(np.asarray(sizes, dtype=np.int64), colptr, rowidx, vals, np.asarray(off, dtype=np.int64), [])
    if rng.random() < 0.3:
        for j in range(nblk):
            np.fill_diagonal(p.block(int(colptr[j])), 0.0)
    return p


def test_spec_corpus():
    from dd_inputs import dense_expand
    rng = np.random.default_rng(77)
    done = 0
    for trial in range(120):
        if done == 40:
            break
        p = _random_block_problem(rng, cplx=(trial % 2 == 1))
        if np.linalg.cond(dense_expand(p)) > 1e10:
            continue
        done += 1
        _parity(p, nrhs=2, seed=trial)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("s", [1, 2, 31, 32, 33, 64, 100, 257, 700])
def test_isolated_block_pivots(s, cplx):
    """One diagonal block alone: every BK decision equals the oracle's (== LAPACK)."""
    rng = np.random.default_rng(s + 1000 * cplx)
    A = rng.standard_normal((s, s))
    if cplx:
        A = A + 1j * rng.standard_normal((s, s))
    A = A + A.T
    if s % 2 == 1:
        np.fill_diagonal(A, 0.0)  # forces 2x2 pivots
    p = Problem(np.array([s]), np.array([0, 1]), np.array([0], dtype=np.int32),
                np.asfortranarray(A).ravel(order="F"), np.array([0]), [])
    X, finfo, sv = run_gpu(p, random_rhs(s, 3, cplx, 0), keep=True)
    piv = sv.pivots()
    sv.close()
    f = bk_factor(A)
    np.testing.assert_array_equal(piv["ipiv"], f["ipiv"])
    np.testing.assert_array_equal(piv["perm"], f["perm"])
    np.testing.assert_allclose(piv["d"], f["d"], rtol=1e-10, atol=1e-12 * np.abs(A).max())


def test_multi_rhs_columns_bitwise_equal_single():
    """k columns solved together are bit-identical to k single solves."""
    import torch
    from tests._gpu import to_dev_colmajor
    p = dd_inputs.config("cfg1", grid=(2, 2, 2), sizes=70)
    B = random_rhs(p.n, 130, False, 3)   # three right-hand-side tiles of 64
    X, _, s = run_gpu(p, B, keep=True)
    for j in (0, 4, 8, 129):
        b = to_dev_colmajor(B[:, j:j + 1], torch)
        s.solve_(b)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(b.cpu().numpy()[:, 0], X[:, j])
    s.close()


def test_deterministic_repeat():
    p = dd_inputs.config("cfg3", grid=(2, 2, 2), sizes=40)
    B = random_rhs(p.n, 5, True, 0)
    X1, f1, _ = run_gpu(p, B)
    X2, f2, _ = run_gpu(p, B)
    np.testing.assert_array_equal(X1, X2)


def test_negation_swaps_inertia_and_spd():
    p = dd_inputs.config("cfg1", grid=(2, 2, 2), sizes=48)
    B = random_rhs(p.n, 2, False, 0)
    _, f1, _ = run_gpu(p, B)
    neg = Problem(p.blk_size, p.colptr, p.rowidx, -p.values, p.val_offset, [])
    _, f2, _ = run_gpu(neg, B)
    assert (f2["npos"], f2["nneg"], f2["nzero"]) == (f1["nneg"], f1["npos"], f1["nzero"])
    assert f1["npos"] + f1["nneg"] == p.n


def test_zero_pivot_and_errors():
    import torch
    import paper_2002_05019_b200 as dd
    A = np.zeros((4, 4))
    A[2, 2] = 5.0
    A[3, 2] = A[2, 3] = 1.0
    p = Problem(np.array([4]), np.array([0, 1]), np.array([0], dtype=np.int32), A.ravel(order="F"), np.array([0]), [])
    X, finfo, s = run_gpu(p, None, keep=True)
    assert finfo["rc"] == dd.DD_ZERO_PIVOT and finfo["first_zero_pivot"] == 1
    with pytest.raises(dd.DDAuxError) as ei:
        s.solve_(torch.zeros(4, 1, dtype=torch.float64, device="cuda"))
    assert ei.value.code == dd.DD_ERR_SINGULAR
    s.close()
    q = dd_inputs.config("cfg0")
    s2 = dd.AuxSolver(q.blk_size, q.colptr, q.rowidx)
    s2.factor_buf = torch.empty(s2.info["factor_bytes"], dtype=torch.uint8, device="cuda")
    with pytest.raises(dd.DDAuxError) as ei:
        s2.solve_(torch.zeros(q.n, 1, dtype=torch.float64, device="cuda"))
    assert ei.value.code == dd.DD_ERR_NOT_FACTORED
    s2.close()


def test_cfg1_full_size():
    """BASELINE configs[1] at full size (n = 36,864, ND order), nrhs 64, vs the oracle."""
    p = dd_inputs.config("cfg1")
    _parity(p, nrhs=64)


def test_adaptive_refinement_policy():
    """refine_tol: the correction is skipped on the device iff every column's berr <= tol."""
    import torch
    import paper_2002_05019_b200 as dd
    from tests._gpu import to_dev_colmajor
    p = dd_inputs.config("cfg3", grid=(2, 2, 2), sizes=60)
    B = random_rhs(p.n, 6, True, 5)
    s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=True)
    vals = torch.from_numpy(p.values).cuda()
    s.factor(vals, p.val_offset)
    out = {}
    for name, steps, tol in [("plain", 0, 0.0), ("always", 1, 0.0), ("skip", 1, 1.0), ("tight", 1, 1e-300)]:
        dd.dd_aux_set_refine(s.h, steps, tol)
        b = to_dev_colmajor(B, torch)
        s.solve_(b)
        torch.cuda.synchronize()
        out[name] = b.cpu().numpy()
    s.close()
    np.testing.assert_array_equal(out["skip"], out["plain"])     # converged -> no correction applied
    np.testing.assert_array_equal(out["tight"], out["always"])   # not converged -> same as always
    assert residual_berr(p, out["always"], B).max() <= TOL_BERR


def test_complex_3m_parity():
    """Complex Schur update with the 3M (Gauss) product: same tolerances as 4M."""
    import torch
    import paper_2002_05019_b200 as dd
    from tests._gpu import to_dev_colmajor
    p = dd_inputs.config("cfg3", grid=(3, 2, 2), sizes=100)
    B = random_rhs(p.n, 5, True, 2)
    s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=True, complex_3m=True)
    s.factor(torch.from_numpy(p.values).cuda(), p.val_offset)
    b = to_dev_colmajor(B, torch)
    s.solve_(b)
    torch.cuda.synchronize()
    X = b.cpu().numpy()
    F = oracle.block_factor(p, list(s.order()))
    s.close()
    Xo, _, _ = oracle.refine_solve(p, F, B, 1)
    assert residual_berr(p, X, B).max() <= TOL_BERR
    assert rel_diff(X, Xo) <= TOL_REL


@pytest.mark.parametrize("name,grid,sizes,tol", [("cfg1", (3, 3, 2), 40, 0.0), ("cfg3", (2, 2, 2), 24, 1e-14)])
def test_cuda_graphs_bitwise_equal_direct(name, grid, sizes, tol):
    """options.use_graphs (a5): the captured-and-replayed factor level loop and solve give the
    bitwise result of direct launches, on first capture, on replay with new right-hand sides and
    after a re-capture for a different buffer; refine_tol > 0 exercises the in-graph ||A||."""
    import torch
    import paper_2002_05019_b200 as dd
    from tests._gpu import to_dev_colmajor
    p = dd_inputs.config(name, grid=grid, sizes=sizes)
    vals = torch.from_numpy(p.values).cuda()
    outs = {}
    for graphs in (False, True):
        s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=p.is_complex, use_graphs=graphs, refine_tol=tol)
        res = []
        for rep in range(2):
            rc, fi = s.factor(vals, p.val_offset)
            assert rc == dd.DD_OK
            for seed in (0, 1):
                B = random_rhs(p.n, 5, p.is_complex, seed)
                Bd = to_dev_colmajor(B, torch)
                s.solve_(Bd)
                torch.cuda.synchronize()
                res.append(Bd.cpu().numpy())
        # a different right-hand-side buffer forces a re-capture of the solve graph
        B = random_rhs(p.n, 3, p.is_complex, 2)
        Bd = to_dev_colmajor(B, torch)
        s.solve_(Bd)
        torch.cuda.synchronize()
        res.append(Bd.cpu().numpy())
        tr = dd.dd_aux_get_trace(s.h, reset=True)
        outs[graphs] = (res, sum(v["launches"] for v in tr.values()))
        s.close()
    for a, b in zip(outs[False][0], outs[True][0]):
        assert np.array_equal(a, b)
    assert outs[False][1] == outs[True][1]  # replayed graphs account for the same kernel launches
    X = outs[True][0][-1]
    assert residual_berr(p, X, random_rhs(p.n, 3, p.is_complex, 2)).max() <= TOL_BERR


@pytest.mark.parametrize("name,grid,sizes", [("cfg2", (3, 3, 2), lambda n, rng: rng.integers(40, 301, n)),
                                             ("cfg3", (3, 2, 2), 90)])
def test_factor_solve_bitwise_reproducible(name, grid, sizes):
    """Two independent factorizations + solves of the same bytes are bitwise equal: every Schur
    update tile sums its contributors in a fixed order and reaches its target (and the solve
    updates reach y) through exactly ONE L2 reduction per element and launch (DESIGN.md section 7,
    K3 / K5), so nothing depends on the order the reductions arrive in.  Ragged interface sizes:
    edge tiles, multi-level gathered K and the split-K backward update all take part."""
    import torch
    import paper_2002_05019_b200 as dd
    from tests._gpu import to_dev_colmajor
    p = dd_inputs.config(name, grid=grid, sizes=sizes)
    vals = torch.from_numpy(p.values).cuda()
    B = random_rhs(p.n, 70, p.is_complex, 5)
    outs = []
    for rep in range(2):
        s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=p.is_complex)
        rc, fi = s.factor(vals, p.val_offset)
        assert rc == dd.DD_OK
        Bd = to_dev_colmajor(B, torch)
        s.solve_(Bd)
        torch.cuda.synchronize()
        piv = s.pivots()
        outs.append((Bd.cpu().numpy(), piv, fi["max_abs_L"]))
        s.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][2] == outs[1][2]
    for k in outs[0][1]:
        assert np.array_equal(np.asarray(outs[0][1][k]), np.asarray(outs[1][1][k])), k
    assert residual_berr(p, outs[0][0], B).max() <= TOL_BERR


def test_complex_4m_parity():
    """Complex Schur update with the four-real-product (4M) form (options.complex_3m = 0)."""
    import torch
    import paper_2002_05019_b200 as dd
    from tests._gpu import to_dev_colmajor
    p = dd_inputs.config("cfg3", grid=(3, 2, 2), sizes=90)
    B = random_rhs(p.n, 33, True, 4)
    s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, complex_=True, complex_3m=False)
    s.factor(torch.from_numpy(p.values).cuda(), p.val_offset)
    b = to_dev_colmajor(B, torch)
    s.solve_(b)
    torch.cuda.synchronize()
    X = b.cpu().numpy()
    F = oracle.block_factor(p, list(s.order()))
    s.close()
    Xo, _, _ = oracle.refine_solve(p, F, B, 1)
    assert residual_berr(p, X, B).max() <= TOL_BERR
    assert rel_diff(X, Xo) <= TOL_REL


def test_padded_ldb_zero_rhs_and_two_refinement_steps():
    """ldb > n (a column-major view into a taller buffer), nrhs = 0 as a no-op, refine_steps = 2."""
    import torch
    import paper_2002_05019_b200 as dd
    p = dd_inputs.config("cfg1", grid=(2, 2, 2), sizes=50)
    B = random_rhs(p.n, 4, False, 9)
    s = dd.AuxSolver(p.blk_size, p.colptr, p.rowidx, refine_steps=2)
    vals = torch.from_numpy(p.values).cuda()
    s.factor(vals, p.val_offset)
    ld = p.n + 13
    buf = torch.full((4, ld), 7.0, dtype=torch.float64, device="cuda")
    buf[:, :p.n] = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    Bv = buf.t()[:p.n]                       # n x 4, stride (1, ld)
    w = s._work(dd.dd_aux_solve_work_bytes(s.h, 4))
    dd.dd_aux_solve(s.h, s.factor_buf, vals, Bv, w, nrhs=4, ldb=ld)
    dd.dd_aux_solve(s.h, s.factor_buf, vals, Bv, w, nrhs=0, ldb=ld)   # no-op
    torch.cuda.synchronize()
    X = Bv.cpu().numpy()
    assert torch.all(buf[:, p.n:] == 7.0)    # padding rows untouched
    F = oracle.block_factor(p, list(s.order()))
    s.close()
    Xo, _, _ = oracle.refine_solve(p, F, B, 2)
    assert rel_diff(X, Xo) <= TOL_REL
    assert residual_berr(p, X, B).max() <= TOL_BERR


@pytest.mark.parametrize("s,cplx", [(3328, False), (1664, True)])
def test_isolated_max_size_block(s, cplx):
    """The largest supported interfaces (3328 real / 1664 complex DoFs, include/dd_aux.h):
    backward error bound, and for the real case Sylvester inertia against numpy's eigvalsh (the
    oracle's O(s^3) Python BK is too slow at this size)."""
    rng = np.random.default_rng(s)
    A = rng.standard_normal((s, s))
    if cplx:
        A = A + 1j * rng.standard_normal((s, s))
    A = A + A.T
    p = Problem(np.array([s]), np.array([0, 1]), np.array([0], dtype=np.int32),
                np.asfortranarray(A).ravel(order="F"), np.array([0]), [])
    B = random_rhs(s, 2, cplx, 3)
    X, finfo, _ = run_gpu(p, B)
    assert residual_berr(p, X, B).max() <= TOL_BERR
    if not cplx:
        ev = np.linalg.eigvalsh(A)
        assert (finfo["npos"], finfo["nneg"], finfo["nzero"]) == (int((ev > 0).sum()), int((ev < 0).sum()), 0)
