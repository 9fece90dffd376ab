"""Host-only checks of the C-ABI library (no GPU needed): the .so loads, exports every
symbol include/dd_aux.h declares, and dd_aux_analyze's integer results (fill, levels,
flops, etree) equal the oracle's independent elimination game for the same order.
"""
import ctypes
import re
import os

import numpy as np
import pytest

import dd_inputs
import oracle
from oracle.block_ldlt import symbolic, flops_factor, flops_solve_per_rhs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    import paper_2002_05019_b200 as dd
    return dd


def test_header_symbols_exported():
    dd = _lib()
    hdr = open(os.path.join(ROOT, "include", "dd_aux.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|double|const char\*)\s+(dd_aux_\w+)\s*\(", hdr, re.M))
    assert declared == set(dd.EXPORTED_SYMBOLS)
    so = ctypes.CDLL(dd.LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert "sm_100a" in dd.dd_aux_version()


@pytest.mark.parametrize("name,kw,order", [
    ("cfg0", {}, "auto"),
    ("cfg1", {}, "nd"),
    ("cfg1", {"grid": (3, 3, 2), "sizes": 17}, "mindeg"),
    ("cfg3", {"grid": (4, 4, 2), "sizes": 8}, "auto"),
    ("cfg2", {"grid": (4, 4, 3), "sizes": lambda n, r: r.integers(3, 40, n)}, "auto"),
])
def test_analyze_matches_oracle_symbolic(name, kw, order):
    dd = _lib()
    p = dd_inputs.config(name, **kw)
    o = {"auto": dd.DD_ORDER_AUTO, "nd": dd.DD_ORDER_ND, "mindeg": dd.DD_ORDER_MINDEG}[order]
    h = dd.dd_aux_analyze(p.blk_size, p.colptr, p.rowidx, dd.DD_COMPLEX128 if p.is_complex else dd.DD_REAL64,
                          dd.dd_aux_default_options(o))
    try:
        info = dd.dd_aux_get_info(h)
        perm = dd.dd_aux_get_order(h)
        assert sorted(perm.tolist()) == list(range(p.nblk))
        sym = symbolic(p.nblk, p.colptr, p.rowidx, perm)
        mu = 4 if p.is_complex else 1
        assert info["n"] == p.n and info["nblk"] == p.nblk and info["nnzb_in"] == p.nnzb
        assert info["nnzb_filled"] == p.nblk + len(sym["orig"]) + len(sym["fill"])
        assert info["flops_factor"] == pytest.approx(flops_factor(p.blk_size, sym, mu), rel=1e-12)
        assert info["flops_solve_per_rhs"] == pytest.approx(flops_solve_per_rhs(p.blk_size, sym, mu), rel=1e-12)
        parent, level, nnz = dd.dd_aux_get_etree(h)
        assert nnz == sum(len(s) for s in sym["struct"])
        np.testing.assert_array_equal(parent, sym["parent"])
        np.testing.assert_array_equal(level, sym["level"])
        assert info["n_levels"] == int(sym["level"].max()) + 1
        assert info["factor_bytes"] > 0 and info["work_bytes"] > 0
    finally:
        dd.dd_aux_destroy(h)


def test_cfg1_nd_quality():
    """Graph ND without METIS reaches the geometric-ND flop count of SURVEY.md App. A (4.24e11)."""
    dd = _lib()
    p = dd_inputs.config("cfg1", sizes=1)  # topology only; flops scale as s^3
    h = dd.dd_aux_analyze(p.blk_size * 256, p.colptr, p.rowidx, dd.DD_REAL64, dd.dd_aux_default_options(dd.DD_ORDER_ND))
    info = dd.dd_aux_get_info(h)
    dd.dd_aux_destroy(h)
    assert info["flops_factor"] <= 4.3e11
    assert info["n_levels"] <= 40


def test_auto_picks_lower_flops():
    dd = _lib()
    p = dd_inputs.config("cfg3", grid=(4, 4, 4), sizes=16)
    res = {}
    for o in (dd.DD_ORDER_AUTO, dd.DD_ORDER_ND, dd.DD_ORDER_MINDEG):
        h = dd.dd_aux_analyze(p.blk_size, p.colptr, p.rowidx, dd.DD_COMPLEX128, dd.dd_aux_default_options(o))
        res[o] = dd.dd_aux_get_info(h)["flops_factor"]
        dd.dd_aux_destroy(h)
    assert res[dd.DD_ORDER_AUTO] == min(res[dd.DD_ORDER_ND], res[dd.DD_ORDER_MINDEG])


def test_user_and_natural_order():
    dd = _lib()
    p = dd_inputs.config("cfg0")
    h = dd.dd_aux_analyze(p.blk_size, p.colptr, p.rowidx, dd.DD_REAL64, dd.dd_aux_default_options(user_order=[2, 0, 3, 1]))
    assert dd.dd_aux_get_order(h).tolist() == [2, 0, 3, 1]
    dd.dd_aux_destroy(h)
    h = dd.dd_aux_analyze(p.blk_size, p.colptr, p.rowidx, dd.DD_REAL64, dd.dd_aux_default_options(dd.DD_ORDER_NATURAL))
    assert dd.dd_aux_get_order(h).tolist() == [0, 1, 2, 3]
    dd.dd_aux_destroy(h)


@pytest.mark.parametrize("bad,rule", [
    (dict(colptr=[0, 1, 2], rowidx=[0, 0]), "diagonal"),
    (dict(colptr=[0, 2, 3], rowidx=[0, 0, 1]), "unsorted"),
    (dict(colptr=[0, 1, 3], rowidx=[0, 1, 0]), "upper"),
    (dict(colptr=[0, 2, 3], rowidx=[0, 5, 1]), "range"),
])
def test_pattern_errors(bad, rule):
    dd = _lib()
    with pytest.raises(dd.DDAuxError) as ei:
        dd.dd_aux_analyze([3, 4], bad["colptr"], bad["rowidx"])
    assert ei.value.code == dd.DD_ERR_PATTERN
    assert rule in str(ei.value)


def test_argument_errors():
    dd = _lib()
    with pytest.raises(dd.DDAuxError) as ei:
        dd.dd_aux_analyze([3, 0], [0, 1, 2], [0, 1])
    assert ei.value.code == dd.DD_ERR_PATTERN
    with pytest.raises(dd.DDAuxError) as ei:
        dd.dd_aux_analyze([3], [0, 1], [0], dtype=7)
    assert ei.value.code == -5
    with pytest.raises(dd.DDAuxError):
        dd.dd_aux_default_options(user_order=[0, 0])  # not a permutation -> rejected at analyze
        dd.dd_aux_analyze([3, 3], [0, 1, 2], [0, 1], opt=dd.dd_aux_default_options(user_order=[0, 0]))


def test_assemble_tables_host():
    """f1 host logic: the assembly's descriptor tables are sized without a GPU and invalid
    clique lists are rejected (DD_ERR_PATTERN) before anything is enqueued."""
    dd = _lib()
    p = dd_inputs.config("cfg0")
    h = dd.dd_aux_analyze(p.blk_size, p.colptr, p.rowidx)
    try:
        cl = [c for _, c in p.cliques]
        ptr, blk = dd.cliques_to_csr(cl)
        nb = dd.dd_aux_assemble_work_bytes(h, ptr, blk)
        # one 32-column chunk per block (s = 32) and one contributor per (clique, lower pair)
        ncon = sum(len(c) * (len(c) + 1) // 2 for c in cl)
        assert nb == (-(-p.nnzb * 32 // 256) * 256) + (-(-ncon * 24 // 256) * 256)
        assert dd.dd_aux_assemble_work_bytes(h, *dd.cliques_to_csr([])) >= 0
        for bad, rule in [([[1, 0]], "ascending"), ([[0, 9]], "range"), ([[0, 0]], "ascending")]:
            with pytest.raises(dd.DDAuxError) as ei:
                dd.dd_aux_assemble_work_bytes(h, *dd.cliques_to_csr(bad))
            assert ei.value.code == dd.DD_ERR_PATTERN and rule in str(ei.value)
        # cfg0 is a 4-cycle: interfaces 0 and 3 never share a subdomain, (3, 0) is not in the pattern
        with pytest.raises(dd.DDAuxError) as ei:
            dd.dd_aux_assemble_work_bytes(h, *dd.cliques_to_csr([[0, 3]]))
        assert ei.value.code == dd.DD_ERR_PATTERN and "not in the pattern" in str(ei.value)
    finally:
        dd.dd_aux_destroy(h)


def test_interface_size_limit():
    """Interfaces above the in-block kernel's shared-memory limit (3328 real / 1664 complex DoFs)
    are rejected at analyze (DD_ERR_PATTERN); the limits themselves are accepted."""
    dd = _lib()
    for dt, lim in ((dd.DD_REAL64, 3328), (dd.DD_COMPLEX128, 1664)):
        with pytest.raises(dd.DDAuxError) as ei:
            dd.dd_aux_analyze([lim + 1], [0, 1], [0], dtype=dt)
        assert ei.value.code == dd.DD_ERR_PATTERN and str(lim) in str(ei.value)
        h = dd.dd_aux_analyze([lim], [0, 1], [0], dtype=dt)
        dd.dd_aux_destroy(h)


def test_schur_mode_host_tables():
    """dd_aux_analyze_partial (f3): kept blocks last, eliminated part scheduled alone, cliques =
    each subdomain's interfaces, flops / levels only over the eliminated positions."""
    import paper_2002_05019_b200 as dd
    from dd_inputs.fem import fem_dd, schur_block_problem
    import oracle
    m = fem_dd(2, 2, 2, 6, seed=0)
    prob, ns, tgt, grp, auxs, info = schur_block_problem(m, leaf=16)
    o = dd.dd_aux_default_options(dd.DD_ORDER_NATURAL)
    h = dd.dd_aux_analyze_partial(prob.blk_size, prob.colptr, prob.rowidx, tgt, grp, auxs, dd.DD_REAL64, o)
    inf = dd.dd_aux_get_info(h)
    assert inf["n_schur"] == ns and inf["n_groups"] == m.nsub and inf["n_aux_dof"] == m.n_dual
    assert dd.dd_aux_schur_cliques(h) == [m.sub_ifaces[p] for p in range(m.nsub)]
    order = dd.dd_aux_get_order(h)
    assert list(order[-ns:]) == list(range(prob.nblk - ns, prob.nblk))
    sym = oracle.symbolic(prob.nblk, prob.colptr, prob.rowidx, list(order))
    ne = prob.nblk - ns
    fl = sum(float(prob.blk_size[k]) ** 3 / 3 + sum(float(prob.blk_size[i]) for i in sym["struct"][k]) *
             float(prob.blk_size[k]) ** 2 + sum(float(prob.blk_size[i]) for i in sym["struct"][k]) ** 2 *
             float(prob.blk_size[k]) for k in order[:ne])
    assert inf["flops_factor"] == pytest.approx(fl, rel=1e-12)
    parent, level, _ = dd.dd_aux_get_etree(h)
    assert inf["n_levels"] == int(max(level[k] for k in order[:ne])) + 1
    # subdomains are independent: no eliminated block's struct leaves its subdomain
    nbp = info["nblk_per_sub"]
    for k in order[:ne]:
        p = k // nbp
        for i in sym["struct"][k]:
            assert (i < ne and i // nbp == p) or (i >= ne and grp[i - ne] == p)
    # errors: size mismatch, bad target, n_schur out of range
    with pytest.raises(dd.DDAuxError):
        dd.dd_aux_analyze_partial(prob.blk_size, prob.colptr, prob.rowidx, tgt, grp, auxs + 1, dd.DD_REAL64, o)
    with pytest.raises(dd.DDAuxError):
        dd.dd_aux_analyze_partial(prob.blk_size, prob.colptr, prob.rowidx, tgt + 100, grp, auxs, dd.DD_REAL64, o)
    dd.dd_aux_destroy(h)


def test_table_validation_random_patterns():
    """compute-sanitizer is closed on the GPU pool: instead every descriptor table the kernels index
    through is bounds-checked on the host (dd_aux_validate) over random block patterns (1-40 DoF
    blocks, 2-30 blocks, every order), the BASELINE patterns, and Schur-mode handles."""
    import paper_2002_05019_b200 as dd
    from dd_inputs.fem import fem_dd, schur_block_problem
    rng = np.random.default_rng(123)
    for trial in range(150):
        nblk = int(rng.integers(2, 31))
        sizes = rng.integers(1, 41, nblk)
        dens = rng.uniform(0.05, 1.0)
        edges = [[u, v] for u in range(nblk) for v in range(u) if rng.random() < dens]
        cp, ri = dd_inputs.block_pattern_from_cliques(nblk, edges)
        order = [dd.DD_ORDER_AUTO, dd.DD_ORDER_ND, dd.DD_ORDER_MINDEG, dd.DD_ORDER_NATURAL][trial % 4]
        h = dd.dd_aux_analyze(sizes, cp, ri, dd.DD_COMPLEX128 if trial % 3 == 0 else dd.DD_REAL64,
                              dd.dd_aux_default_options(order))
        dd.dd_aux_validate(h)
        dd.dd_aux_destroy(h)
    for name, kw in [("cfg1", {}), ("cfg2", dict(grid=(4, 4, 3))), ("cfg3", {})]:
        c = dd_inputs.CONFIGS[name]
        g = kw.get("grid", c["grid"])
        pairs, bs, cl, cp, ri, vo, tot = dd_inputs._topology(*g, c["sizes"], np.random.default_rng(0), c["topology"])
        h = dd.dd_aux_analyze(bs, cp, ri, dd.DD_COMPLEX128 if c["complex_"] else dd.DD_REAL64)
        dd.dd_aux_validate(h)
        dd.dd_aux_destroy(h)
    m = fem_dd(3, 2, 2, 8, seed=1)
    prob, ns, tgt, grp, auxs, info = schur_block_problem(m, leaf=24)
    h = dd.dd_aux_analyze_partial(prob.blk_size, prob.colptr, prob.rowidx, tgt, grp, auxs, dd.DD_REAL64,
                                  dd.dd_aux_default_options(dd.DD_ORDER_AUTO))
    dd.dd_aux_validate(h)
    dd.dd_aux_destroy(h)


def test_schur_mode_argument_errors():
    """dd_aux_analyze_partial rejects bad Schur descriptions (LAPACK-style argument codes)."""
    import paper_2002_05019_b200 as dd
    sizes = np.array([3, 4, 5, 6], dtype=np.int64)
    cp, ri = dd_inputs.block_pattern_from_cliques(4, [[0, 1, 2, 3]])
    o = dd.dd_aux_default_options(dd.DD_ORDER_NATURAL)
    ok = dict(schur_target=[0, 1], schur_group=[0, 0], aux_blk_size=[5, 6])
    h = dd.dd_aux_analyze_partial(sizes, cp, ri, **ok, opt=o)
    assert dd.dd_aux_get_info(h)["n_schur"] == 2
    dd.dd_aux_validate(h)
    dd.dd_aux_destroy(h)
    bad = [dict(schur_target=[], schur_group=[], aux_blk_size=[5]),                  # n_schur = 0
           dict(schur_target=[0, 1, 2, 3], schur_group=[0] * 4, aux_blk_size=sizes),  # n_schur = nblk
           dict(schur_target=[0, 0], schur_group=[0, 0], aux_blk_size=[5]),           # same target twice in a group
           dict(schur_target=[0, 1], schur_group=[0, -1], aux_blk_size=[5, 6]),       # negative group
           dict(schur_target=[1, 0], schur_group=[0, 1], aux_blk_size=[5, 6])]        # size mismatch
    for kw in bad:
        with pytest.raises(dd.DDAuxError):
            dd.dd_aux_analyze_partial(sizes, cp, ri, **kw, opt=o)
