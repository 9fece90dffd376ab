"""Pins for oracle.bk (in-block restricted Bunch-Kaufman), CPU only.

Independent references: LAPACK ?sytrf (lower) via scipy for every pivot decision
(ipiv) and D; reconstruction P A P^T = L D L^T; numpy eigvalsh for Sylvester
inertia; SPEC worked examples (tests/golden/spec_bk_examples.json); exact
power-of-two scaling metamorphic.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg.lapack as lapack

from oracle.bk import bk_factor, d_matrix, inertia_of_d, ALPHA

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_bk_examples.json")


def _sym(rng, n, cplx, zero_diag=False):
    A = rng.standard_normal((n, n))
    if cplx:
        A = A + 1j * rng.standard_normal((n, n))
    A = A + A.T
    if zero_diag:
        np.fill_diagonal(A, 0)
    return A


def _recon(A, f):
    P = f["perm"]
    D = d_matrix(f["d"], f["e"], f["ipiv"])
    return np.linalg.norm(A[np.ix_(P, P)] - f["L"] @ D @ f["L"].T) / np.linalg.norm(A)


def test_alpha():
    assert ALPHA == pytest.approx(0.6403882032022076, abs=1e-15)


@pytest.mark.parametrize("cplx", [False, True])
def test_ipiv_and_d_match_lapack(cplx):
    """Every pivot decision equals LAPACK ?sytrf(lower); D agrees to rounding."""
    rng = np.random.default_rng(11)
    sytrf = lapack.zsytrf if cplx else lapack.dsytrf
    for trial in range(120):
        n = int(rng.integers(1, 140))
        A = _sym(rng, n, cplx, zero_diag=(trial % 4 == 0))
        f = bk_factor(A)
        lu, ipiv, info = sytrf(A, lower=1)
        assert info == 0
        np.testing.assert_array_equal(f["ipiv"], ipiv)
        np.testing.assert_allclose(f["d"], np.diag(lu), rtol=1e-9, atol=1e-11)
        sub = np.where(f["ipiv"][:-1] < 0, np.diag(lu, -1), 0)
        e_or = np.where(f["ipiv"][:-1] < 0, f["e"][:-1], 0)
        # e is stored on the first column of each 2x2 pivot only
        first = np.zeros(n - 1, dtype=bool)
        k = 0
        while k < n - 1:
            if f["ipiv"][k] < 0:
                first[k] = True
                k += 2
            else:
                k += 1
        np.testing.assert_allclose(e_or[first], sub[first], rtol=1e-9, atol=1e-11)
        assert _recon(A, f) < 1e-13


@pytest.mark.parametrize("cplx", [False, True])
def test_structure_of_factor(cplx):
    """L unit lower, perm a permutation; first-test 1x1 multipliers obey |l| <= 1/alpha."""
    rng = np.random.default_rng(5)
    for _ in range(30):
        n = int(rng.integers(2, 60))
        A = _sym(rng, n, cplx)
        f = bk_factor(A)
        L = f["L"]
        assert np.allclose(np.triu(L, 1), 0) and np.allclose(np.diag(L), 1)
        assert sorted(f["perm"]) == list(range(n))
        # first column, first BK test passed (|a_00| >= alpha*colmax): |l| <= 1/alpha
        from oracle.bk import cabs1
        if n > 1 and cabs1(A[0, 0]) >= ALPHA * cabs1(A[1:, 0]).max():
            # cabs1(z/w) <= 2 cabs1(z)/cabs1(w) for complex (cabs1 is within sqrt2 of |.|)
            assert cabs1(L[1:, 0]).max() <= (2.0 if cplx else 1.0) / ALPHA + 1e-12


def test_spec_worked_examples():
    g = json.load(open(GOLD))
    for c in g["cases"]:
        f = bk_factor(np.array(c["A"]))
        np.testing.assert_array_equal(f["L"], np.array(c["L"]))
        np.testing.assert_array_equal(f["d"], np.array(c["d"]))
        np.testing.assert_array_equal(f["e"], np.array(c["e"]))
        np.testing.assert_array_equal(f["perm"], np.array(c["perm"]))
        np.testing.assert_array_equal(f["ipiv"], np.array(c["ipiv"]))
    r = g["recon_20x20_zero_diag"]
    rng = np.random.default_rng(0)
    A = _sym(rng, r["n"], False, zero_diag=True)
    f = bk_factor(A)
    P = f["perm"]
    D = d_matrix(f["d"], f["e"], f["ipiv"])
    err = np.abs(A[np.ix_(P, P)] - f["L"] @ D @ f["L"].T).max()
    assert err <= r["tol_rel_inf"] * np.abs(A).sum(axis=1).max()


@pytest.mark.parametrize("cplx", [False, True])
def test_power_of_two_scaling(cplx):
    """Scaling A by 2^k leaves every decision and L bitwise identical, D scaled exactly."""
    rng = np.random.default_rng(3)
    A = _sym(rng, 57, cplx)
    f0 = bk_factor(A)
    for k in (-7, 3, 20):
        f1 = bk_factor(A * 2.0 ** k)
        np.testing.assert_array_equal(f0["ipiv"], f1["ipiv"])
        np.testing.assert_array_equal(f0["L"], f1["L"])
        np.testing.assert_array_equal(f0["d"] * 2.0 ** k, f1["d"])
        np.testing.assert_array_equal(f0["e"] * 2.0 ** k, f1["e"])


def test_inertia_sylvester():
    rng = np.random.default_rng(8)
    for trial in range(40):
        n = int(rng.integers(1, 90))
        A = _sym(rng, n, False, zero_diag=(trial % 3 == 0))
        f = bk_factor(A)
        ev = np.linalg.eigvalsh(A)
        assert inertia_of_d(f["d"], f["e"], f["ipiv"]) == (int((ev > 0).sum()), int((ev < 0).sum()), 0)
    # negation swaps (p, q); SPD gives (n, 0, 0)
    A = _sym(rng, 40, False)
    f, g = bk_factor(A), bk_factor(-A)
    p, q, z = inertia_of_d(f["d"], f["e"], f["ipiv"])
    assert inertia_of_d(g["d"], g["e"], g["ipiv"]) == (q, p, z)
    G = rng.standard_normal((40, 40))
    S = G.T @ G + 0.1 * np.eye(40)
    h = bk_factor(S)
    assert inertia_of_d(h["d"], h["e"], h["ipiv"]) == (40, 0, 0)


def test_zero_pivot_semantics():
    """LAPACK INFO semantics: first zero pivot reported, no elimination for that column."""
    A = np.zeros((4, 4))
    A[2, 2] = 5.0
    A[3, 2] = A[2, 3] = 1.0
    f = bk_factor(A)
    lu, ipiv, info = lapack.dsytrf(A, lower=1)
    assert f["info"] == info == 1
    np.testing.assert_array_equal(f["ipiv"], ipiv)
    assert f["d"][0] == 0.0 and f["d"][1] == 0.0
