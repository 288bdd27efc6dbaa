"""Pins of the oracle's diagonal preconditioning (R-3):
Ruiz equilibration + one Pock-Chambolle (alpha = 1) pass, and the scaled solve
whose termination is the ORIGINAL LP's.  `-m "not gpu"`.

Each pin is independent of the oracle's code: closed forms (diagonal matrices),
published properties of the two scalings (Pock & Chambolle 2011: with
sigma_i = 1/sum_j|a_ij|, tau_j = 1/sum_i|a_ij| the scaled operator has norm <= 1;
Ruiz 2001: the iteration drives every row and column infinity-norm to 1), the
factorisation A^ = diag(r) A diag(s) recomputed densely with numpy, and the KKT
conditions of the original LP recomputed in numpy at the returned point.
"""
import numpy as np
import pytest

import lpgen
import oracle


def _dense(olp):
    A = np.zeros((olp.m, olp.n))
    for i in range(olp.m):
        for k in range(olp.Ap[i], olp.Ap[i + 1]):
            A[i, olp.Aj[k]] = olp.Ax[k]
    return A


def _lp_from_dense(A, seed=0):
    m, n = A.shape
    rows, cols = np.nonzero(A.T)          # CSR of A^T: row = column of A
    ATp = np.zeros(n + 1, np.int32)
    np.add.at(ATp, rows + 1, 1)
    ATp = np.cumsum(ATp).astype(np.int32)
    import types
    rng = np.random.default_rng(seed)
    return types.SimpleNamespace(m=m, n=n, ATp=ATp, ATj=cols.astype(np.int32), ATx=A.T[rows, cols].copy(),
                                 b=rng.standard_normal(m), c=rng.uniform(0, 1, n), lb=np.zeros(n),
                                 ub=np.full(n, np.inf))


def test_diagonal_matrix_closed_form():
    d = np.array([4.0, 0.25, 9.0, 1e-6, 2.0])
    olp = oracle.OracleLP(_lp_from_dense(np.diag(d)))
    sl = oracle.ScaledLP(olp, ruiz_iters=1, pc=0)
    np.testing.assert_allclose(sl.r, 1 / np.sqrt(d), rtol=1e-15)
    np.testing.assert_allclose(sl.s, 1 / np.sqrt(d), rtol=1e-15)
    np.testing.assert_allclose(_dense(sl.olp), np.eye(5), rtol=0, atol=1e-15)
    # further passes (Ruiz or PC) leave an identity alone
    sl2 = oracle.ScaledLP(olp, ruiz_iters=5, pc=1)
    np.testing.assert_allclose(_dense(sl2.olp), np.eye(5), atol=1e-15)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_pock_chambolle_operator_norm_at_most_one(seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((30, 50)) * (rng.uniform(0, 1, (30, 50)) < 0.2) * np.exp(rng.normal(0, 3, (30, 1)))
    A[A == 0] = 0.0
    keep = np.abs(A).sum(1) > 0
    A = A[keep]
    olp = oracle.OracleLP(_lp_from_dense(A, seed))
    sl = oracle.ScaledLP(olp, ruiz_iters=0, pc=1)
    assert np.linalg.norm(_dense(sl.olp), 2) <= 1.0 + 1e-12


def test_ruiz_equilibrates_row_and_column_max():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((40, 60)) * np.exp(rng.normal(0, 2, (40, 1))) * np.exp(rng.normal(0, 2, (1, 60)))
    A *= rng.uniform(0, 1, A.shape) < 0.3
    A = A[np.abs(A).sum(1) > 0][:, np.abs(A).sum(0) > 0] if (np.abs(A).sum(0) > 0).all() else A
    olp = oracle.OracleLP(_lp_from_dense(A))
    sl = oracle.ScaledLP(olp, ruiz_iters=40, pc=0)
    Ah = np.abs(_dense(sl.olp))
    rmax = Ah.max(1)[Ah.max(1) > 0]
    cmax = Ah.max(0)[Ah.max(0) > 0]
    assert np.all(np.abs(rmax - 1) < 1e-6) and np.all(np.abs(cmax - 1) < 1e-6)


@pytest.mark.parametrize("name", ["c1", "c2-s", "c4-s"])
def test_scaled_matrix_is_diag_r_A_diag_s(name):
    olp = oracle.OracleLP(lpgen.config(name))
    sl = oracle.ScaledLP(olp, 10, 1)
    A, Ah = _dense(olp), _dense(sl.olp)
    ref = sl.r[:, None] * A * sl.s[None, :]
    assert np.abs(Ah - ref).max() <= 1e-13 * np.abs(ref).max()
    np.testing.assert_allclose(sl.olp.b, sl.r * olp.b, rtol=1e-15)
    np.testing.assert_allclose(sl.olp.c, sl.s * olp.c, rtol=1e-15)


@pytest.mark.parametrize("name", ["c1", "c2-s"])
def test_certificate_maps_to_scaled_optimum(name):
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    sl = oracle.ScaledLP(olp, 10, 1)
    sc = oracle.score(sl.olp, lp.x0 / sl.s, lp.y0 / sl.r)
    assert sc["score"] < 1e-12


@pytest.mark.parametrize("name", ["c1", "c2-s", "c4-s"])
def test_scaled_solve_meets_original_criteria(name):
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    x, y, r, sl = oracle.solve_scaled(olp)
    assert r["status"] == 0
    A = _dense(olp)
    z = lp.c - A.T @ y
    rp = np.linalg.norm(lp.b - A @ x)
    lo, hi = np.isfinite(lp.lb), np.isfinite(lp.ub)
    rd = np.linalg.norm(z - np.where(lo, np.maximum(z, 0), 0) + np.where(hi, np.maximum(-z, 0), 0))
    pobj = lp.c @ x
    dobj = lp.b @ y + np.sum(np.where(lo, lp.lb * np.maximum(z, 0), 0)) - np.sum(
        np.where(hi, np.where(hi, lp.ub, 0) * np.maximum(-z, 0), 0))
    tol = 1e-4 * (1 + 1e-9)
    assert rp / (1 + np.linalg.norm(lp.b)) <= tol
    assert rd / (1 + np.linalg.norm(lp.c)) <= tol
    assert abs(pobj - dobj) / (1 + abs(pobj) + abs(dobj)) <= tol
    assert np.all(x >= lp.lb - 1e-12) and np.all(x <= lp.ub + 1e-12)
