"""Pins of the oracle's implicit inequality rows (P:89-92,
P:301-306): dual sign projection, violation-only primal residual, the corner
model's row-sense rule.  `-m "not gpu"`.  Independent references: closed-form
one/two-variable LPs, HiGHS (scipy) optima, and the explicit-slack form of the
same LP (lpgen c4-s) having the same optimum.
"""
import types

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.optimize import linprog

import lpgen
import oracle


def _lp(A, b, c, sense, lb=None, ub=None):
    A = np.asarray(A, float)
    m, n = A.shape
    AT = sp.csr_matrix(A.T)
    return types.SimpleNamespace(m=m, n=n, ATp=AT.indptr.astype(np.int32), ATj=AT.indices.astype(np.int32),
                                 ATx=AT.data.astype(float), b=np.asarray(b, float), c=np.asarray(c, float),
                                 lb=np.zeros(n) if lb is None else np.asarray(lb, float),
                                 ub=np.full(n, np.inf) if ub is None else np.asarray(ub, float),
                                 sense=np.asarray(sense, np.int8))


def _tight(**kw):
    return oracle.default_params(eps_rel=1e-9, max_iters=200000, **kw)


def test_geq_row_closed_form():
    # min x1 + 2 x2  s.t.  x1 + x2 >= 1, x >= 0   ->  x = (1, 0), y = 1 (>= 0)
    olp = oracle.OracleLP(_lp([[1.0, 1.0]], [1.0], [1.0, 2.0], [2]))
    x, y, r = oracle.solve(olp, _tight())
    assert r["status"] == 0
    np.testing.assert_allclose(x, [1.0, 0.0], atol=1e-7)
    np.testing.assert_allclose(y, [1.0], atol=1e-7)


def test_leq_row_closed_form():
    # min -x1 - x2  s.t.  x1 + 2 x2 <= 4, x1 <= 3 (bound), x >= 0 -> x = (3, 0.5), y = -0.5 (<= 0)
    olp = oracle.OracleLP(_lp([[1.0, 2.0]], [4.0], [-1.0, -1.0], [1], ub=[3.0, np.inf]))
    x, y, r = oracle.solve(olp, _tight())
    assert r["status"] == 0
    np.testing.assert_allclose(x, [3.0, 0.5], atol=1e-7)
    np.testing.assert_allclose(y, [-0.5], atol=1e-7)


def test_slack_row_has_zero_residual_and_dual():
    # x1 + x2 <= 10 is slack at the optimum of min x1 s.t. x1 - x2 = 0, x1 + x2 <= 10 -> x = 0
    olp = oracle.OracleLP(_lp([[1.0, -1.0], [1.0, 1.0]], [0.0, 10.0], [1.0, 0.0], [0, 1]))
    x, y, r = oracle.solve(olp, _tight())
    sc = oracle.score(olp, np.zeros(2), np.zeros(2))
    assert sc["rp"] == 0.0                       # zero iterate violates no row (b = (0, 10))
    assert r["status"] == 0 and abs(y[1]) < 1e-7


def test_dual_sign_invariant_along_the_run():
    lp = lpgen.config("c4-s-ineq")
    olp = oracle.OracleLP(lp)
    R = oracle.Run(olp, oracle.default_params(step_size=0.9 / oracle.power_sigma(olp)), mode=oracle.MODE_NONE)
    for _ in range(5):
        R.run(57)
        _, y = R.get()
        assert np.all(y[lp.sense == 1] <= 0.0) and np.all(y[lp.sense == 2] >= 0.0)


def test_implicit_rows_match_highs_and_explicit_slacks():
    lp = lpgen.config("c4-s-ineq")
    A = sp.csr_matrix((lp.ATx, lp.ATj, lp.ATp), shape=(lp.n, lp.m)).T.tocsr()
    eq = lp.sense == 0
    ref = linprog(lp.c, A_ub=A[~eq], b_ub=lp.b[~eq], A_eq=A[eq], b_eq=lp.b[eq], bounds=(0, None),
                  method="highs").fun
    lpe = lpgen.config("c4-s")
    Ae = sp.csr_matrix((lpe.ATx, lpe.ATj, lpe.ATp), shape=(lpe.n, lpe.m)).T.tocsr()
    ref_e = linprog(lpe.c, A_eq=Ae, b_eq=lpe.b, bounds=(0, None), method="highs").fun
    assert ref == pytest.approx(ref_e, rel=1e-9)
    x, y, r = oracle.solve(oracle.OracleLP(lp), oracle.default_params(eps_rel=1e-7, max_iters=200000))
    assert r["status"] == 0 and r["pobj"] == pytest.approx(ref, rel=1e-5)


def test_corner_sense_rule():
    # an inequality row with |y_i| > eps_abs becomes '='; others keep their sense
    olp = oracle.OracleLP(_lp([[1.0, 1.0], [1.0, 0.0], [0.0, 1.0]], [1.0, 5.0, 5.0], [1.0, 1.0], [2, 1, 1]))
    shat, k = oracle.corner_senses(olp, np.array([0.7, -1e-9, -0.2]), 1e-6)
    assert shat.tolist() == [0, 1, 0] and k == 2


def test_corner_push_with_implicit_rows():
    lp = lpgen.config("c4-s-ineq")
    olp = oracle.OracleLP(lp)
    x, y, r = oracle.solve(olp)
    xh, _, z, rc, before, after, model = oracle.corner_push(olp, x, y, floor=100)
    assert rc["status"] == 0 and rc["iterations"] >= 100
    assert model["rows_eq"] == int(np.sum((lp.sense != 0) & (np.abs(y) > 1e-6)))
    # the steering residual is the corner model's (rows made '=' count fully)
    assert rc["rp_norm"] <= model["target"] * (1 + 1e-12)
