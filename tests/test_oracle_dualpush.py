"""Pins of the oracle's dual corner push and push-phase decision (
DESIGN.md readings D-1..D-4) — `-m "not gpu"`."""
import math

import numpy as np
import pytest

import lpgen
import oracle
import lp_brute as brute


def _inf(v):
    return np.array([(-math.inf if x == "-inf" else math.inf if x == "inf" else x) for x in v], float)


def test_dual_bound_map_example(golden):
    """Classification of every column kind (hand example, golden corner_examples.json)."""
    e = golden("corner_examples.json")["dual_bound_map"]
    n = len(e["x"])
    lp = lpgen.LP(m=1, n=n, ATp=np.arange(n + 1, dtype=np.int32), ATj=np.zeros(n, np.int32),
                  ATx=np.ones(n), b=np.array([1.0]), c=np.ones(n), lb=_inf(e["lb"]), ub=_inf(e["ub"]))
    lh, uh, cnt = oracle.dual_corner_model(oracle.OracleLP(lp), e["x"], e["eps_abs"])
    assert lh.tolist() == _inf(e["lhat"]).tolist() and uh.tolist() == _inf(e["uhat"]).tolist()
    assert cnt == e["counts"]


def test_decide_examples(golden):
    for c in golden("corner_examples.json")["decide"]["cases"]:
        assert oracle.corner_decide(c, c["m"]) == (c["primal"], c["dual"]), c


def _dual_vertices(A, c, lb, ub, xs, eps):
    """Brute force: every basic dual solution y = A_B^-T c_B that is feasible for the dual
    corner model of xs (z_j = 0 off, z_j >= 0 at lower, <= 0 at upper)."""
    import itertools
    m, n = A.shape
    out = []
    for B in itertools.combinations(range(n), m):
        AB = A[:, B]
        if abs(np.linalg.det(AB)) < 1e-9:
            continue
        y = np.linalg.solve(AB.T, c[list(B)])
        z = c - A.T @ y
        ok = True
        for j in range(n):
            off = xs[j] - lb[j] > eps and ub[j] - xs[j] > eps
            low = not off and xs[j] - lb[j] <= eps
            if off and abs(z[j]) > 1e-9 or low and z[j] < -1e-9 or (not off and not low) and z[j] > 1e-9:
                ok = False
                break
        if ok:
            out.append(y)
    return out


@pytest.mark.parametrize("seed", [1, 3])
def test_dual_model_face_is_dual_optimal(seed):
    """D-1: every dual vertex feasible for the dual corner model of the planted optimum x0
    is dual OPTIMAL for M (b^T y = opt, by enumeration), and the dual push from the
    phase-1 point ends with every off column's reduced cost at 0 (|z| <= eps_abs,
    recomputed densely) and b^T yhat within tolerance of opt."""
    lp = lpgen.gen_dense(m=4, n=9, n_support=2, n_face=5, seed=seed)   # degenerate: many dual optima
    A = lp.dense_A()
    V = _dual_vertices(A, lp.c, lp.lb, lp.ub, lp.x0, 1e-6)
    assert len(V) >= 1
    for y in V:
        assert lp.b @ y == pytest.approx(lp.opt, rel=1e-9, abs=1e-9)
    olp = oracle.OracleLP(lp)
    x, y, _ = oracle.solve(olp, oracle.default_params(eps_rel=1e-8, max_iters=400000))
    xx, yh, zh, rc, b, a, model = oracle.dual_corner_push(olp, x, y, floor=1, max_iters=400000)
    assert rc["status"] == 0 and rc["iterations"] >= 100
    z = lp.c - A.T @ yh
    off = (x - lp.lb > 1e-6) & (lp.ub - x > 1e-6)
    assert np.all(np.abs(z[off]) <= 1e-6 * (1 + 1e-9))
    assert np.all(z[~off] >= -1e-6)   # l = 0, u = inf: at-lower columns keep z >= 0
    assert a["zero_rc"] >= off.sum()
    assert lp.b @ yh == pytest.approx(lp.opt, rel=1e-5)
    np.testing.assert_array_equal(xx, x)   # the primal point is phase 1's


@pytest.mark.parametrize("name", ["c1", "c3-s"])
def test_dual_push_reduces_estimate(name):
    """On LPs with p >= m off-bound columns the dual push drives the dual-push estimate
    m - d to 0; the objective gap stays at the phase-1 tolerance."""
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    x, y, _ = oracle.solve(olp)
    xx, yh, zh, rc, b, a, model = oracle.dual_corner_push(olp, x, y, floor=10, max_iters=100000)
    assert rc["status"] == 0
    assert model["off"] >= lp.m and b["est_dual_pushes"] > 0 and a["est_dual_pushes"] == 0
    assert oracle.score(olp, x, yh)["score"] <= 1e-4


def test_dual_push_halpern():
    lp = lpgen.config("c1")
    olp = oracle.OracleLP(lp)
    prm = oracle.default_params(method=1, pid=1)
    x, y, _ = oracle.solve(olp, prm)
    _, yh, zh, rc, b, a, _ = oracle.dual_corner_push(olp, x, y, params=prm, floor=10)
    assert rc["status"] == 0 and a["est_dual_pushes"] == 0
