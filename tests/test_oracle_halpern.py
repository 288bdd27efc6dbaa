"""Pins of the oracle's reflected restarted Halpern PDHG and PID primal weight
(readings H-1..H-4) — `-m "not gpu"`.

Hand-worked values (tests/golden/halpern_2x2.json, exact decimals on the 2x2 LP of
pdhg_2x2.json), the fixed point of the Halpern map at a KKT point, and the optimum
against the closed form / brute-force vertex enumeration / HiGHS.
"""
import math

import numpy as np
import pytest
import scipy.optimize
import scipy.sparse as sp

import lpgen
import oracle
import lp_brute as brute
from test_oracle_restart import lp_from_dense

HALPERN = dict(method=1, reflection=1.0)


@pytest.fixture(scope="module")
def g(golden):
    return golden("halpern_2x2.json")


def _run(g, **kw):
    p2 = golden_2x2()
    olp = oracle.OracleLP(lp_from_dense(p2["A"], p2["b"], p2["c"], [0.0, 0.0], [math.inf, math.inf]))
    prm = oracle.default_params(step_size=0.1, primal_weight=1.0, **{**HALPERN, **kw})
    return olp, oracle.Run(olp, prm, x_init=np.array(g["z0"]["x"]), y_init=np.array(g["z0"]["y"]),
                           mode=kw.pop("mode", oracle.MODE_NONE) if "mode" in kw else oracle.MODE_NONE)


def golden_2x2():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "pdhg_2x2.json")) as f:
        return json.load(f)


def test_halpern_hand_steps(g):
    """Two Halpern steps: z1 = T(z0) (lambda = 1/2 with rho = 1), z2 = 2/3(2T(z1) - z1) + 1/3 z0;
    the returned point is T(z) (in the box); r0 = fixed-point residual at the anchor."""
    olp, r = _run(g, restart=0)
    r.run(1)
    xh, yh = r.get()
    np.testing.assert_allclose(xh, g["step1"]["zh"]["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(yh, g["step1"]["zh"]["y"], rtol=0, atol=1e-15)
    x, y = r.get_z()
    np.testing.assert_allclose(x, g["step1"]["z"]["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(y, g["step1"]["z"]["y"], rtol=0, atol=1e-15)
    assert r.restart_state()["S_r"] == pytest.approx(math.sqrt(g["step1"]["r0_sq"]), rel=1e-14)
    r.run(1)
    xh, yh = r.get()
    np.testing.assert_allclose(xh, g["step2"]["zh"]["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(yh, g["step2"]["zh"]["y"], rtol=0, atol=1e-15)
    x, y = r.get_z()
    np.testing.assert_allclose(x, g["step2"]["z"]["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(y, g["step2"]["z"]["y"], rtol=0, atol=1e-15)
    # r0 stays the anchor's residual; the residual at z1 is the next one
    assert r.restart_state()["S_r"] == pytest.approx(math.sqrt(g["step1"]["r0_sq"]), rel=1e-14)


def test_reflection_zero_is_plain_halpern(g):
    """rho = 0: z1 = 1/2 T(z0) + 1/2 z0 (plain Halpern averaging with the anchor)."""
    olp, r = _run(g, restart=0, reflection=0.0)
    r.run(1)
    x, y = r.get_z()
    z0x, z0y = np.array(g["z0"]["x"]), np.array(g["z0"]["y"])
    np.testing.assert_allclose(x, 0.5 * np.array(g["step1"]["zh"]["x"]) + 0.5 * z0x, rtol=0, atol=1e-15)
    np.testing.assert_allclose(y, 0.5 * np.array(g["step1"]["zh"]["y"]) + 0.5 * z0y, rtol=0, atol=1e-15)


@pytest.mark.parametrize("pid", [0, 1])
def test_halpern_restart_and_weight(g, pid):
    """K = 2: the artificial criterion restarts at k = 2; omega from the anchor movement
    (theta smoothing: sqrt(dy/dx); PID with kp + ki = 1, kd = 0: dy/dx); the iterate and
    the anchor become T(z1); t = 0."""
    c = g["restart_K2"]
    olp, r = _run(g, restart=1, check_every=2, pid=pid)
    r.run(2)
    st = r.restart_state()
    assert st["restarts"] == 1 and st["t"] == 0
    ratio = math.sqrt(c["dy_sq"]) / math.sqrt(c["dx_sq"])
    assert r.omega == pytest.approx(ratio if pid else math.sqrt(ratio), rel=1e-14)
    x, y = r.get_z()
    np.testing.assert_allclose(x, c["z_after"]["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(y, c["z_after"]["y"], rtol=0, atol=1e-15)
    assert oracle.score(olp, *r.get())["score"] == pytest.approx(c["score_zh"], rel=1e-14)


def test_pid_gains():
    """PID update on e = log(dy/dx) - log omega over two restarts (hand arithmetic):
    log w1 = log w0 + kp e1 + ki e1 + kd e1;  log w2 = log w1 + kp e2 + ki (e1 + e2) + kd (e2 - e1)."""
    lp = lpgen.config("c1")
    olp = oracle.OracleLP(lp)
    kp, ki, kd = 0.7, 0.2, 0.05
    prm = oracle.default_params(step_size=0.5 / oracle.power_sigma(olp), primal_weight=1.0, method=1, pid=1,
                                kp=kp, ki=ki, kd=kd, check_every=8, beta_art=0.0)   # restart at every check
    r = oracle.Run(olp, prm, mode=oracle.MODE_NONE)
    anchors = [np.concatenate(r.get_z())]
    w = [1.0]
    for _ in range(2):
        r.run(8)
        anchors.append(np.concatenate(r.get_z()))
        w.append(r.omega)
    n = lp.n
    e = []
    for i in (1, 2):
        dx = np.linalg.norm(anchors[i][:n] - anchors[i - 1][:n])
        dy = np.linalg.norm(anchors[i][n:] - anchors[i - 1][n:])
        e.append(math.log(dy / dx) - math.log(w[i - 1]))
    assert math.log(w[1]) == pytest.approx(math.log(w[0]) + (kp + ki + kd) * e[0], rel=1e-12, abs=1e-14)
    assert math.log(w[2]) == pytest.approx(math.log(w[1]) + kp * e[1] + ki * (e[0] + e[1]) + kd * (e[1] - e[0]),
                                           rel=1e-12, abs=1e-14)


@pytest.mark.parametrize("name", ["c1", "c2-s"])
def test_halpern_certificate_fixed_point(name):
    """A KKT point is a fixed point of T, hence of the reflected Halpern map anchored there."""
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    p = oracle.default_params(step_size=0.5 / oracle.power_sigma(olp), method=1, pid=1)
    r = oracle.Run(olp, p, x_init=lp.x0, y_init=lp.y0, mode=oracle.MODE_NONE)
    r.run(200)
    for x, y in (r.get(), r.get_z()):
        assert np.max(np.abs(x - lp.x0)) < 1e-11 * (1 + np.abs(lp.x0).max())
        assert np.max(np.abs(y - lp.y0)) < 1e-11 * (1 + np.abs(lp.y0).max())


def test_halpern_2x2_optimum(golden):
    g2 = golden("pdhg_2x2.json")
    lp = lp_from_dense(g2["A"], g2["b"], g2["c"], [0.0, 0.0], [math.inf, math.inf])
    x, y, res = oracle.solve(oracle.OracleLP(lp), oracle.default_params(eps_rel=1e-10, max_iters=200000, **HALPERN))
    assert res["status"] == 0
    np.testing.assert_allclose(x, g2["optimum"]["x"], atol=1e-8)
    np.testing.assert_allclose(y, g2["optimum"]["y"], atol=1e-8)


@pytest.mark.parametrize("pid", [0, 1])
@pytest.mark.parametrize("seed", [1, 2])
def test_halpern_micro_lp_vs_enumeration(seed, pid):
    lp = lpgen.gen_dense(m=5, n=11, n_support=3, n_face=7, seed=seed)
    best, _, _ = brute.optimum(lp.dense_A(), lp.b, lp.c, lp.lb, lp.ub)
    x, y, res = oracle.solve(oracle.OracleLP(lp), oracle.default_params(eps_rel=1e-8, max_iters=400000, pid=pid,
                                                                         **HALPERN))
    assert res["status"] == 0
    assert abs(res["pobj"] - best) <= 1e-6 * (1 + abs(best))
    assert np.all(x >= lp.lb) and np.all(x <= lp.ub)   # the returned T(z) is in the box


@pytest.mark.parametrize("name", ["c3-s", "c4-s"])
def test_halpern_vs_highs(name):
    lp = lpgen.config(name)
    p, j, v = lp.csr_A()
    A = sp.csr_matrix((v, j, p), shape=(lp.m, lp.n))
    hr = scipy.optimize.linprog(lp.c, A_eq=A, b_eq=lp.b, bounds=(0, None), method="highs")
    x, y, res = oracle.solve(oracle.OracleLP(lp), oracle.default_params(eps_rel=1e-8, max_iters=400000, pid=1,
                                                                         **HALPERN))
    assert res["status"] == 0
    assert abs(res["pobj"] - hr.fun) <= 1e-6 * (1 + abs(hr.fun))


@pytest.mark.parametrize("name", ["c1", "c2-s", "c4-s"])
def test_halpern_termination_claim(name):
    """CONVERGED => the returned T(z) satisfies P:124-126 (dense numpy recomputation)."""
    lp = lpgen.config(name)
    x, y, res = oracle.solve(oracle.OracleLP(lp), oracle.default_params(pid=1, **HALPERN))
    assert res["status"] == 0
    A = lp.dense_A()
    z = lp.c - A.T @ y
    fin_u = np.isfinite(lp.ub)
    rd = np.where(fin_u, 0.0, np.minimum(z, 0.0))
    dobj = lp.b @ y - np.sum(np.where(fin_u, np.where(fin_u, lp.ub, 0) * np.maximum(-z, 0), 0))
    pobj = lp.c @ x
    assert np.linalg.norm(lp.b - A @ x) <= 1e-4 * (1 + np.linalg.norm(lp.b)) * (1 + 1e-12)
    assert np.linalg.norm(rd) <= 1e-4 * (1 + np.linalg.norm(lp.c)) * (1 + 1e-12)
    assert abs(pobj - dobj) <= 1e-4 * (1 + abs(pobj) + abs(dobj)) * (1 + 1e-12)


def test_halpern_corner_push_properties():
    """Algorithm 1 with Halpern steering iterations: bound-map soundness, >= 100 iterations,
    residual target met by the returned T(z)."""
    lp = lpgen.config("c2-s")
    olp = oracle.OracleLP(lp)
    prm = oracle.default_params(pid=1, **HALPERN)
    x, y, _ = oracle.solve(olp, prm)
    xh, _, z, rc, before, after, _ = oracle.corner_push(olp, x, y, params=prm, floor=100)
    assert rc["status"] == 0 and rc["iterations"] >= 100
    assert np.all(xh[z > 1e-6] <= x[z > 1e-6]) and np.all(xh[z < -1e-6] >= x[z < -1e-6])
    assert np.linalg.norm(lp.b - olp.A_times(xh)) <= 1e-4 * (1 + np.linalg.norm(lp.b)) * (1 + 1e-12)
