"""Diagonal preconditioning on the GPU (cpd_problem_scale) against the oracle's
(oracle.ScaledLP / solve_scaled / corner_push_scaled) — `-m gpu`.

Same contract as the unscaled path (BASELINE.json north_star): scale vectors to
rounding, iterates to 1e-9 over 1000 lockstep iterations, termination +-1% with
the objective to 1e-6, corner counts bit-exact on identical (x, z).
"""
import math

import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_13894_b200 as cpd  # noqa: E402

NAMES = ["c1", "c2-s", "c4-s", "c5-s"]


from parity_util import close, worst  # noqa: E402  (norm AND entry-wise bound)


@pytest.fixture(scope="module")
def scaled():
    cache = {}

    def get(name):
        if name not in cache:
            lp = lpgen.config(name)
            olp = oracle.OracleLP(lp)
            sl = oracle.ScaledLP(olp, 10, 1)
            P = cpd.Problem.from_lp(lp).scale(10, 1)
            cache[name] = (lp, olp, sl, P)
        return cache[name]
    return get


@pytest.mark.parametrize("name", NAMES)
def test_scale_vectors(scaled, name):
    lp, olp, sl, P = scaled(name)
    r, s = P.scaling()
    np.testing.assert_allclose(r, sl.r, rtol=1e-13)
    np.testing.assert_allclose(s, sl.s, rtol=1e-13)
    # power iteration on the scaled operator; the score ABI speaks the original space
    assert P.power_sigma(64, 7) == pytest.approx(oracle.power_sigma(sl.olp, 64, 7), rel=1e-11)
    rng = np.random.default_rng(0)
    x = np.minimum(np.maximum(rng.uniform(-1, 3, lp.n), lp.lb), lp.ub)
    y = rng.standard_normal(lp.m)
    g, o = P.score(x, y), oracle.score(olp, x, y)
    for k in ("rp", "rd", "pobj", "dobj", "score"):
        assert g[k] == pytest.approx(o[k], rel=1e-11), k


@pytest.mark.parametrize("name", NAMES)
def test_scaled_lockstep(scaled, name):
    lp, olp, sl, P = scaled(name)
    eta = 0.9 / oracle.power_sigma(sl.olp)
    S = cpd.Solver(P, step_size=eta, restart=1)
    R = oracle.Run(sl.olp, oracle.default_params(step_size=eta, restart=1), mode=oracle.MODE_NONE)
    R.set_original(olp, olp.c, olp.lb, olp.ub, sl.r, sl.s)
    k = 0
    for target in (1, 64, 65, 300, 1000):
        S.step(target - k)
        R.run(target - k)
        k = target
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, sl.s * xo), (name, k)
        assert close(yg, sl.r * yo), (name, k)


@pytest.mark.parametrize("name", ["c1", "c2-s", "c4-s"])
def test_scaled_solve_and_corner(scaled, name):
    lp, olp, sl, P = scaled(name)
    S = cpd.Solver(P)
    r = S.solve()
    xo, yo, ro, _ = oracle.solve_scaled(olp)
    assert r["status"] == ro["status"] == 0
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"])
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
    xg, yg = S.get_iterate()
    assert oracle.score(olp, xg, yg)["score"] <= 1e-4 * (1 + 1e-9)
    # Algorithm 1 from the oracle's phase-1 point on both sides
    S.set_iterate(xo, yo)
    rc, before, after = S.corner_push(seed=1001, candidate_floor=100)
    xh, _, z_o, rco, b_o, _, model = oracle.corner_push_scaled(olp, sl, xo, yo, seed=1001, floor=100)
    assert rc["status"] == rco["status"] == 0
    assert abs(rc["iterations"] - rco["iterations"]) <= max(1, 0.01 * rco["iterations"])
    xg, yg, zg = S.get_iterate(z=True)
    assert close(zg, z_o, 1e-11)
    for k in ("fix_lb", "fix_ub"):
        assert before[k] == b_o[k], k
    ref = oracle.stats(lp.m, xg, zg, lp.lb, lp.ub, model["lhat"], model["uhat"], 1e-6, 100)
    for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc", "candidates"):
        assert after[k] == ref[k], k
