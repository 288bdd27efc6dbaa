"""Implicit inequality rows on the GPU (cpd_problem_set_senses; SURVEY NEXT-2,
P:89-92) against the oracle — `-m gpu`: lockstep iterates (1e-9),
termination (+-1%, objective 1e-6), the corner model's row-sense rule and counts,
alone, with diagonal scaling, and on the split (multi-GPU) path with one rank.
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


from parity_util import close, worst  # noqa: E402  (norm AND entry-wise bound)


@pytest.fixture(scope="module")
def ineq():
    """c4-s-ineq with every capacity cut to the planted routing's load + 0.5, so many
    capacity rows bind (non-zero duals: the P:301-306 rule has rows to change)."""
    lp = lpgen.config("c4-s-ineq")
    K, NA = lp.meta["K"], lp.meta["NA"]
    load = lp.x0.reshape(K, NA).sum(0)
    lp.b = lp.b.copy()
    lp.b[lp.m - NA:] = load + 0.5
    return lp, oracle.OracleLP(lp)


def _problem(lp, kind):
    if kind == "plain":
        return cpd.Problem.from_lp(lp)
    if kind == "scaled":
        return cpd.Problem.from_lp(lp).scale(10, 1)
    return cpd.Problem.create_dist(lp, 0, 1, cpd.nccl_unique_id(), partition=int(kind[-1]), device=0)


@pytest.mark.parametrize("kind", ["plain", "scaled", "dist0", "dist1"])
def test_ineq_lockstep(ineq, kind):
    lp, olp = ineq
    P = _problem(lp, kind)
    if kind == "scaled":
        sl = oracle.ScaledLP(olp, 10, 1)
        eta = 0.9 / oracle.power_sigma(sl.olp)
        R = oracle.Run(sl.olp, oracle.default_params(step_size=eta), mode=oracle.MODE_NONE)
        R.set_original(olp, olp.c, olp.lb, olp.ub, sl.r, sl.s)
        xs, ys = sl.s, sl.r
    else:
        eta = 0.9 / oracle.power_sigma(olp)
        R = oracle.Run(olp, oracle.default_params(step_size=eta), mode=oracle.MODE_NONE)
        xs, ys = 1.0, 1.0
    S = cpd.Solver(P, step_size=eta)
    k = 0
    for target in (1, 64, 65, 500, 1000):
        S.step(target - k)
        R.run(target - k)
        k = target
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xs * xo) and close(yg, ys * yo), (kind, k)
        assert np.all(yg[lp.sense == 1] <= 0.0) and np.all(yg[lp.sense == 2] >= 0.0)


@pytest.mark.parametrize("kind", ["plain", "scaled", "dist1"])
def test_ineq_solve_and_corner(ineq, kind):
    lp, olp = ineq
    P = _problem(lp, kind)
    S = cpd.Solver(P)
    r = S.solve()
    if kind == "scaled":
        xo, yo, ro, sl = oracle.solve_scaled(olp)
    else:
        xo, yo, ro = oracle.solve(olp)
    assert r["status"] == ro["status"] == 0
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"])
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
    S.set_iterate(xo, yo)
    rc, before, after = S.corner_push(seed=1001, candidate_floor=100)
    if kind == "scaled":
        xh, _, z_o, rco, b_o, a_o, model = oracle.corner_push_scaled(olp, sl, xo, yo, seed=1001, floor=100)
    else:
        xh, _, z_o, rco, b_o, a_o, model = oracle.corner_push(olp, xo, yo, seed=1001, floor=100)
    assert rc["status"] == rco["status"] == 0
    assert abs(rc["iterations"] - rco["iterations"]) <= max(1, 0.01 * rco["iterations"])
    assert before["rows_eq"] == after["rows_eq"] == model["rows_eq"]
    assert model["rows_eq"] == int(np.sum((lp.sense != 0) & (np.abs(yo) > 1e-6))) > 0
    xg, yg, zg = S.get_iterate(z=True)
    ref = oracle.stats(lp.m, xg, zg, lp.lb, lp.ub, model["lhat"], model["uhat"], 1e-6, 100)
    for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc", "candidates"):
        assert after[k] == ref[k], k


def test_bad_sense_is_an_error():
    lp = lpgen.config("c4-s-ineq")
    P = cpd.Problem.from_lp(lpgen.config("c4-s"))
    bad = np.zeros(P.m, np.int8)
    bad[3] = 7
    with pytest.raises(cpd.CpdError):
        P.set_senses(bad)
    del lp
