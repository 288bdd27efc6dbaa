"""Parity of the GPU reflected restarted Halpern PDHG + PID primal weight (NEXT-1)
with the oracle (`-m gpu`), through the C-ABI.

Contract as for R-PDHG (BASELINE.json north_star): the iterate (the Halpern sequence z)
within 1e-9 over 1000 lockstep iterations with restarts, element-wise and in norm;
termination status equal, iteration count within +-1%, objective to 1e-6; Algorithm 1
steering iterations likewise; the returned point is T(z) (in the box).
"""
import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_13894_b200 as cpd  # noqa: E402
from parity_util import close, worst  # noqa: E402

CONFIGS = ["c1", "c2-s", "c3-s", "c4-s", "c5-s"]


@pytest.fixture(scope="module")
def problems():
    cache = {}

    def get(name):
        if name not in cache:
            lp = lpgen.config(name)
            cache[name] = (lp, oracle.OracleLP(lp), cpd.Problem.from_lp(lp))
        return cache[name]
    return get


@pytest.mark.parametrize("pid", [0, 1])
@pytest.mark.parametrize("name", CONFIGS)
def test_halpern_lockstep(problems, name, pid):
    lp, olp, P = problems(name)
    eta = 0.9 / oracle.power_sigma(olp)
    kw = dict(step_size=eta, restart=1, method=1, pid=pid)
    S = cpd.Solver(P, **kw)
    R = oracle.Run(olp, oracle.default_params(**kw), mode=oracle.MODE_NONE)
    k = 0
    for target in (1, 2, 63, 64, 65, 128, 300, 1000):
        S.step(target - k)
        R.run(target - k)
        k = target
        xg, yg = S.get_iterate()
        xo, yo = R.get_z()
        assert close(xg, xo), (name, k, worst(xg, xo))
        assert close(yg, yo), (name, k, worst(yg, yo))
    assert R.restart_state()["restarts"] >= 1


@pytest.mark.parametrize("pid", [0, 1])
@pytest.mark.parametrize("name", ["c1", "c2-s", "c3-s", "c4-s"])
def test_halpern_termination(problems, name, pid):
    lp, olp, P = problems(name)
    S = cpd.Solver(P, method=1, pid=pid)
    r = S.solve()
    xo, yo, ro = oracle.solve(olp, oracle.default_params(method=1, pid=pid))
    assert r["status"] == ro["status"] == 0
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"]), (r, ro)
    assert r["restarts"] == ro["restarts"]
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
    xg, yg = S.get_iterate()
    assert np.all(xg >= lp.lb) and np.all(xg <= lp.ub)   # T(z) is returned
    if r["iterations"] == ro["iterations"]:
        assert close(xg, xo, 1e-8) and close(yg, yo, 1e-8)
    assert oracle.score(olp, xg, yg)["score"] <= 1e-4 * (1 + 1e-9)


@pytest.mark.parametrize("name", ["c1", "c2-s"])
def test_halpern_corner_push(problems, name):
    lp, olp, P = problems(name)
    prm = oracle.default_params(method=1, pid=1)
    xo, yo, _ = oracle.solve(olp, prm)
    S = cpd.Solver(P, method=1, pid=1)
    S.set_iterate(xo, yo)
    r, before, after = S.corner_push(seed=1001, candidate_floor=100)
    xh, _, z, ro, bo, ao, model = oracle.corner_push(olp, xo, yo, params=prm, seed=1001, floor=100)
    assert r["status"] == ro["status"] == 0
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"]), (r, ro)
    xg, _, zg = S.get_iterate(z=True)
    if r["iterations"] == ro["iterations"]:
        assert close(xg, xh, 1e-8)
    ref = oracle.stats(lp.m, xg, zg, lp.lb, lp.ub, model["lhat"], model["uhat"], 1e-6, 100)
    for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc", "candidates"):
        assert after[k] == ref[k], k


def test_halpern_corner_lockstep(problems):
    lp, olp, P = problems("c5-s")
    prm = oracle.default_params(method=1, pid=1)
    xo, yo, _ = oracle.solve(olp, oracle.default_params(max_iters=300, method=1, pid=1))
    S = cpd.Solver(P, method=1, pid=1)
    S.set_iterate(xo, yo)
    r, _, _ = S.corner_push(seed=5, max_iters=1000, min_iters=10 ** 9)
    xh, _, _, ro, _, _, _ = oracle.corner_push(olp, xo, yo, params=prm, seed=5, max_iters=1000, min_iters=10 ** 9)
    assert r["status"] == ro["status"] == 1 and r["iterations"] == 1000
    xg, _ = S.get_iterate()
    assert close(xg, xh), worst(xg, xh)


def test_halpern_scaled_zipf_termination():
    """Halpern + PID + diagonal scaling on a Zipf(1.2) LP (C5's recipe, 3,000 x 18,000)."""
    lp = lpgen.gen_sparse(m=3000, n=18000, per_col=12, seed=26, ub=100.0, zipf=1.2, name="c5-xs")
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    P.scale(10, 1)
    S = cpd.Solver(P, method=1, pid=1, max_iters=100000)
    r = S.solve()
    xo, yo, ro, sl = oracle.solve_scaled(olp, oracle.default_params(method=1, pid=1, max_iters=100000))
    assert r["status"] == ro["status"] == 0, (r, ro)
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"]), (r, ro)
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)


def test_halpern_graph_eager_identical(problems):
    lp, olp, P = problems("c4-s")
    a = cpd.Solver(P, use_graph=1, method=1, pid=1)
    b = cpd.Solver(P, use_graph=0, method=1, pid=1)
    ra, rb = a.solve(), b.solve()
    assert ra["iterations"] == rb["iterations"]
    xa, ya = a.get_iterate()
    xb, yb = b.get_iterate()
    assert np.array_equal(xa, xb) and np.array_equal(ya, yb)


def test_halpern_numerical_failure():
    lp = lpgen.config("c1")
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P, step_size=1e150, primal_weight=1.0, method=1)
    r = S.solve()
    _, _, ro = oracle.solve(olp, oracle.default_params(step_size=1e150, primal_weight=1.0, method=1))
    assert r["status"] == ro["status"] == 3 and r["iterations"] == ro["iterations"]


@pytest.mark.parametrize("fmt", [("0", "0"), ("1", "1")])
def test_halpern_every_engine(fmt, monkeypatch):
    """The Halpern epilogues on the TMA plan (k_spmv) and the warp plan + SELL (k_csrw,
    k_dense, short-row SELL passes) of c5-s with forced heavy rows / slabs."""
    warp, sell = fmt
    monkeypatch.setenv("CPD_WARP", warp)
    monkeypatch.setenv("CPD_SELL", sell)
    if warp == "1":
        monkeypatch.setenv("CPD_HEAVY_MIN", "4096")
        monkeypatch.setenv("CPD_SLAB_COLS", "8192")
        monkeypatch.setenv("CPD_SSELL", "2")
    lp = lpgen.config("c5-s")
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    eta = 0.9 / oracle.power_sigma(olp)
    kw = dict(step_size=eta, restart=1, method=1, pid=1)
    S = cpd.Solver(P, **kw)
    R = oracle.Run(olp, oracle.default_params(**kw), mode=oracle.MODE_NONE)
    S.step(300)
    R.run(300)
    xg, yg = S.get_iterate()
    xo, yo = R.get_z()
    assert close(xg, xo) and close(yg, yo), (fmt, worst(xg, xo), worst(yg, yo))
