"""NEXT-4 dual corner push and push-phase decision on the GPU vs the oracle (`-m gpu`)."""
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

KEYS = ("off_bound", "zero_rc", "candidates", "est_primal_pushes", "est_dual_pushes", "is_candidate")


@pytest.mark.parametrize("method", [0, 1])
@pytest.mark.parametrize("name", ["c1", "c2-s", "c3-s", "c4-s"])
def test_dual_push_parity(name, method):
    """Same phase-1 point on both sides: status, iterations +-1%, yhat, the counts d and
    m - d recounted by the oracle from the GPU's (x, zhat) bit-exactly, x unchanged."""
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    prm = oracle.default_params(method=method, pid=method)
    xo, yo, _ = oracle.solve(olp, prm)
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P, method=method, pid=method)
    S.set_iterate(xo, yo)
    r, b, a = S.dual_corner_push(candidate_floor=10, max_iters=20000)
    _, yh, zh, ro, bo, ao, model = oracle.dual_corner_push(olp, xo, yo, params=prm, floor=10, max_iters=20000)
    assert r["status"] == ro["status"], (r, ro)
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"]), (r, ro)
    xg, yg, zg = S.get_iterate(z=True)
    np.testing.assert_array_equal(xg, xo)
    if r["iterations"] == ro["iterations"]:
        assert close(yg, yh, 1e-8), worst(yg, yh)
    for k in KEYS:
        assert b[k] == bo[k], k
    ref = oracle.stats(lp.m, xg, zg, lp.lb, lp.ub, None, None, 1e-6, 10)
    for k in KEYS:
        assert a[k] == ref[k], k


def test_dual_push_lockstep():
    """The dual-model iterations themselves: 1000 iterations (stop disabled) to 1e-9."""
    lp = lpgen.config("c5-s")
    olp = oracle.OracleLP(lp)
    xo, yo, _ = oracle.solve(olp, oracle.default_params(max_iters=400))
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P)
    S.set_iterate(xo, yo)
    r, _, _ = S.dual_corner_push(max_iters=1000, min_iters=10 ** 9)
    _, yh, _, ro, _, _, _ = oracle.dual_corner_push(olp, xo, yo, max_iters=1000, min_iters=10 ** 9)
    assert r["status"] == ro["status"] == 1 and r["iterations"] == 1000
    _, yg = S.get_iterate()
    assert close(yg, yh), worst(yg, yh)


def test_dual_push_lowers_estimate():
    """C1: p = 30 off-bound columns >= m = 20, so the push drives m - d from 20 to 0."""
    lp = lpgen.config("c1")
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P)
    S.solve()
    r, b, a = S.dual_corner_push(candidate_floor=10)
    assert r["status"] == 0 and b["est_dual_pushes"] > 0 and a["est_dual_pushes"] == 0


def test_decide_matches_oracle(golden):
    for c in golden("corner_examples.json")["decide"]["cases"]:
        assert cpd.corner_decide(c, c["m"]) == oracle.corner_decide(c, c["m"]) == (c["primal"], c["dual"])
    rng = np.random.default_rng(5)
    for _ in range(200):
        m = int(rng.integers(1, 50))
        st = dict(off_bound=int(rng.integers(0, 100)), zero_rc=int(rng.integers(0, 100)),
                  is_candidate=int(rng.integers(0, 2)))
        st["est_dual_pushes"] = max(m - st["zero_rc"], 0)
        assert cpd.corner_decide(st, m) == oracle.corner_decide(st, m)


def test_dual_push_refused_on_scaled():
    lp = lpgen.config("c2-s")
    P = cpd.Problem.from_lp(lp)
    P.scale()
    S = cpd.Solver(P)
    with pytest.raises(cpd.CpdError) as ei:
        S.dual_corner_push()
    assert ei.value.code == -8
