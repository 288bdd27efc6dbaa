"""Pins of the oracle's adaptive-restart branch, its bound-dependent dual residual and
the count boundaries (`-m "not gpu"`).

Every expected value is hand-worked (exact rationals, one square root per score) and
stored with its derivation in tests/golden/{restart_2x2,score_bounds,corner_examples}.json;
DESIGN.md §3 "Restart pins" restates the derivations.  Each test is chosen so a
plausible slip in the oracle (never restarting to the average, a flipped necessary
criterion, S_r taken from the wrong candidate, the average-return branch missing,
free columns treated as lower-bounded, the model count taken against the original
bounds, a strict/non-strict comparison swapped) changes a checked value.
"""
import math

import numpy as np
import pytest

import lpgen
import oracle


def _inf(v):
    return [(-math.inf if x == "-inf" else math.inf if x == "inf" else x) for x in v]


def lp_from_dense(A, b, c, l, u):
    A = np.asarray(A, float)
    m, n = A.shape
    AT = np.ascontiguousarray(A.T)
    keep = AT != 0.0
    ATp = np.concatenate([[0], np.cumsum(keep.sum(1))]).astype(np.int32)
    ATj = np.tile(np.arange(m, dtype=np.int32), n).reshape(n, m)[keep]
    return lpgen.LP(m=m, n=n, ATp=ATp, ATj=ATj, ATx=AT[keep], b=np.asarray(b, float),
                    c=np.asarray(c, float), lb=np.asarray(l, float), ub=np.asarray(u, float),
                    name="hand")


@pytest.fixture(scope="module")
def g(golden):
    return golden("restart_2x2.json")


def _olp(g):
    return oracle.OracleLP(lp_from_dense(g["A"], g["b"], g["c"], [0.0, 0.0], [math.inf, math.inf]))


def test_restart_to_average(g):
    """Average wins the check at k = K = 2 and the artificial criterion restarts to it:
    (x, y) <- average, S_r <- S_a, t <- 0, omega <- sqrt(omega dy/dx); the next step
    uses the new tau, sigma from the average (hand values, golden case_avg_restart)."""
    c = g["case_avg_restart"]
    olp = _olp(g)
    p = oracle.default_params(step_size=g["eta"], primal_weight=g["omega0"], check_every=g["K"],
                              restart=1)
    r = oracle.Run(olp, p, x_init=np.array(c["x0"]), y_init=np.array(c["y0"]), mode=oracle.MODE_NONE)
    st = r.restart_state()
    assert st["S_r"] == pytest.approx(c["S_r0"], rel=1e-15)
    # the two candidate scores, recomputed from the hand iterates
    sc = oracle.score(olp, [0.0, 76 / 125], [1517 / 5000, 533 / 5000])["score"]
    sa = oracle.score(olp, c["after_restart"]["x"], c["after_restart"]["y"])["score"]
    assert sc == pytest.approx(c["S_c"], rel=1e-14) and sa == pytest.approx(c["S_a"], rel=1e-14)
    r.run(2)
    x, y = r.get()
    np.testing.assert_allclose(x, c["after_restart"]["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(y, c["after_restart"]["y"], rtol=0, atol=1e-15)
    st = r.restart_state()
    assert st["restarts"] == c["after_restart"]["restarts"] and st["t"] == c["after_restart"]["t"]
    assert st["S_r"] == pytest.approx(c["after_restart"]["S_r"], rel=1e-14)
    assert st["S_prev"] == math.inf
    assert r.omega == pytest.approx(c["omega"], rel=1e-14)
    assert r.result()["returned_average"] == c["returned_average"]
    r.run(1)
    x, y = r.get()
    np.testing.assert_allclose(x, c["k3"]["x"], rtol=0, atol=2e-15)
    np.testing.assert_allclose(y, c["k3"]["y"], rtol=0, atol=2e-15)


def test_necessary_criterion_needs_a_rising_score(g):
    """Artificial criterion off (beta_art = 10): the first check cannot restart on the
    necessary criterion (S_prev = inf) and records S_prev; the second check's candidate
    is <= 0.8 S_r AND above S_prev, so it restarts (golden case_necessary)."""
    c = g["case_necessary"]
    a = g["case_avg_restart"]
    olp = _olp(g)
    p = oracle.default_params(step_size=g["eta"], primal_weight=g["omega0"], check_every=g["K"],
                              restart=1, beta_art=c["beta_art"])
    r = oracle.Run(olp, p, x_init=np.array(a["x0"]), y_init=np.array(a["y0"]), mode=oracle.MODE_NONE)
    r.run(2)
    st = r.restart_state()
    assert st["restarts"] == c["restarts_after_check1"]
    assert st["S_prev"] == pytest.approx(c["S_prev_after_check1"], rel=1e-14)
    assert st["S_r"] == pytest.approx(a["S_r0"], rel=1e-15)
    assert r.omega == 1.0
    r.run(2)
    st = r.restart_state()
    assert st["restarts"] == c["restarts_after_check2"]
    assert st["S_r"] == pytest.approx(c["S_a_check2"], rel=1e-14)
    assert st["S_prev"] == math.inf and st["t"] == 0   # a restart forgets S_prev
    assert r.omega == pytest.approx(c["omega_after_check2"], rel=1e-14)
    x, y = r.get()
    np.testing.assert_allclose(x, c["x_after_check2"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(y, c["y_after_check2"], rtol=0, atol=1e-15)


def test_necessary_criterion_every_iteration(g):
    """The necessary criterion at K = 1 (sufficient and artificial criteria off): the
    first check only records S_prev, the second restarts because its candidate rose
    above S_prev while staying under 0.8 S_r (hand scores from golden case_avg_restart)."""
    a = g["case_avg_restart"]
    olp = _olp(g)
    # check_every = 1. k=1: average == current (t=1), tie -> current, S = S_c(1) = 0.48074,
    # no restart (S_prev = inf), S_prev <- 0.48074.  k=2 (t=2): S_a(2) = 0.49162 < S_c(2),
    # S = 0.49162 > S_prev and <= 0.8 * 41/61 = 0.53770 -> restart to the average.
    p = oracle.default_params(step_size=g["eta"], primal_weight=g["omega0"], check_every=1,
                              restart=1, beta_art=10.0, beta_suff=1e-9)
    r = oracle.Run(olp, p, x_init=np.array(a["x0"]), y_init=np.array(a["y0"]), mode=oracle.MODE_NONE)
    r.run(1)
    assert r.restart_state()["restarts"] == 0
    r.run(1)
    st = r.restart_state()
    assert st["restarts"] == 1
    assert st["S_r"] == pytest.approx(a["S_a"], rel=1e-14)
    x, _ = r.get()
    np.testing.assert_allclose(x, a["after_restart"]["x"], rtol=0, atol=1e-15)


def test_sufficient_criterion_alone(g):
    """Artificial criterion off and S_prev = inf at the first check, so only the
    sufficient criterion can restart: S_a = 0.49162 <= beta_suff S_r holds for
    beta_suff = 0.75 (0.75 * 41/61 = 0.50410) and fails for 0.7 (0.47049)."""
    a = g["case_avg_restart"]
    olp = _olp(g)
    for beta_suff, want in ((0.75, 1), (0.7, 0)):
        p = oracle.default_params(step_size=g["eta"], primal_weight=g["omega0"], check_every=g["K"],
                                  restart=1, beta_art=10.0, beta_suff=beta_suff, beta_nec=0.8)
        r = oracle.Run(olp, p, x_init=np.array(a["x0"]), y_init=np.array(a["y0"]), mode=oracle.MODE_NONE)
        r.run(2)
        assert r.restart_state()["restarts"] == want, beta_suff
        if want:
            assert r.omega == pytest.approx(a["omega"], rel=1e-14)


def test_full_mode_returns_the_average(g):
    """mode full: neither current iterate meets eps_rel = 0.4 but the average at the
    K = 2 check does -> CONVERGED at k = 2 with the AVERAGE returned (golden
    case_return_average; S-4: the return flags which iterate)."""
    c = g["case_return_average"]
    olp = _olp(g)
    p = oracle.default_params(step_size=g["eta"], primal_weight=g["omega0"], check_every=g["K"],
                              restart=1, eps_rel=c["eps_rel"])
    r = oracle.Run(olp, p, x_init=np.array(c["x0"]), y_init=np.array(c["y0"]), mode=oracle.MODE_FULL)
    st = r.run(100)
    res = r.result()
    assert st == c["status"] and res["iterations"] == c["iterations"]
    assert res["returned_average"] == c["returned_average"]
    assert res["score"] == pytest.approx(c["score"], rel=1e-14)
    x, y = r.get()
    np.testing.assert_allclose(x, c["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(y, c["y"], rtol=0, atol=1e-15)


def test_dual_residual_by_bound_kind(golden):
    """r_D_j by which bounds of column j are finite, and the dual objective's bound terms
    (hand example with free, lower-only, upper-only and boxed columns; golden score_bounds)."""
    s = golden("score_bounds.json")
    lp = lp_from_dense(s["A"], s["b"], s["c"], _inf(s["lb"]), _inf(s["ub"]))
    olp = oracle.OracleLP(lp)
    sc = oracle.score(olp, s["x"], s["y"])
    assert sc["rd"] == pytest.approx(s["rd"], rel=1e-15)
    assert sc["dobj"] == s["dobj"] and sc["pobj"] == s["pobj"] and sc["rp"] == s["rp"]
    assert sc["score"] == 2.75
    # each kind alone: only the violating columns contribute
    for j, want in enumerate(s["rd_components"]):
        keep = np.zeros(lp.n, bool)
        keep[j] = True
        sub = lp_from_dense(np.asarray(s["A"])[:, keep], s["b"], np.asarray(s["c"])[keep],
                            np.asarray(_inf(s["lb"]))[keep], np.asarray(_inf(s["ub"]))[keep])
        got = oracle.score(oracle.OracleLP(sub), np.asarray(s["x"])[keep], s["y"])["rd"]
        assert got == want, (s["kinds"][j], got, want)


def test_off_bound_model_uses_corner_bounds(golden):
    """p^ counts w.r.t. M^ (lhat, uhat), not the original bounds (golden model_vs_original)."""
    e = golden("corner_examples.json")["model_vs_original"]
    st = oracle.stats(1, e["x"], None, e["lb"], e["ub"], e["lhat"], e["uhat"])
    assert st["off_bound"] == e["off_bound"]
    assert st["off_bound_model"] == e["off_bound_model"]


def test_reduced_cost_counts_at_exactly_eps(golden):
    """|z| == eps_abs: counted by d ('at 0', <=), not by the candidate count (<)."""
    e = golden("corner_examples.json")["eps_boundary"]
    st = oracle.stats(e["m"], e["x"], e["z"], e["lb"], e["ub"], eps_abs=e["eps_abs"])
    assert st["zero_rc"] == e["zero_rc"]
    assert st["candidates"] == e["candidates"]
    assert st["est_dual_pushes"] == e["est_dual"]
