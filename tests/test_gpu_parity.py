"""Parity of the CUDA path (through the C-ABI) with the CPU oracle — `-m gpu`.

Tolerances (BASELINE.json north_star, SURVEY §8(c) "Parity contract"):
  * iterates, first 1000 iterations: ||v_gpu - v_orc||_2 <= 1e-9 ||v_orc||_2 + 1e-14 sqrt(len)
  * termination: iteration count within +-1% of the oracle's (and +-1 iteration), same
    status, final objective within 1e-6 relative
  * corner statistics: bit-exact given identical (x, z)
Inputs are the seeded lpgen configs (reduced sizes spanning several plan entries,
long rows and ragged tails; full BASELINE sizes in test_gpu_fullsize.py).
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

ITER_RTOL = 1e-9
CONFIGS = ["c1", "c2-s", "c3-s", "c4-s", "c5-s"]


from parity_util import close, worst  # noqa: E402  (norm AND entry-wise bound)


@pytest.fixture(scope="module")
def problems():
    cache = {}

    def get(name):
        if name not in cache:
            lp = lpgen.config(name)
            cache[name] = (lp, oracle.OracleLP(lp), cpd.Problem.from_lp(lp))
        return cache[name]
    return get


@pytest.mark.parametrize("name", CONFIGS)
def test_power_sigma(problems, name):
    lp, olp, P = problems(name)
    assert P.power_sigma(128, 7) == pytest.approx(oracle.power_sigma(olp, 128, 7), rel=1e-12)


@pytest.mark.parametrize("name", CONFIGS)
def test_score_random_point(problems, name):
    lp, olp, P = problems(name)
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 3, lp.n)
    y = rng.standard_normal(lp.m)
    g, o = P.score(x, y), oracle.score(olp, x, y)
    for k in ("rp", "rd", "pobj", "dobj", "score"):
        assert g[k] == pytest.approx(o[k], rel=1e-12, abs=1e-300), k


def test_score_mixed_bounds():
    """Free, lower-only, upper-only and boxed columns (all branches of the S-6 terms)."""
    lp = lpgen.gen_dense(m=7, n=23, n_support=3, n_face=8, seed=9, ub=5.0, n_upper=2)
    lb, ub = lp.lb.copy(), lp.ub.copy()
    lb[:4] = -np.inf
    ub[4:8] = np.inf
    lb[8:10] = -np.inf
    ub[8:10] = np.inf
    lp.lb, lp.ub = lb, ub
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 4, lp.n)
    y = rng.standard_normal(lp.m)
    g, o = P.score(x, y), oracle.score(olp, x, y)
    for k in ("rp", "rd", "pobj", "dobj", "score"):
        assert g[k] == pytest.approx(o[k], rel=1e-12), k


@pytest.mark.parametrize("name", CONFIGS)
@pytest.mark.parametrize("restart", [1, 0])
def test_lockstep_iterates(problems, name, restart):
    """cpd_step vs oracle step, eta given explicitly (S-2), restarts as configured."""
    lp, olp, P = problems(name)
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=restart)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=restart), mode=oracle.MODE_NONE)
    k = 0
    for target in (1, 2, 3, 10, 63, 64, 65, 128, 129, 300, 640, 1000):
        S.step(target - k)
        R.run(target - k)
        k = target
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xo), (name, k, np.abs(xg - xo).max())
        assert close(yg, yo), (name, k, np.abs(yg - yo).max())


def test_2x2_hand_step_on_gpu(golden):
    """The hand-worked 2x2 iterates (tests/golden/pdhg_2x2.json) through the C-ABI."""
    g = golden("pdhg_2x2.json")
    A = np.array(g["A"])
    lp = lpgen.LP(m=2, n=2, ATp=np.array([0, 2, 4], np.int32), ATj=np.array([0, 1, 0, 1], np.int32),
                  ATx=A.T.reshape(-1).copy(), b=np.array(g["b"]), c=np.array(g["c"]),
                  lb=np.zeros(2), ub=np.full(2, np.inf))
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P, step_size=0.1, primal_weight=1.0, restart=0)
    S.set_iterate(np.array(g["x_init"]), np.array(g["y_init"]))
    for st in g["steps"]:
        S.step(1)
        x, y = S.get_iterate()
        np.testing.assert_allclose(x, st["x"], atol=1e-15, rtol=0)
        np.testing.assert_allclose(y, st["y"], atol=1e-15, rtol=0)


@pytest.mark.parametrize("name", ["c1", "c2-s", "c3-s", "c4-s"])
def test_solve_termination_parity(problems, name):
    """Phase 1 to eps_rel = 1e-4: same status, iterations within +-1%, objective 1e-6."""
    lp, olp, P = problems(name)
    S = cpd.Solver(P)
    r = S.solve()
    xo, yo, ro = oracle.solve(olp, oracle.default_params())
    assert r["status"] == ro["status"] == 0
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"])
    assert r["returned_average"] == ro["returned_average"]
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
    assert r["restarts"] == ro["restarts"]
    xg, yg = S.get_iterate()
    if r["iterations"] == ro["iterations"]:
        assert close(xg, xo, 1e-8) and close(yg, yo, 1e-8)
    # the returned point satisfies P:124-126 by the oracle's own score
    assert oracle.score(olp, xg, yg)["score"] <= 1e-4 * (1 + 1e-9)


@pytest.mark.parametrize("name", ["c1", "c2-s"])
def test_corner_push_parity(problems, name):
    """Algorithm 1 + P:391-395 stop from the SAME phase-1 point on both sides."""
    lp, olp, P = problems(name)
    xo, yo, _ = oracle.solve(olp, oracle.default_params())
    S = cpd.Solver(P)
    S.set_iterate(xo, yo)
    r, before, after = S.corner_push(seed=1001, candidate_floor=100)
    xh_o, _, z_o, ro, b_o, a_o, model = oracle.corner_push(olp, xo, yo, seed=1001, floor=100)
    assert r["status"] == ro["status"] == 0
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"])
    xg, yg, zg = S.get_iterate(z=True)
    np.testing.assert_array_equal(yg, yo)      # y returned is phase 1's
    assert close(zg, z_o, 1e-12)
    if r["iterations"] == ro["iterations"]:
        assert close(xg, xh_o, 1e-8)
    for k in ("fix_lb", "fix_ub"):
        assert before[k] == b_o[k], k
    # counts are bit-exact given identical inputs: recount the GPU's x^ with the oracle
    ref = oracle.stats(lp.m, xg, zg, lp.lb, lp.ub, model["lhat"], model["uhat"], 1e-6, 100)
    for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc", "candidates",
              "est_primal_pushes", "est_dual_pushes", "is_candidate"):
        assert after[k] == ref[k], k


@pytest.mark.parametrize("name", ["c2-s", "c5-s"])
def test_corner_lockstep_iterates(problems, name):
    """First 1000 corner iterations (ITER_LIMIT at K) match the oracle's to 1e-9."""
    lp, olp, P = problems(name)
    xo, yo, _ = oracle.solve(olp, oracle.default_params(max_iters=300))
    for K in (100, 1000):
        S = cpd.Solver(P)
        S.set_iterate(xo, yo)
        r, _, _ = S.corner_push(seed=5, max_iters=K, min_iters=10 ** 9)
        xh_o, _, _, ro, _, _, _ = oracle.corner_push(olp, xo, yo, seed=5, max_iters=K, min_iters=10 ** 9)
        assert r["status"] == ro["status"] == 1 and r["iterations"] == K
        xg, _ = S.get_iterate()
        assert close(xg, xh_o), (name, K, np.abs(xg - xh_o).max())


@pytest.mark.parametrize("name", CONFIGS)
def test_stats_bit_exact(problems, name):
    """cpd_compute_stats == oracle counts on identical (x, z, lhat, uhat), including
    values exactly at eps_abs distance and at the bounds."""
    lp, olp, P = problems(name)
    rng = np.random.default_rng(3)
    n = lp.n
    x = rng.uniform(0, 2e-6, n)
    x[::7] = 0.0
    x[1::11] = 1e-6              # exactly eps_abs above the lower bound
    z = rng.uniform(-2e-6, 2e-6, n)
    z[::5] = 1e-6
    z[2::5] = -1e-6
    lh = np.where(rng.random(n) < 0.3, x, lp.lb)
    uh = np.where(rng.random(n) < 0.3, x, lp.ub)
    g = P.stats(x, z, lh, uh, eps_abs=1e-6, floor=10)
    o = oracle.stats(lp.m, x, z, lp.lb, lp.ub, lh, uh, 1e-6, 10)
    for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc", "candidates",
              "est_primal_pushes", "est_dual_pushes", "is_candidate"):
        assert g[k] == o[k], k


def test_one_by_one():
    """Degenerate sizes: m = n = 1."""
    lp = lpgen.LP(m=1, n=1, ATp=np.array([0, 1], np.int32), ATj=np.array([0], np.int32),
                  ATx=np.array([1.0]), b=np.array([1.0]), c=np.array([1.0]), lb=np.zeros(1),
                  ub=np.array([10.0]))
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P, eps_rel=1e-9)
    r = S.solve()
    x, y = S.get_iterate()
    ro = oracle.solve(oracle.OracleLP(lp), oracle.default_params(eps_rel=1e-9))[2]
    assert r["status"] == 0 and abs(r["iterations"] - ro["iterations"]) <= 1
    assert abs(x[0] - 1) < 1e-8 and abs(y[0] - 1) < 1e-8


def test_empty_rows_and_columns():
    """Rows of A with no nonzeros (b_i = 0) and a column with no nonzeros."""
    lp = lpgen.config("c5-s")
    assert lp.meta["empty_rows"] > 0
    ATp = np.concatenate([lp.ATp, [lp.ATp[-1]]]).astype(np.int32)   # extra empty column
    lp2 = lpgen.LP(m=lp.m, n=lp.n + 1, ATp=ATp, ATj=lp.ATj, ATx=lp.ATx, b=lp.b,
                   c=np.concatenate([lp.c, [0.5]]), lb=np.zeros(lp.n + 1), ub=np.full(lp.n + 1, 100.0))
    olp = oracle.OracleLP(lp2)
    P = cpd.Problem.from_lp(lp2)
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta)
    R = oracle.Run(olp, oracle.default_params(step_size=eta), mode=oracle.MODE_NONE)
    S.step(200)
    R.run(200)
    xg, yg = S.get_iterate()
    xo, yo = R.get()
    assert close(xg, xo) and close(yg, yo)


def test_iteration_limit_and_warm_start(problems):
    lp, olp, P = problems("c2-s")
    S = cpd.Solver(P, max_iters=77)
    r = S.solve()
    ro = oracle.solve(olp, oracle.default_params(max_iters=77))[2]
    assert r["status"] == ro["status"] == 1 and r["iterations"] == 77
    # warm start from a converged point terminates at once (k = 0)
    S2 = cpd.Solver(P)
    r2 = S2.solve()
    r3 = S2.solve()
    assert r2["status"] == 0 and r3["status"] == 0 and r3["iterations"] <= 1


def test_nonfinite_is_numerical_failure():
    """Overflowing iterates report NUMERICAL_FAILURE at the first offending iteration."""
    lp = lpgen.config("c1")
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    eta = 1e150   # absurd step: overflows within a few iterations
    S = cpd.Solver(P, step_size=eta, primal_weight=1.0)
    r = S.solve()
    _, _, ro = oracle.solve(olp, oracle.default_params(step_size=eta, primal_weight=1.0))
    assert r["status"] == ro["status"] == 3
    assert r["iterations"] == ro["iterations"]


def test_graph_and_eager_identical(problems):
    lp, olp, P = problems("c4-s")
    a = cpd.Solver(P, use_graph=1)
    b = cpd.Solver(P, use_graph=0)
    ra, rb = a.solve(), b.solve()
    assert ra["iterations"] == rb["iterations"]
    xa, ya = a.get_iterate()
    xb, yb = b.get_iterate()
    assert np.array_equal(xa, xb) and np.array_equal(ya, yb)   # deterministic reductions


@pytest.mark.parametrize("name", ["c2-s", "c5-s"])
def test_trajectory_matches_oracle(problems, name):
    """Fig. 1 analogue: the steering phase's off-bound count (w.r.t. the
    ORIGINAL bounds, tolerance eps_abs, S-10) and ||b - A x_k|| every 64 iterations.
    The oracle runs the same Algorithm 1 model 64 iterations at a time in lockstep and
    counts with its own orc_stats: counts bit-exact, residual norms to 1e-9."""
    lp, olp, P = problems(name)
    xo, yo, _ = oracle.solve(olp, oracle.default_params(max_iters=3000))
    S = cpd.Solver(P)
    S.set_iterate(xo, yo)
    r, before, after = S.corner_push(seed=1001, candidate_floor=100, max_iters=5000)
    k, off, rp = S.trajectory()
    # oracle: Algorithm 1 line 2, then PDHG on M^ from (x*, 0), primal-only stop
    z = oracle.reduced_costs(olp, yo)
    lh, uh, ch, _, _ = oracle.corner_model(olp, xo, z, 1e-6, 1.0, 1001)
    p2 = oracle.default_params(max_iters=5000, primal_weight=0.0)
    R = oracle.Run(olp, p2, c=ch, lb=lh, ub=uh, x_init=xo, y_init=None, mode=oracle.MODE_PRIMAL_ONLY,
                   target=1e-4 * (1.0 + olp.nb), min_iters=100)
    ko, offo, rpo = [], [], []
    while True:
        st = R.run(64 - R.k % 64)
        if R.k % 64 == 0:
            x, _ = R.get()
            ko.append(R.k)
            offo.append(oracle.stats(lp.m, x, None, lp.lb, lp.ub)["off_bound"])
            rpo.append(float(np.linalg.norm(lp.b - olp.A_times(x))))
        if st != -1:
            break
    assert r["iterations"] == R.k, (r["iterations"], R.k)
    assert list(k) == ko
    assert list(off) == offo, (list(off)[:8], offo[:8])
    np.testing.assert_allclose(rp, rpo, rtol=1e-9, atol=1e-12)
    assert off[0] <= before["off_bound"] + before["fix_lb"] + before["fix_ub"]


@pytest.mark.parametrize("fmt", [("0", "0", "0"), ("1", "0", "0"), ("0", "1", "0"), ("1", "1", "0"),
                                 ("1", "1", "1")])
@pytest.mark.parametrize("name", ["c1", "c2-s", "c3-s", "c4-s", "c5-s"])
def test_every_spmv_format_lockstep(name, fmt, monkeypatch):
    """Each SpMV engine (TMA plan k_spmv / warp-item k_csrw (+ k_dense heavy rows,
    + column-slab passes of the rows items) for A; SELL-32 k_sell or the TMA plan for A^T) meets the
    1e-9 iterate contract, restarts on."""
    warp, sell, short = fmt
    monkeypatch.setenv("CPD_WARP", warp)
    monkeypatch.setenv("CPD_SELL", sell)
    monkeypatch.setenv("CPD_SHORT", short)
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=1)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=1), mode=oracle.MODE_NONE)
    S.step(300)
    R.run(300)
    xg, yg = S.get_iterate()
    xo, yo = R.get()
    assert close(xg, xo) and close(yg, yo), (name, fmt)
    assert P.power_sigma(128, 7) == pytest.approx(oracle.power_sigma(olp, 128, 7), rel=1e-12)


@pytest.mark.parametrize("slabs", ["2", "3", "7", "0"])
@pytest.mark.parametrize("name", ["c2-s", "c3-s", "c5-s"])
def test_short_row_slab_passes_lockstep(name, slabs, monkeypatch):
    """k_csrw slab mode: the rows items summed over 2 / 3 / 7 column slabs (running
    sums between passes, epilogue on the last) or over the long pieces' slabs with
    the passes interleaved (0); same 1e-9 iterate contract and oracle score."""
    monkeypatch.setenv("CPD_WARP", "1")
    monkeypatch.setenv("CPD_SHORT", "1")
    monkeypatch.setenv("CPD_SHORT_SLABS", slabs)
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=1)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=1), mode=oracle.MODE_NONE)
    for k in (1, 64, 300):
        S.step(k - R.k)
        R.run(k - R.k)
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xo) and close(yg, yo), (name, slabs, k)
    x = np.random.default_rng(3).uniform(0, 2, lp.n)
    y = np.random.default_rng(4).standard_normal(lp.m)
    assert P.score(x, y)["rp"] == pytest.approx(oracle.score(olp, x, y)["rp"], rel=1e-12)


@pytest.mark.parametrize("short", ["0", "1"])
@pytest.mark.parametrize("push", ["1", "0"])
@pytest.mark.parametrize("name", ["c5-s", "c2-s"])
def test_short_row_push_lockstep(name, push, short, monkeypatch):
    """The short-row push (primal step scatters a_ij x+_j into an L2-resident m-vector
    with fp64 atomics; the dual step reads it instead of gathering x+) meets the same
    1e-9 contract as the pull path; with CPD_WARP=1 so that C2's A takes the
    warp plan too; with and without the rows items' column-slab passes (which the
    push replaces for the dual step)."""
    monkeypatch.setenv("CPD_PUSH", push)
    monkeypatch.setenv("CPD_SHORT", short)
    monkeypatch.setenv("CPD_WARP", "1")
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=1)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=1), mode=oracle.MODE_NONE)
    for k in (64, 300, 1000):
        S.step(k - R.k)
        R.run(k - R.k)
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xo) and close(yg, yo), (name, push, short, k)
    # termination through the push path (c5-s hits the iteration limit on both sides)
    S2 = cpd.Solver(P, max_iters=5000)
    r = S2.solve()
    xo, yo, ro = oracle.solve(olp, oracle.default_params(max_iters=5000))
    assert r["status"] == ro["status"]
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"])
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
