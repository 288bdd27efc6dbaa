"""Parity through the dual step's full-size engine paths on reduced LPs (`-m gpu`).

At the default thresholds only the full C5 LP reaches the heavy-row dense-block
kernel (k_dense: rows >= 131,072 nonzeros) and long-row pieces cut at several
4 Mi-column slab boundaries; c5-s (20,000 x 100,000, Zipf rows, top row 95k
nonzeros) is a single slab without heavy rows.  The plan thresholds are runtime
env overrides (CPD_HEAVY_MIN, CPD_SLAB_COLS, read at problem creation), so here
c5-s is planned with heavy rows >= 4,096 nonzeros and 8,192-column slabs (13 slabs
for the long pieces, 2 column halves for the short rows): every sub-kernel of the
full-size dual step runs — k_dense, multi-slab pieces, the short rows' slab passes,
k_finish (CTA-per-row and warp-per-row) — and is held to the north_star contract
(iterates within 1e-9 over 1000 iterations with restarts on and off, corner
iterates, termination within +-1% with the objective to 1e-6), element-wise and in
norm (tests/parity_util.py).
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

FORCE = {"CPD_HEAVY_MIN": "4096", "CPD_SLAB_COLS": "8192", "CPD_WARP": "1", "CPD_SHORT": "1"}
# a Zipf(1.2) LP the oracle solves to eps_rel = 1e-4 in seconds (same recipe as C5)
ZIPF_TERM = dict(m=3000, n=18000, per_col=12, seed=26, ub=100.0, zipf=1.2, name="c5-xs")


@pytest.fixture(scope="module")
def forced():
    """c5-s planned with the full-size engine paths (env read at creation only)."""
    import os
    old = {k: os.environ.get(k) for k in FORCE}
    os.environ.update(FORCE)
    try:
        lp = lpgen.config("c5-s")
        P = cpd.Problem.from_lp(lp)
        lpz = lpgen.gen_sparse(**ZIPF_TERM)
        Pz = cpd.Problem.from_lp(lpz)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return lp, oracle.OracleLP(lp), P, lpz, oracle.OracleLP(lpz), Pz


def test_forced_plan_reaches_every_engine(forced):
    lp, olp, P, lpz, olpz, Pz = forced
    pi = P.plan_info()
    assert pi["warp"] == 1
    assert pi["heavy_rows"] >= 2, pi
    assert pi["dense_blocks"] >= 12, pi
    assert pi["slabs"] >= 12, pi
    assert pi["short_slabs"] >= 2, pi
    assert pi["long_pieces"] > pi["long_rows"] - pi["heavy_rows"], pi   # rows cut into several pieces
    # the default plan of the same LP has none of these
    Pd = cpd.Problem.from_lp(lp)
    d = Pd.plan_info()
    assert d["heavy_rows"] == 0 and d["slabs"] == 1, d


@pytest.mark.parametrize("restart", [1, 0])
def test_forced_lockstep_1000(forced, restart):
    lp, olp, P, *_ = forced
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=restart)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=restart), mode=oracle.MODE_NONE)
    k = 0
    for target in (1, 2, 63, 64, 65, 128, 129, 500, 1000):
        S.step(target - k)
        R.run(target - k)
        k = target
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xo), (k, worst(xg, xo))
        assert close(yg, yo), (k, worst(yg, yo))
    assert S.counters()["launches"] > 0


def test_forced_power_sigma_and_score(forced):
    lp, olp, P, *_ = forced
    assert P.power_sigma(128, 7) == pytest.approx(oracle.power_sigma(olp, 128, 7), rel=1e-12)
    rng = np.random.default_rng(8)
    x, y = rng.uniform(0, 3, lp.n), rng.standard_normal(lp.m)
    g, o = P.score(x, y), oracle.score(olp, x, y)
    for k in ("rp", "rd", "pobj", "dobj", "score"):
        assert g[k] == pytest.approx(o[k], rel=1e-12), k


def test_forced_corner_lockstep(forced):
    lp, olp, P, *_ = forced
    xo, yo, _ = oracle.solve(olp, oracle.default_params(max_iters=300))
    S = cpd.Solver(P)
    S.set_iterate(xo, yo)
    r, before, after = S.corner_push(seed=5, max_iters=1000, min_iters=10 ** 9)
    xh, _, z, ro, b_o, a_o, model = oracle.corner_push(olp, xo, yo, seed=5, max_iters=1000, min_iters=10 ** 9)
    assert r["status"] == ro["status"] == 1 and r["iterations"] == 1000
    xg, yg, zg = S.get_iterate(z=True)
    assert close(xg, xh), worst(xg, xh)
    assert close(zg, z, 1e-12), worst(zg, z)
    for k in ("fix_lb", "fix_ub", "off_bound", "off_bound_strict", "zero_rc", "candidates"):
        assert before[k] == b_o[k], k
    ref = oracle.stats(lp.m, xg, zg, lp.lb, lp.ub, model["lhat"], model["uhat"], 1e-6, 100_000)
    for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc", "candidates"):
        assert after[k] == ref[k], k


def test_forced_termination_zipf(forced):
    """A Zipf(1.2) LP (C5's recipe, reduced to 3,000 x 18,000) through the forced engine
    paths, to eps_rel = 1e-4.  Plain R-PDHG does not get there on these LPs (oracle, a
    2,000 x 10,000 one: score 0.07 after 60,000 iterations; the Zipf head makes ||A||
    huge), so both sides run with the diagonal preconditioning (R-3; oracle:
    5,809 iterations, 8 s): same status,
    iterations within +-1%, objective to 1e-6; then the steering phase from the same
    phase-1 point stops at the same iteration +-1%."""
    *_, lpz, olpz, Pz = forced
    pz = Pz.plan_info()
    assert pz["heavy_rows"] >= 1 and pz["slabs"] >= 2, pz
    Pz.scale(10, 1)
    S = cpd.Solver(Pz, max_iters=100000)
    r = S.solve()
    xo, yo, ro, sl = oracle.solve_scaled(olpz, oracle.default_params(max_iters=100000))
    assert r["status"] == ro["status"] == 0, (r, ro)
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"]), (r, ro)
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
    S.close()
    S2 = cpd.Solver(Pz)
    S2.set_iterate(xo, yo)
    rc, _, _ = S2.corner_push(seed=1001, candidate_floor=100)
    _, _, _, rco, _, _, _ = oracle.corner_push_scaled(olpz, sl, xo, yo, seed=1001, floor=100)
    assert rc["status"] == rco["status"] == 0
    assert abs(rc["iterations"] - rco["iterations"]) <= max(1, 0.01 * rco["iterations"]), (rc, rco)


@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_short_row_sell_modes(mode, monkeypatch):
    """The short-row suffix of A's warp plan: rows items (0), one SELL-32 pass (1) or two
    column-half SELL passes with running sums (2, C5's default): 1e-9 lockstep with
    restarts, check passes and power iteration included."""
    monkeypatch.setenv("CPD_SSELL", mode)
    monkeypatch.setenv("CPD_WARP", "1")
    lp = lpgen.config("c5-s")
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    assert P.plan_info()["warp"] == 1
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=1)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=1), mode=oracle.MODE_NONE)
    for k in (1, 64, 65, 300):
        S.step(k - R.k)
        R.run(k - R.k)
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xo) and close(yg, yo), (mode, k, worst(xg, xo), worst(yg, yo))
    assert P.power_sigma(128, 7) == pytest.approx(oracle.power_sigma(olp, 128, 7), rel=1e-12)
    S2 = cpd.Solver(P, max_iters=2000)
    r = S2.solve()
    _, _, ro = oracle.solve(olp, oracle.default_params(max_iters=2000))
    assert r["status"] == ro["status"] and r["iterations"] == ro["iterations"]
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)


@pytest.mark.parametrize("hotd", ["0", "1", "3", "6", "16"])
def test_hot_row_fusion_lockstep(hotd, monkeypatch):
    """Hot-row fusion: the primal step forms A x+ of the longest rows from
    per-lane shared-memory accumulators over the last entries of each lane (A^T's SELL
    lanes hold their entries in descending row order; earlier hot entries are re-read),
    the fused dual step sums the per-warp partials instead of running k_dense on those
    rows.  Off, one, three, six (the default) and sixteen rows (> one SELL round of
    entries per lane: the re-read path) — 1e-9 lockstep over 1000 iterations with
    restarts (check passes use the unfused plan), graph vs eager bit-identical (the
    fused sums are in a fixed order), termination objective vs the oracle."""
    for k, v in FORCE.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("CPD_HOTD", hotd)
    lp = lpgen.config("c5-s")
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    pi = P.plan_info()
    assert pi["fused_rows"] == min(int(hotd), pi["heavy_rows"]), pi
    if hotd == "16":
        assert pi["fused_rows"] > 6, pi
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=1)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=1), mode=oracle.MODE_NONE)
    k = 0
    for target in (1, 2, 64, 65, 300, 1000):
        S.step(target - k)
        R.run(target - k)
        k = target
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xo) and close(yg, yo), (hotd, k, worst(xg, xo), worst(yg, yo))
    a = cpd.Solver(P, max_iters=700, use_graph=1)
    b = cpd.Solver(P, max_iters=700, use_graph=0)
    ra, rb = a.solve(), b.solve()
    assert ra["iterations"] == rb["iterations"] == 700
    xa, ya = a.get_iterate()
    xb, yb = b.get_iterate()
    assert np.array_equal(xa, xb) and np.array_equal(ya, yb)
    _, _, ro = oracle.solve(olp, oracle.default_params(max_iters=700))
    assert ra["status"] == ro["status"] and ra["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)


def test_hot_row_fusion_solve_time_switch(forced, monkeypatch):
    """CPD_FUSE=0 at solve time runs the unfused plan on the same (fused-planned)
    problem; both agree with the oracle's corner push (Algorithm 1 uses the same
    primal/dual pair) and termination."""
    lp, olp, P, *_ = forced
    assert P.plan_info()["fused_rows"] >= 2
    xo, yo, ro = oracle.solve(olp, oracle.default_params(max_iters=3000))
    for fuse in ("1", "0"):
        monkeypatch.setenv("CPD_FUSE", fuse)
        S = cpd.Solver(P, max_iters=3000)
        r = S.solve()
        assert r["status"] == ro["status"] and abs(r["iterations"] - ro["iterations"]) <= max(1, ro["iterations"] // 100)
        assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
        S = cpd.Solver(P)
        S.set_iterate(xo, yo)
        rc, _, _ = S.corner_push(seed=3, max_iters=400, min_iters=10 ** 9)
        xh, _, _, rco, _, _, _ = oracle.corner_push(olp, xo, yo, seed=3, max_iters=400, min_iters=10 ** 9)
        xg, _ = S.get_iterate()
        assert rc["iterations"] == rco["iterations"] == 400
        assert close(xg, xh), (fuse, worst(xg, xh))


@pytest.mark.parametrize("hotd", ["0", "6", "16"])
@pytest.mark.parametrize("pid", [0, 1])
def test_hot_row_fusion_halpern_lockstep(hotd, pid, monkeypatch):
    """Hot-row fusion under the reflected restarted Halpern method (NEXT-1): the fused
    primal step forms A xh of the longest rows from xh_j, the dual step's k_finish sums
    those partials — Halpern iterates (z = T-sequence, T(z) returned) within 1e-9 of the
    oracle over 1000 iterations with restarts, PID off and on; the corner push (Algorithm
    1 on the Halpern pair) with the fused rows against the oracle's."""
    for k, v in FORCE.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("CPD_HOTD", hotd)
    lp = lpgen.config("c5-s")
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.from_lp(lp)
    assert P.plan_info()["fused_rows"] == min(int(hotd), P.plan_info()["heavy_rows"])
    eta = 0.9 / oracle.power_sigma(olp)
    kw = dict(step_size=eta, restart=1, method=1, pid=pid)
    S = cpd.Solver(P, **kw)
    R = oracle.Run(olp, oracle.default_params(**kw), mode=oracle.MODE_NONE)
    k = 0
    for target in (1, 2, 64, 65, 300, 1000):
        S.step(target - k)
        R.run(target - k)
        k = target
        xg, yg = S.get_iterate()
        xo, yo = R.get_z()
        assert close(xg, xo) and close(yg, yo), (hotd, pid, k, worst(xg, xo), worst(yg, yo))
    assert R.restart_state()["restarts"] >= 1
    if pid == 1 and hotd == "6":
        xo, yo, _ = oracle.solve(olp, oracle.default_params(max_iters=500, method=1, pid=1))
        S = cpd.Solver(P, method=1, pid=1)
        S.set_iterate(xo, yo)
        rc, _, _ = S.corner_push(seed=3, max_iters=300, min_iters=10 ** 9)
        xh, _, _, rco, _, _, _ = oracle.corner_push(olp, xo, yo, params=oracle.default_params(method=1, pid=1),
                                                    seed=3, max_iters=300, min_iters=10 ** 9)
        xg, _ = S.get_iterate()
        assert rc["iterations"] == rco["iterations"] == 300
        assert close(xg, xh), worst(xg, xh)
