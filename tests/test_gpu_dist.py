"""The distributed (split) path on ONE GPU — `-m gpu`.

cpd_problem_create_dist with world = 1 and a forced partition runs every pass of
the multi-GPU schedule: the split product into the reduce-scatter
buffer, NCCL reduce-scatter / all-gather / allreduce over a 1-rank communicator,
the owned-slice epilogue and the device decisions on allreduced totals.  It must
meet the same parity contract against the oracle as the single-GPU path
(BASELINE.json north_star: 1e-9 over 1000 iterations, termination +-1%, objective
1e-6, counts bit-exact).  Ranks > 1 differ only in the partition and in what
the collectives move (tests/test_dist_cpu.py covers that algebra with gloo).
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
def dist_problems():
    cache = {}
    uid = cpd.nccl_unique_id()

    def get(name, part):
        if (name, part) not in cache:
            lp = lpgen.config(name)
            if name not in cache:
                cache[name] = (lp, oracle.OracleLP(lp))
            lp, olp = cache[name]
            # a fresh id per communicator
            P = cpd.Problem.create_dist(lp, 0, 1, cpd.nccl_unique_id(), partition=part, device=0)
            cache[(name, part)] = P
        lp, olp = cache[name]
        return lp, olp, cache[(name, part)]
    del uid
    return get


@pytest.mark.parametrize("part", [0, 1])
def test_dist_info(dist_problems, part):
    lp, _, P = dist_problems("c2-s", part)
    d = P.dist_info()
    assert d["world"] == 1 and d["rank"] == 0 and d["partition"] == part
    assert d["own_m"] == lp.m and d["own_n"] == lp.n
    assert d["L"] == (lp.n if part == 0 else lp.m)


@pytest.mark.parametrize("part", [0, 1])
@pytest.mark.parametrize("name", ["c2-s", "c5-s"])
def test_dist_power_and_score(dist_problems, name, part):
    lp, olp, P = dist_problems(name, part)
    assert P.power_sigma(128, 7) == pytest.approx(oracle.power_sigma(olp, 128, 7), rel=1e-12)
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 3, lp.n)
    y = rng.standard_normal(lp.m)
    g, o = P.score(x, y), oracle.score(olp, x, y)
    for k in ("rp", "rd", "pobj", "dobj", "score"):
        assert g[k] == pytest.approx(o[k], rel=1e-12), k


@pytest.mark.parametrize("part", [0, 1])
@pytest.mark.parametrize("name", ["c1", "c2-s", "c4-s", "c5-s"])
def test_dist_lockstep_iterates(dist_problems, name, part):
    lp, olp, P = dist_problems(name, part)
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
        assert close(xg, xo), (name, part, k, np.abs(xg - xo).max())
        assert close(yg, yo), (name, part, k, np.abs(yg - yo).max())


@pytest.mark.parametrize("part", [0, 1])
@pytest.mark.parametrize("name", ["c1", "c2-s", "c3-s"])
def test_dist_solve_and_corner(dist_problems, name, part):
    lp, olp, P = dist_problems(name, part)
    S = cpd.Solver(P)
    r = S.solve()
    xo, yo, ro = oracle.solve(olp, oracle.default_params())
    assert r["status"] == ro["status"] == 0
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"])
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
    # Algorithm 1 from the oracle's phase-1 point on both sides
    S.set_iterate(xo, yo)
    rc, before, after = S.corner_push(seed=1001, candidate_floor=100)
    xh_o, _, z_o, rco, b_o, a_o, model = oracle.corner_push(olp, xo, yo, seed=1001, floor=100)
    assert rc["status"] == rco["status"] == 0
    assert abs(rc["iterations"] - rco["iterations"]) <= max(1, 0.01 * rco["iterations"])
    xg, yg, zg = S.get_iterate(z=True)
    np.testing.assert_array_equal(yg, yo)
    assert close(zg, z_o, 1e-12)
    for k in ("fix_lb", "fix_ub"):
        assert before[k] == b_o[k], k
    ref = oracle.stats(lp.m, xg, zg, lp.lb, lp.ub, model["lhat"], model["uhat"], 1e-6, 100)
    for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc", "candidates"):
        assert after[k] == ref[k], k


@pytest.mark.parametrize("part", [0, 1])
@pytest.mark.parametrize("name", ["c2-s", "c5-s"])
def test_fused_p2p_split_path(name, part, monkeypatch):
    """CPD_P2P=1: the split product stores its row sums straight into the owner's
    NCCL symmetric window (peer memory) instead of a separate reduce-scatter; with
    one rank the peer is this GPU.  Same 1e-9 iterate contract and termination."""
    monkeypatch.setenv("CPD_P2P", "1")
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    P = cpd.Problem.create_dist(lp, 0, 1, cpd.nccl_unique_id(), partition=part, device=0)
    eta = 0.9 / oracle.power_sigma(olp)
    S = cpd.Solver(P, step_size=eta, restart=1)
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=1), mode=oracle.MODE_NONE)
    for k in (1, 65, 1000):
        S.step(k - R.k)
        R.run(k - R.k)
        xg, yg = S.get_iterate()
        xo, yo = R.get()
        assert close(xg, xo) and close(yg, yo), (name, part, k)
    S2 = cpd.Solver(P, max_iters=3000)
    r = S2.solve()
    xo, yo, ro = oracle.solve(olp, oracle.default_params(max_iters=3000))
    assert r["status"] == ro["status"]
    assert abs(r["iterations"] - ro["iterations"]) <= max(1, 0.01 * ro["iterations"])
    assert r["pobj"] == pytest.approx(ro["pobj"], rel=1e-6)
