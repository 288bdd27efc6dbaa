"""Pins of the CPU oracle against what the paper and mathematics fix (`-m "not gpu"`).

Each test names the passage it pins and the kind of pin (closed form, published
value, invariant, brute force, library routine). None of them re-types the
oracle's own formula: they check it against facts a dropped term, a wrong sign,
a wrong index or a transposed operand would violate.
"""
import math

import numpy as np
import pytest
import scipy.optimize
import scipy.sparse as sp

import lpgen
import oracle
import lp_brute as brute


def lp_from_dense(A, b, c, l, u, name="dense"):
    A = np.asarray(A, float)
    m, n = A.shape
    AT = np.ascontiguousarray(A.T)
    ATp = (np.arange(n + 1) * m).astype(np.int32)
    ATj = np.tile(np.arange(m, dtype=np.int32), n)
    keep = AT.reshape(-1) != 0.0
    cnt = (AT != 0).sum(1)
    ATp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    return lpgen.LP(m=m, n=n, ATp=ATp, ATj=ATj[keep], ATx=AT.reshape(-1)[keep],
                    b=np.asarray(b, float), c=np.asarray(c, float), lb=np.asarray(l, float),
                    ub=np.asarray(u, float), name=name)


def scipy_A(lp):
    p, j, x = lp.csr_A()
    return sp.csr_matrix((x, j, p), shape=(lp.m, lp.n))


# ---------------------------------------------------------------- published values
def test_splitmix64_published_outputs(golden):
    """SplitMix64 reference outputs for seed 0 (published value; golden/splitmix64.json)."""
    g = golden("splitmix64.json")
    got = [format(oracle.splitmix(g["seed"], j), "016x") for j in range(len(g["outputs_hex"]))]
    assert got == g["outputs_hex"]
    # U(seed, j) = top 53 bits / 2^53, in [0, 1)
    u = [oracle.u01(0, j) for j in range(4)]
    assert u[0] == (int(g["outputs_hex"][0], 16) >> 11) / 2.0 ** 53
    assert all(0.0 <= v < 1.0 for v in u)


def test_pdhg_2x2_hand_steps(golden):
    """One and two PDHG updates on the hand-worked 2x2 (north_star update)."""
    g = golden("pdhg_2x2.json")
    ub = [math.inf if v == "inf" else v for v in g["ub"]]
    lp = lp_from_dense(g["A"], g["b"], g["c"], g["lb"], ub)
    olp = oracle.OracleLP(lp)
    # tau = eta/omega, sigma = eta*omega  => eta = 0.1, omega = 1 gives tau = sigma = 0.1
    p = oracle.default_params(restart=0, primal_weight=1.0, step_size=0.1)
    r = oracle.Run(olp, p, x_init=np.array(g["x_init"]), y_init=np.array(g["y_init"]),
                   mode=oracle.MODE_NONE)
    for st in g["steps"]:
        r.run(1)
        x, y = r.get()
        np.testing.assert_allclose(x, st["x"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(y, st["y"], rtol=0, atol=1e-15)


def test_pdhg_2x2_converges_to_hand_optimum(golden):
    """The 2x2 LP's unique optimum x=(1,1), y=(1.5,-0.5), obj 3 (closed form)."""
    g = golden("pdhg_2x2.json")
    lp = lp_from_dense(g["A"], g["b"], g["c"], g["lb"], [math.inf, math.inf])
    olp = oracle.OracleLP(lp)
    x, y, res = oracle.solve(olp, oracle.default_params(eps_rel=1e-10, max_iters=200000))
    assert res["status"] == 0
    np.testing.assert_allclose(x, g["optimum"]["x"], atol=1e-8)
    np.testing.assert_allclose(y, g["optimum"]["y"], atol=1e-8)
    assert abs(res["pobj"] - g["optimum"]["obj"]) < 1e-8


def test_one_by_one_closed_form():
    """min x s.t. x = 1, x in [0,10]  ->  x = 1, y = 1, z = 0 (closed form)."""
    lp = lp_from_dense([[1.0]], [1.0], [1.0], [0.0], [10.0])
    olp = oracle.OracleLP(lp)
    x, y, res = oracle.solve(olp, oracle.default_params(eps_rel=1e-9))
    assert res["status"] == 0
    assert abs(x[0] - 1.0) < 1e-8 and abs(y[0] - 1.0) < 1e-8
    assert abs(oracle.reduced_costs(olp, y)[0]) < 1e-8


# ----------------------------------------------------------- residuals and score
def test_zero_iterate_primal_residual_is_b():
    """r_P = b - A x: at x = 0 the primal residual norm is ||b||."""
    lp = lpgen.config("c1")
    olp = oracle.OracleLP(lp)
    s = oracle.score(olp, np.zeros(lp.n), np.zeros(lp.m))
    assert s["rp"] == pytest.approx(np.linalg.norm(lp.b), rel=1e-15)
    # y = 0 => z = c; with l = 0, u = inf the dual violation is the negative part of c
    assert s["rd"] == pytest.approx(np.linalg.norm(np.minimum(lp.c, 0.0)), rel=1e-14)


@pytest.mark.parametrize("n_upper", [0, 3])
def test_certificate_has_zero_score(n_upper):
    """A KKT point (x0, y0, z0) has r_P = 0, r_D = 0 and zero gap.

    With n_upper > 0 some planted variables sit at a FINITE upper bound with
    z0 < 0: the gap only closes if the dual objective carries the bound terms
    with the right signs (S-6)."""
    lp = lpgen.gen_dense(m=8, n=20, n_support=5, n_face=10, seed=3, ub=4.0, n_upper=n_upper)
    olp = oracle.OracleLP(lp)
    s = oracle.score(olp, lp.x0, lp.y0)
    assert s["score"] < 1e-13
    # and a perturbed point does not
    s2 = oracle.score(olp, lp.x0 + 1e-3, lp.y0)
    assert s2["score"] > 1e-6


@pytest.mark.parametrize("ub", [math.inf, 6.0])
def test_weak_duality_identity_on_vertices(ub):
    """c^T x - b^T y = x^T z for feasible x and any y; with box bounds the
    gap is sum (x-l) z+ + (u-x) z- >= 0 and vanishes exactly on the optimal face
    (fixing rule P:104-107). Checked on every vertex of a micro LP (brute force)."""
    lp = lpgen.gen_dense(m=4, n=9, n_support=2, n_face=5, seed=5, ub=ub,
                         n_upper=(2 if math.isfinite(ub) else 0))
    olp = oracle.OracleLP(lp)
    A = lp.dense_A()
    V = brute.vertices(A, lp.b, lp.lb, lp.ub)
    assert len(V) >= 2
    z0 = lp.z0
    on_face_seen = 0
    for x in V:
        s = oracle.score(olp, x, lp.y0)
        zp, zm = np.maximum(z0, 0), np.maximum(-z0, 0)
        fin_u = np.isfinite(lp.ub)
        expect = np.sum((x - lp.lb) * zp) + np.sum(np.where(fin_u, (np.where(fin_u, lp.ub, 0) - x) * zm, 0))
        assert s["pobj"] - s["dobj"] == pytest.approx(expect, abs=1e-9 * (1 + abs(s["pobj"])))
        assert s["pobj"] - s["dobj"] >= -1e-9
        if expect < 1e-12:
            on_face_seen += 1
            assert abs(s["pobj"] - lp.opt) < 1e-9 * (1 + abs(lp.opt))
    assert on_face_seen >= 1


# --------------------------------------------------------------- operator norm
def test_power_sigma_special_cases():
    """[[2]] -> 2 and I_5 -> 1 (closed form)."""
    assert oracle.power_sigma(oracle.OracleLP(lp_from_dense([[2.0]], [1], [1], [0], [1]))) == pytest.approx(2.0, rel=1e-12)
    I5 = lp_from_dense(np.eye(5), np.ones(5), np.ones(5), np.zeros(5), np.ones(5))
    assert oracle.power_sigma(oracle.OracleLP(I5)) == pytest.approx(1.0, rel=1e-12)


@pytest.mark.parametrize("name,rel", [("c1", 1e-9), ("c2-s", 1e-2)])
def test_power_sigma_vs_svd(name, rel):
    """sigma_hat vs the largest singular value from LAPACK SVD (library routine).

    sqrt(||A^T A v||) with ||v|| = 1 never exceeds sigma_max (it is a Rayleigh-type
    lower bound); c2-s's top singular values are clustered (random sparse), so 128
    power iterations are held to SPEC's 1% there."""
    lp = lpgen.config(name)
    smax = np.linalg.svd(lp.dense_A(), compute_uv=False)[0]
    est = oracle.power_sigma(oracle.OracleLP(lp))
    assert est == pytest.approx(smax, rel=rel)
    assert est <= smax * (1 + 1e-12)


def test_power_sigma_transport_closed_form():
    """Transportation incidence K_{S,T}: ||A||_2 = sqrt(S+T) (closed form)."""
    lp = lpgen.gen_transport(S=30, T=20, seed=1)
    assert oracle.power_sigma(oracle.OracleLP(lp)) == pytest.approx(math.sqrt(50.0), rel=1e-10)


# ---------------------------------------------------------------- iteration facts
@pytest.mark.parametrize("name", ["c1", "c2-s"])
def test_certificate_is_fixed_point(name):
    """A KKT point is a fixed point of the PDHG map (x+ = x, y+ = y), so starting
    there the iterates do not move (restarts on, termination off)."""
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    p = oracle.default_params(step_size=0.5 / oracle.power_sigma(olp))
    r = oracle.Run(olp, p, x_init=lp.x0, y_init=lp.y0, mode=oracle.MODE_NONE)
    r.run(200)
    x, y = r.get()
    assert np.max(np.abs(x - lp.x0)) < 1e-11 * (1 + np.abs(lp.x0).max())
    assert np.max(np.abs(y - lp.y0)) < 1e-11 * (1 + np.abs(lp.y0).max())


def _dense_terms(lp, x, y):
    A = lp.dense_A()
    rp = lp.b - A @ x
    z = lp.c - A.T @ y
    return np.linalg.norm(rp), z


@pytest.mark.parametrize("name", ["c1", "c2-s", "c4-s"])
def test_termination_claim_holds(name):
    """When the oracle reports CONVERGED, the returned point satisfies P:124-126
    (recomputed densely with numpy; in these LPs l = 0 so r_D is the negative
    part of z, or 0 where u is finite too)."""
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    x, y, res = oracle.solve(olp, oracle.default_params(eps_rel=1e-4))
    assert res["status"] == 0
    eps = 1e-4
    rp, z = _dense_terms(lp, x, y)
    fin_u = np.isfinite(lp.ub)
    rd = np.where(fin_u, 0.0, np.minimum(z, 0.0))
    dobj = lp.b @ y - np.sum(np.where(fin_u, np.where(fin_u, lp.ub, 0) * np.maximum(-z, 0), 0))
    pobj = lp.c @ x
    assert rp <= eps * (1 + np.linalg.norm(lp.b)) * (1 + 1e-12)
    assert np.linalg.norm(rd) <= eps * (1 + np.linalg.norm(lp.c)) * (1 + 1e-12)
    assert abs(pobj - dobj) <= eps * (1 + abs(pobj) + abs(dobj)) * (1 + 1e-12)
    assert np.all(x >= lp.lb) and np.all(x <= lp.ub)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_micro_lp_optimum_vs_vertex_enumeration(seed):
    """Converged objective vs the brute-force optimum over all vertices; x lies on
    the planted optimal face {x_j = 0 where z0_j > 0} up to the tolerance."""
    lp = lpgen.gen_dense(m=5, n=11, n_support=3, n_face=7, seed=seed)
    olp = oracle.OracleLP(lp)
    best, optv, _ = brute.optimum(lp.dense_A(), lp.b, lp.c, lp.lb, lp.ub)
    assert best == pytest.approx(lp.opt, rel=1e-9)
    x, y, res = oracle.solve(olp, oracle.default_params(eps_rel=1e-8, max_iters=400000))
    assert res["status"] == 0
    assert abs(res["pobj"] - best) <= 1e-6 * (1 + abs(best))
    off_face = lp.z0 > 0
    assert np.max(x[off_face]) < 1e-5


def test_bounded_micro_lp_vs_vertex_enumeration():
    """Box LP with active finite upper bounds: converged objective vs enumeration."""
    lp = lpgen.gen_dense(m=4, n=9, n_support=2, n_face=5, seed=11, ub=3.0, n_upper=2)
    olp = oracle.OracleLP(lp)
    best, _, _ = brute.optimum(lp.dense_A(), lp.b, lp.c, lp.lb, lp.ub)
    x, y, res = oracle.solve(olp, oracle.default_params(eps_rel=1e-8, max_iters=400000))
    assert res["status"] == 0
    assert abs(res["pobj"] - best) <= 1e-6 * (1 + abs(best))


@pytest.mark.parametrize("name", ["c3-s", "c4-s"])
def test_optimum_vs_highs(name):
    """Transportation / multicommodity optima from HiGHS (scipy.optimize.linprog,
    library routine); transportation data are integral and totally unimodular so
    the optimum is an integer."""
    lp = lpgen.config(name)
    A = scipy_A(lp)
    hr = scipy.optimize.linprog(lp.c, A_eq=A, b_eq=lp.b, bounds=(0, None), method="highs")
    assert hr.status == 0
    if name == "c3-s":
        assert hr.fun == pytest.approx(round(hr.fun), abs=1e-6)
    olp = oracle.OracleLP(lp)
    x, y, res = oracle.solve(olp, oracle.default_params(eps_rel=1e-8, max_iters=400000))
    assert res["status"] == 0
    assert abs(res["pobj"] - hr.fun) <= 1e-6 * (1 + abs(hr.fun))
    # HiGHS's own optimal (x, y) is a KKT point: the oracle's score of it is ~0,
    # which fixes the oracle's sign convention for y against an independent solver.
    s = oracle.score(olp, hr.x, hr.eqlin.marginals)
    assert s["score"] < 1e-9


def test_determinism_bitwise():
    """Identical inputs -> bitwise-identical trajectory."""
    lp = lpgen.config("c2-s")
    olp = oracle.OracleLP(lp)
    a = oracle.solve(olp, oracle.default_params(max_iters=500))
    b = oracle.solve(olp, oracle.default_params(max_iters=500))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_restart_checks_fall_on_multiples_of_K():
    """Restarts reset t at a check (t % K == 0), so checks always fall on k % K == 0
    (the property the GPU schedule's static check slot relies on)."""
    lp = lpgen.config("c2-s")
    olp = oracle.OracleLP(lp)
    r = oracle.Run(olp, oracle.default_params(), mode=oracle.MODE_NONE)
    last = 0
    for k in range(1, 1500):
        r.run(1)
        res = r.result()
        if res["restarts"] != last:
            assert k % 64 == 0
            last = res["restarts"]
    assert last >= 2


# ------------------------------------------------------------------ Algorithm 1
def test_corner_bound_map_example(golden):
    """Algorithm 1 bound map on S:331's example (z=(-1,0,1), x=(2,3,4))."""
    g = golden("corner_examples.json")["bound_map"]
    lp = lp_from_dense(np.ones((1, 3)), [1.0], [0, 0, 0], g["lb"], g["ub"])
    olp = oracle.OracleLP(lp)
    lh, uh, ch, fl, fu = oracle.corner_model(olp, g["x"], g["z"], g["eps_abs"], 1.0, 42)
    assert lh.tolist() == g["lhat"] and uh.tolist() == g["uhat"]
    assert (fl, fu) == (g["fix_lb"], g["fix_ub"])
    # Uniform([0,1]^n) objective drawn from the counter-based generator
    assert ch.tolist() == [oracle.u01(42, j) for j in range(3)]
    lh2, uh2, ch2, _, _ = oracle.corner_model(olp, g["x"], g["z"], g["eps_abs"], 1.0, 42)
    assert np.array_equal(ch, ch2)
    # strictness: |z| exactly eps_abs does not fix
    lh3, uh3, _, fl3, fu3 = oracle.corner_model(olp, g["x"], [-1e-6, 0, 1e-6], 1e-6, 1.0, 1)
    assert (fl3, fu3) == (0, 0)


def test_count_examples(golden):
    """Off-bound counts, push estimates, candidate rule."""
    g = golden("corner_examples.json")
    n = g["off_bound_all_at_lb"]["n"]
    s = oracle.stats(3, np.zeros(n), None, np.zeros(n), np.ones(n))
    assert s["off_bound"] == g["off_bound_all_at_lb"]["expect"]
    n = g["off_bound_interior"]["n"]
    s = oracle.stats(3, np.ones(n), None, np.zeros(n), np.full(n, 2.0), eps_abs=1e-6)
    assert s["off_bound"] == g["off_bound_interior"]["expect"]
    assert s["off_bound_strict"] == n
    # push estimate: m=3, p=10 off-bound, d=1 zero reduced cost
    pe = g["push_estimate"]
    n = 12
    x = np.zeros(n)
    x[:pe["p"]] = 1.0
    z = np.ones(n)
    z[:pe["d"]] = 0.0
    s = oracle.stats(pe["m"], x, z, np.zeros(n), np.full(n, 5.0))
    assert (s["off_bound"], s["zero_rc"]) == (pe["p"], pe["d"])
    assert (s["est_primal_pushes"], s["est_dual_pushes"]) == (pe["est_primal"], pe["est_dual"])
    # candidate threshold: m=10, count=20
    cd = g["candidate"]
    n = 30
    x = np.zeros(n)
    x[:cd["count"]] = 1.0
    z = np.ones(n)
    z[:cd["count"]] = 0.0
    s_f = oracle.stats(cd["m"], x, z, np.zeros(n), np.full(n, 5.0), floor=cd["floor_false"])
    s_t = oracle.stats(cd["m"], x, z, np.zeros(n), np.full(n, 5.0), floor=cd["floor_true"])
    assert s_f["candidates"] == cd["count"] and s_f["is_candidate"] == 0 and s_t["is_candidate"] == 1
    # infinite bounds never count as "at bound" (free variable is off-bound)
    s = oracle.stats(1, np.zeros(2), None, np.full(2, -np.inf), np.full(2, np.inf))
    assert s["off_bound"] == 2


@pytest.mark.parametrize("name", ["c1", "c2-s"])
def test_corner_push_properties(name):
    """Algorithm 1 + P:391-395 stop: bound-map soundness (x^_j <= x_j where z_j > eps,
    >= where z_j < -eps — exact, by projection), >= 100 iterations, the primal
    residual back at eps_rel (1 + ||b||) (recomputed with scipy), objective of M
    preserved to the phase-1 tolerance scale, y and z returned from phase 1."""
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    x, y, res = oracle.solve(olp)
    xh, y2, z, rc, before, after, model = oracle.corner_push(olp, x, y, floor=100)
    assert rc["status"] == 0
    assert rc["iterations"] >= 100
    eps = 1e-6
    assert np.all(xh[z > eps] <= x[z > eps])
    assert np.all(xh[z < -eps] >= x[z < -eps])
    A = scipy_A(lp)
    assert np.linalg.norm(lp.b - A @ xh) <= 1e-4 * (1 + np.linalg.norm(lp.b)) * (1 + 1e-12)
    assert np.array_equal(y2, y)
    np.testing.assert_allclose(z, lp.c - A.T @ y, rtol=0, atol=1e-12 * (1 + np.abs(lp.c).max()))
    assert abs(lp.c @ xh - lp.opt) <= 5e-3 * (1 + abs(lp.opt))
    assert after["off_bound_model"] <= before["off_bound"] + before["fix_lb"] + before["fix_ub"]


def test_primal_only_never_returns_before_min_iters():
    """Starting from an already-feasible x, the primal-only stop still runs >= min_iters."""
    lp = lpgen.config("c1")
    olp = oracle.OracleLP(lp)
    xh, _, _, rc, _, _, _ = oracle.corner_push(olp, lp.x0, lp.y0, min_iters=100, floor=10)
    assert rc["status"] == 0 and rc["iterations"] >= 100
    xh, _, _, rc, _, _, _ = oracle.corner_push(olp, lp.x0, lp.y0, min_iters=37, floor=10)
    assert rc["iterations"] >= 37


def test_corner_model_vertex_micro():
    """On a micro LP, running PDHG on M^ to a tight full tolerance lands on the
    c^-minimal vertex of M^, found by brute force (random objective => unique)."""
    lp = lpgen.gen_dense(m=4, n=10, n_support=2, n_face=6, seed=21)
    olp = oracle.OracleLP(lp)
    x, y, _ = oracle.solve(olp, oracle.default_params(eps_rel=1e-9, max_iters=400000))
    z = oracle.reduced_costs(olp, y)
    lh, uh, ch, fl, fu = oracle.corner_model(olp, x, z, 1e-6, 1.0, 7)
    hat = lpgen.LP(m=lp.m, n=lp.n, ATp=lp.ATp, ATj=lp.ATj, ATx=lp.ATx, b=lp.b, c=ch, lb=lh, ub=uh)
    best, optv, _ = brute.optimum(lp.dense_A(), lp.b, ch, lh, uh)
    assert len(optv) == 1
    xh, yh, res = oracle.solve(oracle.OracleLP(hat), oracle.default_params(eps_rel=1e-10, max_iters=2000000),
                               x_init=x)
    assert res["status"] == 0
    np.testing.assert_allclose(xh, optv[0], atol=1e-5)
