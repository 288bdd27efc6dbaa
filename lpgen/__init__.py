"""Seeded synthetic LP generators (test/bench input infrastructure).

This module is the ONLY code shared by the oracle side (``oracle/``) and the CUDA
side (``paper_2511_13894_b200``): it builds problem instances and holds none of the
method's arithmetic (no PDHG step, no residual/score, no corner rule, no statistic).
Constructing ``b = A x0`` and ``c = A^T y0 + z0`` from a planted certificate is
instance construction (BASELINE.json configs 1,2,5 "construct b and c from seeded
x0 ... y0, z0"), done here with numpy/scipy.

Every generator returns an :class:`LP` holding CSR(A^T) (row j of A^T = column j
of A, row indices sorted ascending within each column) plus b, c, lb, ub and,
where the construction plants one, the optimal certificate (x0, y0, z0).

Recipes follow SURVEY.md §8(d) readings of BASELINE.json configs 1-5:

* ``c1``: tiny dense degenerate LP, m=20, n=40 (BASELINE.json config 1).
* ``c2``: random sparse LP, m=10,000, n=50,000, 8 nnz/column, 0<=x<=100 (config 2).
* ``c3``: 2,000 x 2,000 transportation LP, n=4e6, m=4,000 (config 3).
* ``c4``: 100x100 grid multicommodity flow, 50 commodities, explicit slacks (config 4).
* ``c5``: m=4e6, n=2e7, 12 distinct Zipf(1.2) rows/column, nnz=2.4e8 (config 5).

The paper's own model sets are not available; these
synthetic LPs stand in for them (large optimal faces by construction, the
paper's selection property).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = ["LP", "gen_dense", "gen_sparse", "gen_transport", "gen_multicommodity",
           "config", "CONFIGS", "transpose_csr"]


@dataclasses.dataclass
class LP:
    m: int
    n: int
    ATp: np.ndarray          # int32 [n+1]  CSR(A^T) row pointer
    ATj: np.ndarray          # int32 [nnz]  row index i of A
    ATx: np.ndarray          # float64 [nnz]
    b: np.ndarray            # float64 [m]
    c: np.ndarray            # float64 [n]
    lb: np.ndarray           # float64 [n]  (may hold -inf)
    ub: np.ndarray           # float64 [n]  (may hold +inf)
    x0: Optional[np.ndarray] = None
    y0: Optional[np.ndarray] = None
    z0: Optional[np.ndarray] = None
    opt: Optional[float] = None
    sense: Optional[np.ndarray] = None   # int8 [m]: 0 '=', 1 '<=', 2 '>=' (None: all '=')
    name: str = ""
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.ATp[-1])

    def csr_A(self):
        """CSR(A) = transpose of CSR(A^T) (scipy; input plumbing only)."""
        return transpose_csr(self.n, self.m, self.ATp, self.ATj, self.ATx)

    def dense_A(self) -> np.ndarray:
        A = np.zeros((self.m, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.ATp))
        A[self.ATj, rows] = self.ATx
        return A


def transpose_csr(nrows, ncols, p, j, x):
    """Transpose a CSR matrix (nrows x ncols) -> CSR of its transpose, sorted columns.

    Stable counting sort via numpy; used to hand CSR(A) to callers that want both
    layouts. Pure data movement.
    """
    p = np.asarray(p, dtype=np.int64)
    j = np.asarray(j)
    nnz = int(p[-1])
    counts = np.bincount(j, minlength=ncols)
    tp = np.zeros(ncols + 1, dtype=np.int64)
    np.cumsum(counts, out=tp[1:])
    order = np.argsort(j, kind="stable")
    src_row = np.repeat(np.arange(nrows, dtype=np.int32), np.diff(p))
    tj = src_row[order].astype(np.int32)
    tx = np.asarray(x)[order]
    assert tp[-1] == nnz
    return tp.astype(np.int32), tj, np.ascontiguousarray(tx, dtype=np.float64)


def _finish(m, n, ATp, ATj, ATx, x0, y0, z0, lb, ub, name, meta):
    """b = A x0, c = A^T y0 + z0 (instance construction from the planted certificate)."""
    cnt = np.diff(ATp.astype(np.int64))
    colrep = np.repeat(x0, cnt)
    b = np.bincount(ATj, weights=ATx * colrep, minlength=m).astype(np.float64)
    del colrep
    prod = ATx * y0[ATj]
    aty = np.add.reduceat(prod, ATp[:-1].astype(np.int64)) if len(prod) else np.zeros(n)
    aty = np.where(cnt > 0, aty, 0.0)  # reduceat quirk on empty segments
    c = aty + z0
    opt = float(np.dot(c, x0))
    return LP(m=m, n=n, ATp=ATp, ATj=ATj, ATx=ATx, b=b, c=c, lb=lb, ub=ub,
              x0=x0, y0=y0, z0=z0, opt=opt, name=name, meta=meta)


def gen_dense(m=20, n=40, n_support=12, n_face=30, seed=1, ub=math.inf, n_upper=0,
              name="c1"):
    """BASELINE.json config 1: dense N(0,1) A, planted optimum.

    S = n_support random columns with x0_S ~ U[1,10] (U[1, 0.9 ub] if ub < 11); Z = S + (n_face - n_support)
    more columns; z0 = 0 on Z, U[0.5,1.5] off Z; y0 ~ N(0,1). Optionally
    (``n_upper`` > 0, finite ``ub``) n_upper columns off Z are planted AT their
    upper bound with z0 = -U[0.5,1.5] (box-LP KKT), exercising the bound terms of
    the dual objective.
    """
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n))
    perm = rng.permutation(n)
    S = perm[:n_support]
    Z = perm[:n_face]
    x0 = np.zeros(n)
    x0[S] = rng.uniform(1.0, min(10.0, 0.9 * ub), n_support)
    z0 = rng.uniform(0.5, 1.5, n)
    z0[Z] = 0.0
    if n_upper:
        assert math.isfinite(ub) and n_face + n_upper <= n
        U = perm[n_face:n_face + n_upper]
        x0[U] = ub
        z0[U] = -rng.uniform(0.5, 1.5, n_upper)
    y0 = rng.standard_normal(m)
    AT = np.ascontiguousarray(A.T)
    ATp = (np.arange(n + 1) * m).astype(np.int32)
    ATj = np.tile(np.arange(m, dtype=np.int32), n)
    ATx = AT.reshape(-1).copy()
    lb = np.zeros(n)
    ubv = np.full(n, ub)
    meta = dict(recipe="dense", seed=seed, support=np.sort(S).tolist(), face=np.sort(Z).tolist())
    return _finish(m, n, ATp, ATj, ATx, x0, y0, z0, lb, ubv, name, meta)


def _zipf_sampler(m, s):
    """Exact discrete rank-frequency sampler p_r ∝ (r+1)^-s, r in [0,m) (inverse CDF)."""
    w = np.arange(1, m + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    head = min(m, 1 << 16)
    cdf_head = cdf[:head]

    def draw(rng, size):
        u = rng.random(size)
        r = np.searchsorted(cdf_head, u, side="right")
        tail = r >= head
        if tail.any():
            r[tail] = np.searchsorted(cdf, u[tail], side="right")
        np.minimum(r, m - 1, out=r)
        return r.astype(np.int32)
    return draw


def _distinct_rows(rng, n, k, m, draw):
    """n columns x k DISTINCT row indices; duplicates are redrawn (SURVEY S-18)."""
    R = draw(rng, (n, k)).astype(np.int32)
    R.sort(axis=1)
    dup = np.zeros(R.shape, dtype=bool)
    dup[:, 1:] = R[:, 1:] == R[:, :-1]
    bad = np.nonzero(dup.any(axis=1))[0]
    rounds = 0
    while bad.size:
        sub = R[bad]
        d = np.zeros(sub.shape, dtype=bool)
        d[:, 1:] = sub[:, 1:] == sub[:, :-1]
        sub[d] = draw(rng, int(d.sum()))
        sub.sort(axis=1)
        R[bad] = sub
        d = np.zeros(sub.shape, dtype=bool)
        d[:, 1:] = sub[:, 1:] == sub[:, :-1]
        bad = bad[d.any(axis=1)]
        rounds += 1
        if rounds > 10000:
            raise RuntimeError("distinct-row redraw did not converge")
    return R


def gen_sparse(m=10_000, n=50_000, per_col=8, seed=2, ub=100.0, support_frac=0.2,
               face_frac=0.4, zipf=None, name="c2"):
    """BASELINE.json configs 2 and 5.

    Each column has exactly ``per_col`` distinct rows, uniform (config 2) or
    Zipf(``zipf``) over ranks mapped by a seeded permutation (config 5), values
    U[-1,1]. x0: ``support_frac`` of columns ~U[0,10]; z0 = 0 on a face of
    ``face_frac`` columns containing the support, U[0.5,1.5] elsewhere; y0 ~ N(0,1);
    b = A x0, c = A^T y0 + z0; bounds 0 <= x <= ub.
    """
    rng = np.random.default_rng(seed)
    if zipf is None:
        def draw(r, size):
            return r.integers(0, m, size=size, dtype=np.int32)
        rowperm = None
    else:
        ranks = _zipf_sampler(m, zipf)
        rowperm = rng.permutation(m).astype(np.int32)

        def draw(r, size):
            return rowperm[ranks(r, size)]
    R = _distinct_rows(rng, n, per_col, m, draw)
    ATj = R.reshape(-1)
    del R
    ATx = rng.uniform(-1.0, 1.0, ATj.size)
    ATx[ATx == 0.0] = 0.5  # no explicit zeros (probability ~2^-53)
    ATp = (np.arange(n + 1, dtype=np.int64) * per_col).astype(np.int32)
    perm = rng.permutation(n)
    ns = int(round(support_frac * n))
    nf = int(round(face_frac * n))
    x0 = np.zeros(n)
    x0[perm[:ns]] = rng.uniform(0.0, 10.0, ns)
    z0 = rng.uniform(0.5, 1.5, n)
    z0[perm[:nf]] = 0.0
    del perm
    y0 = rng.standard_normal(m)
    lb = np.zeros(n)
    ubv = np.full(n, ub)
    rowdeg = np.bincount(ATj, minlength=m)
    meta = dict(recipe="sparse", seed=seed, per_col=per_col, zipf=zipf,
                row_nnz_max=int(rowdeg.max()), empty_rows=int((rowdeg == 0).sum()))
    del rowdeg
    return _finish(m, n, ATp, ATj, ATx, x0, y0, z0, lb, ubv, name, meta)


def gen_transport(S=2000, T=2000, seed=3, amount_max=1000, cost_max=100, name="c3"):
    """BASELINE.json config 3: balanced transportation LP.

    Column (i,j) -> i*T + j with ones in supply row i and demand row S+j.
    Supplies/demands integer U{1..amount_max}, balanced by +-1 steps at seeded
    random demand indices (kept in [1, amount_max]); costs integer U{1..cost_max}.
    """
    rng = np.random.default_rng(seed)
    s = rng.integers(1, amount_max + 1, S).astype(np.int64)
    d = rng.integers(1, amount_max + 1, T).astype(np.int64)
    D = int(s.sum() - d.sum())
    while D != 0:
        cand = np.unique(rng.integers(0, T, size=min(abs(D), T)))
        ok = cand[d[cand] < amount_max] if D > 0 else cand[d[cand] > 1]
        take = ok[:abs(D)]
        d[take] += 1 if D > 0 else -1
        D -= len(take) if D > 0 else -len(take)
    n = S * T
    m = S + T
    cols = np.arange(n, dtype=np.int64)
    ATj = np.empty(2 * n, dtype=np.int32)
    ATj[0::2] = (cols // T).astype(np.int32)
    ATj[1::2] = (S + cols % T).astype(np.int32)
    ATx = np.ones(2 * n)
    ATp = (np.arange(n + 1, dtype=np.int64) * 2).astype(np.int32)
    b = np.concatenate([s, d]).astype(np.float64)
    c = rng.integers(1, cost_max + 1, n).astype(np.float64)
    return LP(m=m, n=n, ATp=ATp, ATj=ATj, ATx=ATx, b=b, c=c, lb=np.zeros(n),
              ub=np.full(n, np.inf), name=name,
              meta=dict(recipe="transport", seed=seed, S=S, T=T, total=int(s.sum())))


def gen_multicommodity(G=100, K=50, seed=4, name="c4", implicit=False):
    """BASELINE.json config 4: grid multicommodity flow.

    Arcs both directions between 4-neighbours of a GxG grid; cost ~U[1,10],
    cap ~U[50,200]; K commodities with distinct (s,t), demand ~U[1,20].
    Columns: flows k*NA + a, then explicit capacity slacks K*NA + a (cost 0).
    Rows: conservation k*V + v (out - in = d_k[v=s_k] - d_k[v=t_k]), then capacity
    K*V + a (sum_k x_ka + s_a = cap_a). Feasible by construction: each commodity
    routed on its row-then-column L-path; a capacity below the routed load is
    raised to load+1 (count recorded in meta).

    implicit=True: the capacity rows are inequalities sum_k x_ka <= cap_a (row
    sense 1) without slack columns, the form practical LP solvers use and the
    paper's corner rule for.
    """
    rng = np.random.default_rng(seed)
    V = G * G
    tails, heads = [], []
    for r in range(G):
        for cc in range(G - 1):
            u, v = r * G + cc, r * G + cc + 1
            tails += [u, v]
            heads += [v, u]
    for r in range(G - 1):
        for cc in range(G):
            u, v = r * G + cc, (r + 1) * G + cc
            tails += [u, v]
            heads += [v, u]
    tail = np.array(tails, dtype=np.int64)
    head = np.array(heads, dtype=np.int64)
    NA = tail.size
    cost = rng.uniform(1.0, 10.0, NA)
    cap = rng.uniform(50.0, 200.0, NA)
    pairs = set()
    src, dst = [], []
    while len(src) < K:
        s_, t_ = (int(v) for v in rng.integers(0, V, 2))
        if s_ == t_ or (s_, t_) in pairs:
            continue
        pairs.add((s_, t_))
        src.append(s_)
        dst.append(t_)
    dem = rng.uniform(1.0, 20.0, K)
    arc_id = {(int(a), int(bb)): i for i, (a, bb) in enumerate(zip(tail, head))}
    x0 = np.zeros(K * NA + NA)
    load = np.zeros(NA)
    for k in range(K):
        r1, c1 = divmod(src[k], G)
        r2, c2 = divmod(dst[k], G)
        path = []
        cc = c1
        while cc != c2:
            nc = cc + (1 if c2 > cc else -1)
            path.append(arc_id[(r1 * G + cc, r1 * G + nc)])
            cc = nc
        r = r1
        while r != r2:
            nr = r + (1 if r2 > r else -1)
            path.append(arc_id[(r * G + c2, nr * G + c2)])
            r = nr
        for a in path:
            x0[k * NA + a] += dem[k]
            load[a] += dem[k]
    raised = load > cap
    cap[raised] = load[raised] + 1.0
    x0[K * NA:] = cap - load
    n = K * NA + NA
    m = K * V + NA
    # CSR(A^T): flow (k,a): rows k*V+tail (+1), k*V+head (-1), K*V+a (+1), sorted.
    kk = np.repeat(np.arange(K, dtype=np.int64), NA)
    aa = np.tile(np.arange(NA, dtype=np.int64), K)
    r_t = kk * V + tail[aa]
    r_h = kk * V + head[aa]
    r_c = K * V + aa
    lo = np.minimum(r_t, r_h)
    hi = np.maximum(r_t, r_h)
    v_lo = np.where(r_t < r_h, 1.0, -1.0)
    ATj = np.empty(3 * K * NA + NA, dtype=np.int32)
    ATx = np.empty(3 * K * NA + NA)
    ATj[0:3 * K * NA:3] = lo
    ATj[1:3 * K * NA:3] = hi
    ATj[2:3 * K * NA:3] = r_c
    ATx[0:3 * K * NA:3] = v_lo
    ATx[1:3 * K * NA:3] = -v_lo
    ATx[2:3 * K * NA:3] = 1.0
    ATj[3 * K * NA:] = (K * V + np.arange(NA)).astype(np.int32)
    ATx[3 * K * NA:] = 1.0
    ATp = np.concatenate([np.arange(K * NA + 1, dtype=np.int64) * 3,
                          3 * K * NA + np.arange(1, NA + 1, dtype=np.int64)]).astype(np.int32)
    b = np.zeros(m)
    for k in range(K):
        b[k * V + src[k]] += dem[k]
        b[k * V + dst[k]] -= dem[k]
    b[K * V:] = cap
    c = np.concatenate([np.tile(cost, K), np.zeros(NA)])
    meta = dict(recipe="multicommodity", seed=seed, G=G, K=K, NA=NA, raised_caps=int(raised.sum()),
                implicit=implicit)
    if implicit:   # drop the slack columns; capacity rows become '<='
        nf = K * NA
        lp = LP(m=m, n=nf, ATp=ATp[:nf + 1].copy(), ATj=ATj[:3 * nf].copy(), ATx=ATx[:3 * nf].copy(), b=b,
                c=c[:nf].copy(), lb=np.zeros(nf), ub=np.full(nf, np.inf), x0=x0[:nf].copy(), name=name, meta=meta)
        lp.sense = np.concatenate([np.zeros(K * V, np.int8), np.ones(NA, np.int8)])
        return lp
    return LP(m=m, n=n, ATp=ATp, ATj=ATj, ATx=ATx, b=b, c=c, lb=np.zeros(n),
              ub=np.full(n, np.inf), x0=x0, name=name, meta=meta)


# name -> (factory, kwargs). "full" sizes are BASELINE.json's; "-s" variants are the
# reduced sizes parity tests use (same recipes, several tiles + ragged tails).
CONFIGS = {
    "c1": (gen_dense, dict(m=20, n=40, n_support=12, n_face=30, seed=1)),
    "c2": (gen_sparse, dict(m=10_000, n=50_000, per_col=8, seed=2, ub=100.0)),
    "c3": (gen_transport, dict(S=2000, T=2000, seed=3)),
    "c4": (gen_multicommodity, dict(G=100, K=50, seed=4)),
    "c5": (gen_sparse, dict(m=4_000_000, n=20_000_000, per_col=12, seed=5, ub=100.0,
                            zipf=1.2, name="c5")),
    # reduced variants
    "c2-s": (gen_sparse, dict(m=1000, n=5000, per_col=8, seed=12, ub=100.0, name="c2-s")),
    "c3-s": (gen_transport, dict(S=60, T=50, seed=13, name="c3-s")),
    "c4-s": (gen_multicommodity, dict(G=10, K=5, seed=14, name="c4-s")),
    "c4-ineq": (gen_multicommodity, dict(G=100, K=50, seed=4, name="c4-ineq", implicit=True)),
    "c4-s-ineq": (gen_multicommodity, dict(G=10, K=5, seed=14, name="c4-s-ineq", implicit=True)),
    "c5-s": (gen_sparse, dict(m=20_000, n=100_000, per_col=12, seed=15, ub=100.0,
                              zipf=1.2, name="c5-s")),
}


def config(name: str, **overrides) -> LP:
    fn, kw = CONFIGS[name]
    kw = dict(kw)
    kw.update(overrides)
    kw.setdefault("name", name)
    return fn(**kw)
