"""ctypes shim over oracle/oracle.c — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module. It never touches the CUDA library and the CUDA
library never touches it.

Paper citations for every routine are in oracle/oracle.c's header and at each
function there (PAPER.md line numbers, SURVEY.md §8(c) readings).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared",
          "-D_POSIX_C_SOURCE=199309L"]
_lock = threading.Lock()
_lib = None

MODE_FULL, MODE_PRIMAL_ONLY, MODE_NONE, MODE_DUAL_ONLY = 0, 1, 2, 3
STATUS = {0: "converged", 1: "iter_limit", 2: "time_limit", 3: "numerical_failure", -1: "running"}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no SIMD/OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class LPStruct(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32),
                ("Ap", C.c_void_p), ("Aj", C.c_void_p), ("Ax", C.c_void_p),
                ("ATp", C.c_void_p), ("ATj", C.c_void_p), ("ATx", C.c_void_p),
                ("b", C.c_void_p), ("sense", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("eps_rel", C.c_double), ("eps_abs", C.c_double), ("max_iters", C.c_int64),
                ("time_limit_s", C.c_double), ("check_every", C.c_int32),
                ("step_scale", C.c_double), ("step_size", C.c_double),
                ("power_iters", C.c_int32), ("seed", C.c_uint64),
                ("primal_weight", C.c_double), ("restart", C.c_int32),
                ("beta_suff", C.c_double), ("beta_nec", C.c_double),
                ("beta_art", C.c_double), ("theta", C.c_double),
                ("method", C.c_int32), ("reflection", C.c_double), ("pid", C.c_int32),
                ("kp", C.c_double), ("ki", C.c_double), ("kd", C.c_double)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("returned_average", C.c_int32),
                ("iterations", C.c_int64), ("restarts", C.c_int64),
                ("pobj", C.c_double), ("dobj", C.c_double), ("gap", C.c_double),
                ("rp_norm", C.c_double), ("rd_norm", C.c_double), ("score", C.c_double),
                ("step_size", C.c_double), ("primal_weight", C.c_double), ("wall_s", C.c_double)]


class Score(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("rp", "rd", "pobj", "dobj", "r_p", "r_d", "r_g", "score")]


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("off_bound", "off_bound_strict", "off_bound_model",
                                         "zero_rc", "candidates", "fix_lb", "fix_ub",
                                         "est_primal_pushes", "est_dual_pushes")] + \
               [("is_candidate", C.c_int32)]


def _as_dict(s):
    return {k: getattr(s, k) for k, _ in s._fields_}


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            P = C.c_void_p
            L.orc_splitmix.restype = C.c_uint64
            L.orc_splitmix.argtypes = [C.c_uint64, C.c_int64]
            L.orc_u01.restype = C.c_double
            L.orc_u01.argtypes = [C.c_uint64, C.c_int64]
            L.orc_transpose.argtypes = [C.c_int32, C.c_int32, P, P, P, P, P, P]
            L.orc_spmv.argtypes = [C.c_int32, P, P, P, P, P]
            L.orc_norm2.restype = C.c_double
            L.orc_norm2.argtypes = [C.c_int64, P]
            L.orc_score.argtypes = [C.POINTER(LPStruct), P, P, P, C.c_double, C.c_double, P, P,
                                    C.POINTER(Score)]
            L.orc_power_sigma.restype = C.c_double
            L.orc_power_sigma.argtypes = [C.POINTER(LPStruct), C.c_int32, C.c_uint64]
            L.orc_create.restype = P
            L.orc_create.argtypes = [C.POINTER(LPStruct), C.POINTER(Params), P, P, P, P, P,
                                     C.c_int, C.c_double, C.c_int64, C.c_double]
            L.orc_run.restype = C.c_int
            L.orc_run.argtypes = [P, C.c_int64]
            L.orc_get.argtypes = [P, P, P]
            L.orc_get_z.argtypes = [P, P, P]
            L.orc_result_of.argtypes = [P, C.POINTER(Result)]
            L.orc_destroy.argtypes = [P]
            L.orc_get_eta.restype = C.c_double
            L.orc_get_eta.argtypes = [P]
            L.orc_get_omega.restype = C.c_double
            L.orc_get_omega.argtypes = [P]
            L.orc_get_k.restype = C.c_int64
            L.orc_get_k.argtypes = [P]
            L.orc_get_restart_state.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
            L.orc_reduced_costs.argtypes = [C.POINTER(LPStruct), P, P, P]
            L.orc_corner_model.argtypes = [C.c_int32, P, P, P, P, C.c_double, C.c_double,
                                           C.c_uint64, P, P, P, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]
            L.orc_stats.argtypes = [C.c_int32, C.c_int32, P, P, P, P, P, P, C.c_double,
                                    C.c_int64, C.POINTER(Stats)]
            L.orc_scale.argtypes = [C.c_int32, C.c_int32, P, P, P, C.c_int32, C.c_int32, P, P]
            L.orc_dual_corner_model.argtypes = [C.c_int32, P, P, P, C.c_double, P, P, P]
            L.orc_corner_senses.restype = C.c_int64
            L.orc_corner_senses.argtypes = [C.c_int32, P, P, C.c_double, P]
            L.orc_set_original.argtypes = [P, C.POINTER(LPStruct), P, P, P, P, P]
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def default_params(**kw) -> Params:
    """Defaults of SURVEY §8(b) cpd_params (same meaning as the CUDA side's)."""
    p = Params(eps_rel=1e-4, eps_abs=1e-6, max_iters=100000, time_limit_s=0.0, check_every=64,
               step_scale=0.9, step_size=0.0, power_iters=128, seed=7, primal_weight=0.0,
               restart=1, beta_suff=0.2, beta_nec=0.8, beta_art=0.36, theta=0.5,
               method=0, reflection=1.0, pid=0, kp=0.99, ki=0.01, kd=0.0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class OracleLP:
    """The oracle's own copy of an LP: CSR(A^T) from the generator, CSR(A) built
    by the oracle's counting-sort transpose (orc_transpose)."""

    def __init__(self, lp):
        L = lib()
        self.m, self.n = int(lp.m), int(lp.n)
        self.ATp = np.ascontiguousarray(lp.ATp, dtype=np.int32)
        self.ATj = np.ascontiguousarray(lp.ATj, dtype=np.int32)
        self.ATx = _f64(lp.ATx)
        nnz = int(self.ATp[-1])
        self.Ap = np.zeros(self.m + 1, dtype=np.int32)
        self.Aj = np.zeros(max(nnz, 1), dtype=np.int32)
        self.Ax = np.zeros(max(nnz, 1), dtype=np.float64)
        L.orc_transpose(self.n, self.m, _p(self.ATp), _p(self.ATj), _p(self.ATx),
                        _p(self.Ap), _p(self.Aj), _p(self.Ax))
        self.b = _f64(lp.b)
        self.c = _f64(lp.c)
        self.lb = _f64(lp.lb)
        self.ub = _f64(lp.ub)
        sense = getattr(lp, "sense", None)
        self.sense = None if sense is None else np.ascontiguousarray(sense, dtype=np.int8)
        self.s = LPStruct(self.m, self.n, _p(self.Ap), _p(self.Aj), _p(self.Ax),
                          _p(self.ATp), _p(self.ATj), _p(self.ATx), _p(self.b), _p(self.sense))
        self.nb = float(L.orc_norm2(self.m, _p(self.b)))

    def with_b(self, b):
        """The same LP with another right-hand side (shares every other array)."""
        import copy
        o = copy.copy(self)
        o.b = _f64(b).copy()
        o.s = LPStruct(self.m, self.n, _p(self.Ap), _p(self.Aj), _p(self.Ax),
                       _p(self.ATp), _p(self.ATj), _p(self.ATx), _p(o.b), _p(self.sense))
        o.nb = float(lib().orc_norm2(self.m, _p(o.b)))
        return o

    def with_senses(self, sense):
        """The same LP with other row senses (shares every array)."""
        import copy
        o = copy.copy(self)
        o.sense = None if sense is None else np.ascontiguousarray(sense, dtype=np.int8)
        o.s = LPStruct(self.m, self.n, _p(self.Ap), _p(self.Aj), _p(self.Ax),
                       _p(self.ATp), _p(self.ATj), _p(self.ATx), _p(self.b), _p(o.sense))
        return o

    def A_times(self, v):
        out = np.zeros(self.m)
        v = _f64(v)
        lib().orc_spmv(self.m, _p(self.Ap), _p(self.Aj), _p(self.Ax), _p(v), _p(out))
        return out

    def AT_times(self, v):
        out = np.zeros(self.n)
        v = _f64(v)
        lib().orc_spmv(self.n, _p(self.ATp), _p(self.ATj), _p(self.ATx), _p(v), _p(out))
        return out


def score(olp: OracleLP, x, y, c=None, lb=None, ub=None):
    c = olp.c if c is None else _f64(c)
    lb = olp.lb if lb is None else _f64(lb)
    ub = olp.ub if ub is None else _f64(ub)
    L = lib()
    nc = float(L.orc_norm2(olp.n, _p(c)))
    out = Score()
    x = _f64(x)
    y = _f64(y)
    L.orc_score(C.byref(olp.s), _p(c), _p(lb), _p(ub), olp.nb, nc, _p(x), _p(y), C.byref(out))
    return _as_dict(out)


def power_sigma(olp: OracleLP, iters=128, seed=7) -> float:
    return float(lib().orc_power_sigma(C.byref(olp.s), iters, seed))


def u01(seed, j) -> float:
    return float(lib().orc_u01(seed, j))


def splitmix(seed, j) -> int:
    return int(lib().orc_splitmix(seed, j))


class Run:
    """One R-PDHG run; supports lockstep stepping for parity."""

    def __init__(self, olp: OracleLP, params: Params, c=None, lb=None, ub=None, x_init=None,
                 y_init=None, mode=MODE_FULL, target=0.0, min_iters=0, eta=0.0):
        self.olp = olp
        self.params = params
        self._keep = [_f64(c) if c is not None else olp.c, _f64(lb) if lb is not None else olp.lb,
                      _f64(ub) if ub is not None else olp.ub, _f64(x_init), _f64(y_init)]
        cc, ll, uu, xi, yi = self._keep
        self.h = lib().orc_create(C.byref(olp.s), C.byref(params), _p(cc), _p(ll), _p(uu),
                                  _p(xi), _p(yi), mode, target, min_iters, eta)

    def set_original(self, olp: "OracleLP", c, lb, ub, r, s):
        """This run is the scaled image of `olp` (orc_set_original): scores on the original."""
        keep = [_f64(c), _f64(lb), _f64(ub), _f64(r), _f64(s)]
        self._keep += keep + [olp]
        lib().orc_set_original(self.h, C.byref(olp.s), *[_p(a) for a in keep])

    def run(self, steps) -> int:
        return int(lib().orc_run(self.h, steps))

    @property
    def k(self):
        return int(lib().orc_get_k(self.h))

    @property
    def eta(self):
        return float(lib().orc_get_eta(self.h))

    @property
    def omega(self):
        return float(lib().orc_get_omega(self.h))

    def restart_state(self) -> dict:
        """S_r, S_prev, t (iterations since the last restart) and the restart count."""
        sr, sp, t, nr = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        lib().orc_get_restart_state(self.h, C.byref(sr), C.byref(sp), C.byref(t), C.byref(nr))
        return dict(S_r=sr.value, S_prev=sp.value, t=t.value, restarts=nr.value)

    def get(self):
        x = np.zeros(self.olp.n)
        y = np.zeros(self.olp.m)
        lib().orc_get(self.h, _p(x), _p(y))
        return x, y

    def get_z(self):
        """The internal iterate (Halpern: the Halpern sequence z, not T(z))."""
        x = np.zeros(self.olp.n)
        y = np.zeros(self.olp.m)
        lib().orc_get_z(self.h, _p(x), _p(y))
        return x, y

    def result(self) -> dict:
        r = Result()
        lib().orc_result_of(self.h, C.byref(r))
        return _as_dict(r)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_destroy(h)
            self.h = None


class ScaledLP:
    """Diagonal preconditioning of an LP (orc_scale, R-3):
    `olp` = the scaled LP  A^ = diag(r) A diag(s), b^ = r b, c^ = s c, l^ = l / s, u^ = u / s,
    with x = s x^, y = r y^, z = z^ / s."""

    def __init__(self, olp: OracleLP, ruiz_iters=10, pc=1):
        import types
        m, n = olp.m, olp.n
        Ax = olp.Ax.copy()
        self.r = np.zeros(m)
        self.s = np.zeros(n)
        lib().orc_scale(m, n, _p(olp.Ap), _p(olp.Aj), _p(Ax), int(ruiz_iters), int(pc), _p(self.r), _p(self.s))
        nnz = int(olp.Ap[-1])
        tp = np.zeros(n + 1, np.int32)
        tj = np.zeros(max(nnz, 1), np.int32)
        tx = np.zeros(max(nnz, 1))
        lib().orc_transpose(m, n, _p(olp.Ap), _p(olp.Aj), _p(Ax), _p(tp), _p(tj), _p(tx))
        ns = types.SimpleNamespace(m=m, n=n, ATp=tp, ATj=tj[:nnz], ATx=tx[:nnz], b=self.r * olp.b,
                                   c=self.s * olp.c, lb=olp.lb / self.s, ub=olp.ub / self.s, sense=olp.sense)
        self.olp = OracleLP(ns)
        self.orig = olp


def solve_scaled(olp: OracleLP, params: Params = None, ruiz_iters=10, pc=1, x_init=None, y_init=None):
    """Phase 1 on the diagonally scaled LP, terminated by the ORIGINAL LP's criteria
    (P:119-131); returns the unscaled (x, y, result) and the ScaledLP."""
    params = params or default_params()
    sl = ScaledLP(olp, ruiz_iters, pc)
    xi = None if x_init is None else _f64(x_init) / sl.s
    yi = None if y_init is None else _f64(y_init) / sl.r
    r = Run(sl.olp, params, x_init=xi, y_init=yi)
    r.set_original(olp, olp.c, olp.lb, olp.ub, sl.r, sl.s)
    r.run(np.iinfo(np.int64).max)
    xh, yh = r.get()
    return sl.s * xh, sl.r * yh, r.result(), sl


def corner_push_scaled(olp: OracleLP, sl: "ScaledLP", x, y, params: Params = None, eps_abs=1e-6,
                       obj_scale=1.0, seed=1001, obj=None, min_iters=100, max_iters=100000, eta=0.0,
                       floor=100_000):
    """Algorithm 1 in the original space (z = c - A^T y, bound map, Uniform objective),
    steering iterations on the scaled corner model (c^ s, l^ / s, u^ / s) from x / s, y = 0,
    stopped by the ORIGINAL ||b - A x||.  Returns as corner_push."""
    params = params or default_params()
    z = reduced_costs(olp, y)
    lh, uh, ch, fl, fu = corner_model(olp, x, z, eps_abs, obj_scale, seed)
    if obj is not None:
        ch = _f64(obj)
    before = stats(olp.m, x, z, olp.lb, olp.ub, lh, uh, eps_abs, floor)
    p2 = default_params(**{k: getattr(params, k) for k, _ in Params._fields_})
    p2.max_iters = max_iters
    p2.primal_weight = 0.0
    target = params.eps_rel * (1.0 + olp.nb)
    shat, nrows_eq = corner_senses(olp, y, eps_abs)
    sc_m = sl.olp.with_senses(shat) if olp.sense is not None else sl.olp
    or_m = olp.with_senses(shat) if olp.sense is not None else olp
    r = Run(sc_m, p2, c=sl.s * ch, lb=lh / sl.s, ub=uh / sl.s, x_init=_f64(x) / sl.s, y_init=None,
            mode=MODE_PRIMAL_ONLY, target=target, min_iters=min_iters, eta=eta)
    r.set_original(or_m, ch, lh, uh, sl.r, sl.s)
    r.run(np.iinfo(np.int64).max)
    xh, _ = r.get()
    xh = sl.s * xh
    res = r.result()
    after = stats(olp.m, xh, z, olp.lb, olp.ub, lh, uh, eps_abs, floor)
    before["fix_lb"] = after["fix_lb"] = fl
    before["fix_ub"] = after["fix_ub"] = fu
    return xh, y, z, res, before, after, dict(lhat=lh, uhat=uh, chat=ch, target=target, shat=shat,
                                              rows_eq=nrows_eq)


def corner_senses(olp: OracleLP, y, eps_abs=1e-6):
    """Corner-model row senses: (shat, #rows made equality)."""
    if olp.sense is None:
        return None, 0
    shat = np.zeros(olp.m, np.int8)
    y = _f64(y)
    k = lib().orc_corner_senses(olp.m, _p(olp.sense), _p(y), eps_abs, _p(shat))
    return shat, int(k)


def solve(olp: OracleLP, params: Params = None, **kw):
    """Phase 1: R-PDHG to eps_rel (or the limits). Returns (x, y, result)."""
    params = params or default_params()
    r = Run(olp, params, **kw)
    r.run(np.iinfo(np.int64).max)
    x, y = r.get()
    return x, y, r.result()


def reduced_costs(olp: OracleLP, y, c=None):
    z = np.zeros(olp.n)
    c = olp.c if c is None else _f64(c)
    y = _f64(y)
    lib().orc_reduced_costs(C.byref(olp.s), _p(c), _p(y), _p(z))
    return z


def corner_model(olp: OracleLP, x, z, eps_abs=1e-6, obj_scale=1.0, seed=1001, lb=None, ub=None):
    """Algorithm 1 line 2: (lhat, uhat, chat, fix_lb, fix_ub)."""
    n = olp.n
    lh, uh, ch = np.zeros(n), np.zeros(n), np.zeros(n)
    fl, fu = C.c_int64(0), C.c_int64(0)
    # keep every converted array alive across the call (pointers are borrowed)
    x, z = _f64(x), _f64(z)
    lb = olp.lb if lb is None else _f64(lb)
    ub = olp.ub if ub is None else _f64(ub)
    lib().orc_corner_model(n, _p(x), _p(z), _p(lb), _p(ub),
                           eps_abs, obj_scale, seed, _p(lh), _p(uh), _p(ch),
                           C.byref(fl), C.byref(fu))
    return lh, uh, ch, int(fl.value), int(fu.value)


def stats(m, x, z=None, lb=None, ub=None, lhat=None, uhat=None, eps_abs=1e-6, floor=100_000):
    """Corner statistics a10."""
    x = _f64(x)
    n = x.size
    out = Stats()
    z, lb, ub, lhat, uhat = (_f64(a) for a in (z, lb, ub, lhat, uhat))
    lib().orc_stats(m, n, _p(x), _p(z), _p(lb), _p(ub), _p(lhat), _p(uhat), eps_abs, floor,
                    C.byref(out))
    return _as_dict(out)


def corner_push(olp: OracleLP, x, y, params: Params = None, eps_abs=1e-6, obj_scale=1.0,
                seed=1001, obj=None, min_iters=100, max_iters=100000, eta=0.0, floor=100_000):
    """Algorithm 1 with the P:391-395 stop: returns (xhat, y, z, result,
    stats_before, stats_after, model). y, z are phase-1's."""
    params = params or default_params()
    z = reduced_costs(olp, y)
    lh, uh, ch, fl, fu = corner_model(olp, x, z, eps_abs, obj_scale, seed)
    if obj is not None:
        ch = _f64(obj)
    shat, nrows_eq = corner_senses(olp, y, eps_abs)
    before = stats(olp.m, x, z, olp.lb, olp.ub, lh, uh, eps_abs, floor)
    p2 = default_params(**{k: getattr(params, k) for k, _ in Params._fields_})
    p2.max_iters = max_iters
    p2.primal_weight = 0.0   # fresh omega from ||chat||/||b|| (S-8)
    target = params.eps_rel * (1.0 + olp.nb)
    mhat = olp.with_senses(shat) if olp.sense is not None else olp
    r = Run(mhat, p2, c=ch, lb=lh, ub=uh, x_init=x, y_init=None, mode=MODE_PRIMAL_ONLY,
            target=target, min_iters=min_iters, eta=eta)
    r.run(np.iinfo(np.int64).max)
    xh, _ = r.get()
    res = r.result()
    after = stats(olp.m, xh, z, olp.lb, olp.ub, lh, uh, eps_abs, floor)
    before["fix_lb"] = after["fix_lb"] = fl
    before["fix_ub"] = after["fix_ub"] = fu
    return xh, y, z, res, before, after, dict(lhat=lh, uhat=uh, chat=ch, target=target, shat=shat,
                                              rows_eq=nrows_eq)


def dual_corner_model(olp: OracleLP, x, eps_abs=1e-6):
    """NEXT-4 dual corner model bounds (orc_dual_corner_model): (lhat, uhat, class counts)."""
    x = _f64(x)
    lh, uh = np.zeros(olp.n), np.zeros(olp.n)
    cnt = np.zeros(3, np.int64)
    lib().orc_dual_corner_model(olp.n, _p(x), _p(olp.lb), _p(olp.ub), eps_abs, _p(lh), _p(uh), _p(cnt))
    return lh, uh, dict(off=int(cnt[0]), lower=int(cnt[1]), upper=int(cnt[2]))


def dual_corner_push(olp: OracleLP, x, y, params: Params = None, eps_abs=1e-6, min_iters=100,
                     max_iters=100000, eta=0.0, floor=100_000):
    """NEXT-4 (D-1..D-4): PDHG on the dual corner model (A, b, c, lhat, uhat) from
    (x, y), stopped at k >= min_iters once every column's dual violation is <= eps_abs
    (D-3).  Returns (x, yhat, zhat, result, stats_before, stats_after, model): x is phase
    1's; d = #{|z_j| <= eps_abs} and the dual-push estimate m - d before / after."""
    params = params or default_params()
    lh, uh, cnt = dual_corner_model(olp, x, eps_abs)
    z0 = reduced_costs(olp, y)
    before = stats(olp.m, x, z0, olp.lb, olp.ub, None, None, eps_abs, floor)
    p2 = default_params(**{k: getattr(params, k) for k, _ in Params._fields_})
    p2.max_iters = max_iters
    p2.primal_weight = 0.0
    p2.eps_abs = eps_abs
    r = Run(olp, p2, c=olp.c, lb=lh, ub=uh, x_init=x, y_init=y, mode=MODE_DUAL_ONLY, target=0.0,
            min_iters=min_iters, eta=eta)
    r.run(np.iinfo(np.int64).max)
    _, yh = r.get()
    res = r.result()
    zh = reduced_costs(olp, yh)
    after = stats(olp.m, x, zh, olp.lb, olp.ub, None, None, eps_abs, floor)
    return _f64(x), yh, zh, res, before, after, dict(lhat=lh, uhat=uh, **cnt)


def corner_decide(st: dict, m: int):
    """On-the-fly choice of the push phases from the phase-1 statistics (NEXT-4, P:200-210,
    P:438-452; reading D-4): (primal, dual) booleans."""
    primal = bool(st["is_candidate"])
    dual = st["est_dual_pushes"] > 0 and min(m, st["off_bound"]) > st["zero_rc"]
    return primal, dual
