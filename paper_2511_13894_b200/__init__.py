"""Thin Python binding of libcpd (include/cpd.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only converts
numpy arrays / torch CUDA tensors to pointers and C structs.  There is no CPU
fallback: if libcpd.so is missing it is built with nvcc (sm_100a) or the import
fails loudly; if no CUDA device is usable the C calls fail with CPD_E_CUDA.

Names mirror the C ABI (cpd_problem_create, cpd_solve, ...); `Problem` and
`Solver` are small conveniences over the same calls.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build

__all__ = ["lib", "Params", "Result", "Stats", "CornerParams", "Problem", "Solver", "CpdError",
           "cpd_params_default", "cpd_corner_params_default", "HOST", "DEVICE", "STATUS",
           "DECLARED_SYMBOLS"]

HOST, DEVICE = 0, 1
STATUS = {-1: "running", 0: "converged", 1: "iter_limit", 2: "time_limit", 3: "numerical_failure"}

# Every symbol include/cpd.h declares (checked by tests/test_abi.py).
DECLARED_SYMBOLS = [
    "cpd_last_error", "cpd_version", "cpd_problem_create", "cpd_problem_destroy", "cpd_problem_info",
    "cpd_params_default", "cpd_corner_params_default", "cpd_solver_create", "cpd_solver_destroy",
    "cpd_solve", "cpd_corner_push", "cpd_step", "cpd_get_iterate", "cpd_set_iterate", "cpd_get_stats",
    "cpd_get_trajectory", "cpd_power_sigma", "cpd_problem_score", "cpd_compute_stats",
    "cpd_get_kernel_times", "cpd_kernel_bytes", "cpd_solver_counters",
    "cpd_partition", "cpd_nccl_get_unique_id", "cpd_problem_create_dist", "cpd_problem_dist_info",
    "cpd_problem_scale", "cpd_problem_get_scaling", "cpd_problem_set_senses", "cpd_problem_plan_info",
    "cpd_dist_layout", "cpd_dual_corner_push", "cpd_corner_decide",
    "cpd_memcache_info", "cpd_memcache_release",
]


class CpdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"cpd error {code}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("eps_rel", C.c_double), ("eps_abs", C.c_double), ("max_iters", C.c_int64),
                ("time_limit_s", C.c_double), ("check_every", C.c_int32), ("step_scale", C.c_double),
                ("step_size", C.c_double), ("power_iters", C.c_int32), ("seed", C.c_uint64),
                ("primal_weight", C.c_double), ("restart", C.c_int32), ("beta_suff", C.c_double),
                ("beta_nec", C.c_double), ("beta_art", C.c_double), ("theta", C.c_double),
                ("use_graph", C.c_int32), ("profile", C.c_int32),
                ("method", C.c_int32), ("reflection", C.c_double), ("pid", C.c_int32),
                ("kp", C.c_double), ("ki", C.c_double), ("kd", C.c_double)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("returned_average", C.c_int32), ("iterations", C.c_int64),
                ("restarts", C.c_int64), ("pobj", C.c_double), ("dobj", C.c_double), ("gap", C.c_double),
                ("rp_norm", C.c_double), ("rd_norm", C.c_double), ("score", C.c_double),
                ("step_size", C.c_double), ("primal_weight", C.c_double), ("wall_s", C.c_double)]


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("off_bound", "off_bound_strict", "off_bound_model", "zero_rc",
                                         "candidates", "fix_lb", "fix_ub", "est_primal_pushes",
                                         "est_dual_pushes")] + [("is_candidate", C.c_int32), ("rows_eq", C.c_int64)]


class CornerParams(C.Structure):
    _fields_ = [("eps_abs", C.c_double), ("obj_scale", C.c_double), ("seed", C.c_uint64),
                ("obj", C.c_void_p), ("obj_mem", C.c_int32), ("min_iters", C.c_int64),
                ("max_iters", C.c_int64), ("time_limit_s", C.c_double), ("traj_every", C.c_int32),
                ("candidate_floor", C.c_int64)]


def as_dict(s):
    return {k: getattr(s, k) for k, _ in s._fields_}


_lib = None


def lib():
    """Load libcpd.so (building it with nvcc if it is missing)."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if not os.path.exists(path):
            path = _build.build()
        L = C.CDLL(path)
        P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        sig = {
            "cpd_last_error": (C.c_char_p, []),
            "cpd_version": (C.c_int, []),
            "cpd_problem_create": (C.c_int, [I32, I32, I64, P, P, P, P, P, P, P, P, P, P, I32, I32,
                                             C.POINTER(P)]),
            "cpd_problem_destroy": (C.c_int, [P]),
            "cpd_problem_info": (C.c_int, [P, P]),
            "cpd_problem_plan_info": (C.c_int, [P, P]),
            "cpd_params_default": (None, [C.POINTER(Params)]),
            "cpd_corner_params_default": (None, [C.POINTER(CornerParams)]),
            "cpd_solver_create": (C.c_int, [P, C.POINTER(Params), C.POINTER(P)]),
            "cpd_solver_destroy": (C.c_int, [P]),
            "cpd_solve": (C.c_int, [P, C.POINTER(Result)]),
            "cpd_corner_push": (C.c_int, [P, C.POINTER(CornerParams), C.POINTER(Result),
                                          C.POINTER(Stats), C.POINTER(Stats)]),
            "cpd_step": (C.c_int, [P, I64]),
            "cpd_dual_corner_push": (C.c_int, [P, C.POINTER(CornerParams), C.POINTER(Result), C.POINTER(Stats),
                                               C.POINTER(Stats)]),
            "cpd_corner_decide": (C.c_int, [C.POINTER(Stats), I32, C.POINTER(I32), C.POINTER(I32)]),
            "cpd_get_iterate": (C.c_int, [P, P, P, P, I32]),
            "cpd_set_iterate": (C.c_int, [P, P, P, I32]),
            "cpd_get_stats": (C.c_int, [P, I64, C.POINTER(Stats)]),
            "cpd_get_trajectory": (C.c_int, [P, P, P, P, I64, C.POINTER(I64)]),
            "cpd_power_sigma": (C.c_int, [P, I32, C.c_uint64, C.POINTER(D)]),
            "cpd_problem_score": (C.c_int, [P, P, P, I32, P]),
            "cpd_compute_stats": (C.c_int, [P, P, P, P, P, D, I64, I32, C.POINTER(Stats)]),
            "cpd_get_kernel_times": (C.c_int, [P, P, P, P, I32, C.POINTER(I32), I32]),
            "cpd_kernel_bytes": (C.c_int, [P, C.c_char_p, C.POINTER(D)]),
            "cpd_memcache_info": (C.c_int, [I32, C.POINTER(I64)]),
            "cpd_memcache_release": (C.c_int, [I32]),
            "cpd_solver_counters": (C.c_int, [P, P]),
            "cpd_partition": (C.c_int, [I32, I32, P, P, I32, I32, P]),
            "cpd_dist_layout": (C.c_int, [I32, I32, P, P, I32, I32, I32, P]),
            "cpd_nccl_get_unique_id": (C.c_int, [C.c_char_p]),
            "cpd_problem_create_dist": (C.c_int, [I32, I32, C.c_char_p, I32, I32, I32, I64, P, P, P, P, P, P,
                                                  P, I32, C.POINTER(P)]),
            "cpd_problem_dist_info": (C.c_int, [P, P]),
            "cpd_problem_scale": (C.c_int, [P, I32, I32]),
            "cpd_problem_set_senses": (C.c_int, [P, P, I32]),
            "cpd_problem_get_scaling": (C.c_int, [P, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise CpdError(rc, lib().cpd_last_error().decode())
    return rc


def _ptr(a, dtype=None, device=None):
    """(pointer, mem, keepalive) for a numpy array / torch tensor / None.

    Host arrays are converted to a contiguous copy of `dtype`.  A CUDA tensor is
    passed by pointer, so it must already have exactly that dtype, be contiguous and
    live on `device` (the problem's GPU): anything else raises ValueError instead of
    being reinterpreted by the library."""
    if a is None:
        return None, HOST, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.is_cuda:
                want = {np.dtype(np.int32): torch.int32, np.dtype(np.float64): torch.float64,
                        np.dtype(np.int8): torch.int8}.get(np.dtype(dtype)) if dtype is not None else None
                if want is not None and a.dtype != want:
                    raise ValueError(f"CUDA tensor has dtype {a.dtype}, the ABI expects {want}")
                if not a.is_contiguous():
                    raise ValueError("CUDA tensor must be contiguous")
                if device is not None and a.device.index != int(device):
                    raise ValueError(f"CUDA tensor is on cuda:{a.device.index}, the problem on cuda:{device}")
                return a.data_ptr(), DEVICE, a
            a = a.numpy()
    except ImportError:
        pass
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, HOST, arr


def cpd_params_default(**kw) -> Params:
    p = Params()
    lib().cpd_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def cpd_corner_params_default(**kw) -> CornerParams:
    p = CornerParams()
    lib().cpd_corner_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def partition(m, n, ATp, ATj, world, partition):
    """cpd_partition: block bounds [world + 1] (host only, no device needed)."""
    ATp = np.ascontiguousarray(ATp, np.int32)
    ATj = np.ascontiguousarray(ATj, np.int32)
    out = np.zeros(world + 1, np.int64)
    _check(lib().cpd_partition(int(m), int(n), ATp.ctypes.data, ATj.ctypes.data, int(world), int(partition),
                               out.ctypes.data))
    return out


def dist_layout(m, n, ATp, ATj, world, partition, rank):
    """cpd_dist_layout: the slice / block layout of `rank` (host only, no device)."""
    ATp = np.ascontiguousarray(ATp, np.int32)
    ATj = np.ascontiguousarray(ATj, np.int32)
    out = np.zeros(12, np.int64)
    _check(lib().cpd_dist_layout(int(m), int(n), ATp.ctypes.data, ATj.ctypes.data, int(world), int(partition),
                                 int(rank), out.ctypes.data))
    keys = ("partition", "split", "L", "block_begin", "block_end", "own_len_m", "own_len_n", "gofs_m",
            "gofs_n", "poff_m", "poff_n", "local_rows_AT")
    return dict(zip(keys, out.tolist()))


def corner_decide(st: dict, m: int):
    """cpd_corner_decide (host only): (primal, dual) push phases from phase-1 statistics."""
    S = Stats()
    for k, _ in Stats._fields_:
        setattr(S, k, int(st.get(k, 0)))
    p, d = C.c_int32(), C.c_int32()
    _check(lib().cpd_corner_decide(C.byref(S), int(m), C.byref(p), C.byref(d)))
    return bool(p.value), bool(d.value)


def nccl_unique_id() -> bytes:
    """cpd_nccl_get_unique_id: 128 bytes, to be broadcast to every rank by the caller."""
    buf = C.create_string_buffer(128)
    _check(lib().cpd_nccl_get_unique_id(buf))
    return buf.raw


def memcache_info(device=0) -> int:
    """cpd_memcache_info: idle bytes the library's device-memory cache holds."""
    b = C.c_int64()
    _check(lib().cpd_memcache_info(int(device), C.byref(b)))
    return b.value


def memcache_release(device=0):
    """cpd_memcache_release: cudaFree every idle cached buffer of `device`."""
    _check(lib().cpd_memcache_release(int(device)))


class Problem:
    """cpd_problem_create / cpd_problem_destroy.  Arrays: numpy (host) or torch CUDA
    tensors (device); CSR(A) and/or CSR(A^T) (a missing layout is built on the device)."""

    def __init__(self, m, n, *, A=None, AT=None, b, c, lb=None, ub=None, device=0):
        self.m, self.n = int(m), int(n)
        keep = []
        ptrs = []
        mems = set()
        nnz = None
        for layout in (A, AT):
            if layout is None:
                ptrs += [None, None, None]
                continue
            p_, j_, x_ = layout
            for a, dt in ((p_, np.int32), (j_, np.int32), (x_, np.float64)):
                ptr, mem, k = _ptr(a, dt, device)
                ptrs.append(ptr)
                keep.append(k)
                mems.add(mem)
            nnz = int(j_.shape[0]) if nnz is None else nnz
        for a in (b, c, lb, ub):
            ptr, mem, k = _ptr(a, np.float64, device)
            ptrs.append(ptr)
            keep.append(k)
            if a is not None:
                mems.add(mem)
        if len(mems) != 1:
            raise ValueError("all arrays must live on the host or all on the device")
        self.mem = mems.pop()
        h = C.c_void_p()
        _check(lib().cpd_problem_create(self.m, self.n, nnz, *ptrs, self.mem, device, C.byref(h)))
        self.h = h
        self.nnz = nnz
        self.device = device

    @classmethod
    def from_lp(cls, lp, device=0, both=False, on_device=False):
        """From an lpgen.LP (CSR(A^T) given; CSR(A) built on the device unless both=True)."""
        AT = (lp.ATp, lp.ATj, lp.ATx)
        A = lp.csr_A() if both else None
        vecs = dict(b=lp.b, c=lp.c, lb=lp.lb, ub=lp.ub)
        if on_device:
            import torch
            dev = torch.device("cuda", device)
            conv = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dev)  # noqa: E731
            AT = tuple(conv(a) for a in AT)
            A = tuple(conv(a) for a in A) if A else None
            vecs = {k: conv(v) for k, v in vecs.items()}
        P = cls(lp.m, lp.n, A=A, AT=AT, device=device, **vecs)
        if getattr(lp, "sense", None) is not None:
            P.set_senses(lp.sense)
        return P

    @classmethod
    def create_dist(cls, lp, rank, world, uid: bytes, partition=-1, device=0):
        """cpd_problem_create_dist: this rank's block of the GLOBAL LP (host arrays)."""
        self = cls.__new__(cls)
        self.m, self.n = int(lp.m), int(lp.n)
        arrs = [np.ascontiguousarray(lp.ATp, np.int32), np.ascontiguousarray(lp.ATj, np.int32),
                np.ascontiguousarray(lp.ATx, np.float64)]
        vecs = [np.ascontiguousarray(v, np.float64) if v is not None else None for v in (lp.b, lp.c, lp.lb, lp.ub)]
        ptrs = [a.ctypes.data for a in arrs] + [v.ctypes.data if v is not None else None for v in vecs]
        h = C.c_void_p()
        idb = C.create_string_buffer(bytes(uid), 128)
        _check(lib().cpd_problem_create_dist(int(rank), int(world), idb, int(partition), self.m, self.n,
                                             int(lp.ATp[-1]), *ptrs, int(device), C.byref(h)))
        self.h = h
        self.nnz = int(lp.ATp[-1])
        self.mem = HOST
        self.device = device
        if getattr(lp, "sense", None) is not None:
            self.set_senses(lp.sense)
        return self

    def set_senses(self, sense):
        """cpd_problem_set_senses: int8 row senses (0 '=', 1 '<=', 2 '>='), global rows."""
        a = np.ascontiguousarray(sense, dtype=np.int8)
        _check(lib().cpd_problem_set_senses(self.h, a.ctypes.data, HOST))
        return self

    def scale(self, ruiz_iters=10, pock_chambolle=1):
        """cpd_problem_scale: diagonal preconditioning (call before creating solvers)."""
        _check(lib().cpd_problem_scale(self.h, int(ruiz_iters), int(pock_chambolle)))
        return self

    def scaling(self):
        r, s = np.zeros(self.m), np.zeros(self.n)
        _check(lib().cpd_problem_get_scaling(self.h, r.ctypes.data, s.ctypes.data))
        return r, s

    def dist_info(self):
        out = (C.c_int64 * 10)()
        _check(lib().cpd_problem_dist_info(self.h, out))
        keys = ("world", "rank", "partition", "L", "own_m", "own_n", "gofs_m", "gofs_n", "local_rows_A",
                "local_rows_AT")
        return dict(zip(keys, list(out)))

    def info(self):
        out = (C.c_int64 * 8)()
        _check(lib().cpd_problem_info(self.h, out))
        keys = ("m", "n", "nnz", "long_rows_A", "long_rows_AT", "plan_entries_A", "plan_entries_AT",
                "uniform_bounds")
        return dict(zip(keys, list(out)))

    def plan_info(self):
        """cpd_problem_plan_info: which SpMV engine paths the plans use."""
        out = (C.c_int64 * 16)()
        _check(lib().cpd_problem_plan_info(self.h, out))
        keys = ("warp", "heavy_rows", "dense_blocks", "slabs", "short_slabs", "long_rows", "long_pieces",
                "rows_items", "sell_AT", "hot_rows", "tma_entries", "cols_renumbered", "fused_rows", "fused_nnz")
        return dict(zip(keys, list(out)))

    def power_sigma(self, iters=128, seed=7):
        s = C.c_double()
        _check(lib().cpd_power_sigma(self.h, iters, seed, C.byref(s)))
        return s.value

    def score(self, x, y):
        out = np.zeros(8)
        px, mx, kx = _ptr(x, np.float64, self.device)
        py, my, ky = _ptr(y, np.float64, self.device)
        _check(lib().cpd_problem_score(self.h, px, py, mx, out.ctypes.data))
        return dict(zip(("rp", "rd", "pobj", "dobj", "r_p", "r_d", "r_g", "score"), out.tolist()))

    def stats(self, x, z=None, lhat=None, uhat=None, eps_abs=1e-6, floor=100_000):
        st = Stats()
        args = [_ptr(a, np.float64, self.device) for a in (x, z, lhat, uhat)]
        mems = {m for (p, m, _), a in zip(args, (x, z, lhat, uhat)) if a is not None}
        mem = mems.pop() if mems else HOST
        _check(lib().cpd_compute_stats(self.h, *[p for p, _, _ in args], eps_abs, floor, mem, C.byref(st)))
        return as_dict(st)

    def close(self):
        if getattr(self, "h", None):
            # solvers first (the C ABI refuses to free a problem with live solvers; a
            # garbage-collected cycle may finalise the problem before its solvers)
            for s in list(getattr(self, "_solvers", ())):
                s.close()
            if lib().cpd_problem_destroy(self.h) == 0:
                self.h = None
            else:   # a solver still alive (GC cleared the weak set first): its close() retries
                self._pending_close = True

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """cpd_solver_* calls on one Problem."""

    def __init__(self, problem: Problem, params: Params = None, **kw):
        self.problem = problem
        self.params = params or cpd_params_default(**kw)
        h = C.c_void_p()
        _check(lib().cpd_solver_create(problem.h, C.byref(self.params), C.byref(h)))
        self.h = h
        import weakref
        if not hasattr(problem, "_solvers"):
            problem._solvers = weakref.WeakSet()
        problem._solvers.add(self)

    def solve(self):
        r = Result()
        _check(lib().cpd_solve(self.h, C.byref(r)))
        return as_dict(r)

    def corner_push(self, params: CornerParams = None, **kw):
        cp = params or cpd_corner_params_default(**kw)
        keep = None
        if "obj" in kw and kw["obj"] is not None and not isinstance(kw["obj"], int):
            p, mem, keep = _ptr(kw["obj"], np.float64, self.problem.device)
            cp.obj, cp.obj_mem = p, mem
        r, before, after = Result(), Stats(), Stats()
        _check(lib().cpd_corner_push(self.h, C.byref(cp), C.byref(r), C.byref(before), C.byref(after)))
        del keep
        return as_dict(r), as_dict(before), as_dict(after)

    def dual_corner_push(self, params: CornerParams = None, **kw):
        """cpd_dual_corner_push (NEXT-4): (result, stats_before, stats_after)."""
        cp = params or cpd_corner_params_default(**kw)
        r, before, after = Result(), Stats(), Stats()
        _check(lib().cpd_dual_corner_push(self.h, C.byref(cp), C.byref(r), C.byref(before), C.byref(after)))
        return as_dict(r), as_dict(before), as_dict(after)

    def step(self, k):
        _check(lib().cpd_step(self.h, int(k)))

    def get_iterate(self, z=False):
        P = self.problem
        x, y = np.zeros(P.n), np.zeros(P.m)
        zz = np.zeros(P.n) if z else None
        _check(lib().cpd_get_iterate(self.h, x.ctypes.data, y.ctypes.data,
                                     zz.ctypes.data if z else None, HOST))
        return (x, y, zz) if z else (x, y)

    def get_iterate_device(self, x, y, z=None):
        """Copy into caller-owned torch CUDA tensors (device to device)."""
        for a in (x, y, z):
            if a is not None:
                _ptr(a, np.float64, self.problem.device)   # dtype / contiguity / device checks
        _check(lib().cpd_get_iterate(self.h, x.data_ptr(), y.data_ptr(),
                                     z.data_ptr() if z is not None else None, DEVICE))

    def set_iterate(self, x=None, y=None):
        px, mx, kx = _ptr(x, np.float64, self.problem.device)
        py, my, ky = _ptr(y, np.float64, self.problem.device)
        mem = mx if x is not None else my
        _check(lib().cpd_set_iterate(self.h, px, py, mem))

    def stats(self, floor=100_000):
        st = Stats()
        _check(lib().cpd_get_stats(self.h, floor, C.byref(st)))
        return as_dict(st)

    def trajectory(self, cap=1 << 16):
        k = np.zeros(cap, np.int64)
        off = np.zeros(cap, np.int64)
        rp = np.zeros(cap)
        n = C.c_int64()
        _check(lib().cpd_get_trajectory(self.h, k.ctypes.data, off.ctypes.data, rp.ctypes.data, cap,
                                        C.byref(n)))
        L = min(n.value, cap)
        return k[:L], off[:L], rp[:L]

    def kernel_times(self, reset=False):
        cap = 16
        names = (C.c_char_p * cap)()
        ms = np.zeros(cap)
        nl = np.zeros(cap, np.int64)
        L = C.c_int32()
        _check(lib().cpd_get_kernel_times(self.h, names, ms.ctypes.data, nl.ctypes.data, cap, C.byref(L),
                                          1 if reset else 0))
        return {names[i].decode(): (float(ms[i]), int(nl[i])) for i in range(L.value)}

    def kernel_bytes(self, name):
        b = C.c_double()
        _check(lib().cpd_kernel_bytes(self.h, name.encode(), C.byref(b)))
        return b.value

    def counters(self):
        out = (C.c_int64 * 4)()
        _check(lib().cpd_solver_counters(self.h, out))
        return dict(zip(("launches", "graph_launches", "graph_kernels_phase1", "graph_kernels_corner"),
                        list(out)))

    def close(self):
        if getattr(self, "h", None):
            lib().cpd_solver_destroy(self.h)
            self.h = None
            P = getattr(self, "problem", None)
            if P is not None and getattr(P, "_pending_close", False):
                P._pending_close = False
                P.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
