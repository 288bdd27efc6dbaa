"""Validation and error paths of the §8(b) boundary on the GPU (`-m gpu`).

include/cpd.h promises negative codes (never a crash, never a silent reinterpretation)
for invalid input: CPD_E_CSR for a bad row pointer, a column out of range, an unsorted
or duplicate column, an explicit zero or a CSR(A) / CSR(A^T) mismatch; CPD_E_NONFINITE
for NaN/Inf in A, b or c; CPD_E_BOUNDS for lb > ub, NaN bounds, lb = +inf, ub = -inf;
CPD_E_STATE for scale / set_senses while a solver is alive.  Each case corrupts one
array of a small valid LP (both on the host and as device tensors), checks the code
and the offending index in the message, then checks the untouched LP still creates.
"""
import math

import numpy as np
import pytest

import lpgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_13894_b200 as cpd  # noqa: E402

E_ARG, E_DIM, E_BOUNDS, E_CSR, E_NONFINITE, E_STATE = -1, -2, -3, -4, -5, -8


@pytest.fixture(scope="module")
def lp():
    return lpgen.config("c2-s")


def arrays(lp):
    A = lp.csr_A()
    return dict(Ap=A[0].copy(), Aj=A[1].copy(), Ax=A[2].copy(), ATp=lp.ATp.copy(), ATj=lp.ATj.copy(),
                ATx=lp.ATx.copy(), b=lp.b.copy(), c=lp.c.copy(), lb=lp.lb.copy(), ub=lp.ub.copy())


def create(lp, a, layouts=("AT",), on_device=False):
    conv = (lambda v: torch.as_tensor(np.ascontiguousarray(v)).cuda()) if on_device else (lambda v: v)
    A = (conv(a["Ap"]), conv(a["Aj"]), conv(a["Ax"])) if "A" in layouts else None
    AT = (conv(a["ATp"]), conv(a["ATj"]), conv(a["ATx"])) if "AT" in layouts else None
    return cpd.Problem(lp.m, lp.n, A=A, AT=AT, b=conv(a["b"]), c=conv(a["c"]), lb=conv(a["lb"]),
                       ub=conv(a["ub"]))


def expect(lp, a, code, where=None, **kw):
    with pytest.raises(cpd.CpdError) as ei:
        create(lp, a, **kw)
    assert ei.value.code == code, str(ei.value)
    if where is not None:
        assert str(where) in str(ei.value), str(ei.value)


@pytest.mark.parametrize("on_device", [False, True])
def test_valid_lp_creates(lp, on_device):
    P = create(lp, arrays(lp), layouts=("A", "AT"), on_device=on_device)
    assert P.info()["nnz"] == lp.ATp[-1]


@pytest.mark.parametrize("on_device", [False, True])
def test_bad_rowptr(lp, on_device):
    a = arrays(lp)
    a["ATp"][7], a["ATp"][8] = a["ATp"][8], a["ATp"][7]   # decreasing pair
    expect(lp, a, E_CSR, "rowptr", on_device=on_device)
    a = arrays(lp)
    a["ATp"][0] = 1
    expect(lp, a, E_CSR, "rowptr at index 0", on_device=on_device)


@pytest.mark.parametrize("on_device", [False, True])
def test_column_out_of_range(lp, on_device):
    a = arrays(lp)
    a["ATj"][11] = lp.m   # row index of A^T entry = column of A^T must be < m
    expect(lp, a, E_CSR, "out of range at nonzero 11", on_device=on_device)
    a = arrays(lp)
    a["ATj"][5] = -3
    expect(lp, a, E_CSR, "out of range at nonzero 5", on_device=on_device)


@pytest.mark.parametrize("on_device", [False, True])
def test_unsorted_and_duplicate_columns(lp, on_device):
    a = arrays(lp)
    s, e = int(a["ATp"][3]), int(a["ATp"][4])
    assert e - s >= 2
    a["ATj"][s], a["ATj"][s + 1] = a["ATj"][s + 1], a["ATj"][s]   # unsorted
    expect(lp, a, E_CSR, f"at nonzero {s + 1}", on_device=on_device)
    a = arrays(lp)
    a["ATj"][s + 1] = a["ATj"][s]                                  # duplicate (i, j)
    expect(lp, a, E_CSR, "strictly increasing", on_device=on_device)


@pytest.mark.parametrize("on_device", [False, True])
def test_explicit_zero_and_nonfinite_value(lp, on_device):
    a = arrays(lp)
    a["ATx"][17] = 0.0
    expect(lp, a, E_CSR, "nonzero 17", on_device=on_device)
    a = arrays(lp)
    a["ATx"][19] = math.nan
    expect(lp, a, E_CSR, "nonzero 19", on_device=on_device)


@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("vec,idx,val", [("b", 9, math.nan), ("b", 0, math.inf), ("c", 33, math.nan),
                                         ("c", 4999, -math.inf)])
def test_nonfinite_b_c(lp, on_device, vec, idx, val):
    a = arrays(lp)
    a[vec][idx] = val
    expect(lp, a, E_NONFINITE, idx, on_device=on_device)


@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("l,u", [(5.0, 4.0), (math.nan, 1.0), (0.0, math.nan), (math.inf, math.inf),
                                 (-math.inf, -math.inf)])
def test_bad_bounds(lp, on_device, l, u):
    a = arrays(lp)
    a["lb"][21], a["ub"][21] = l, u
    expect(lp, a, E_BOUNDS, 21, on_device=on_device)


def test_infinite_bounds_are_allowed(lp):
    a = arrays(lp)
    a["lb"][:10] = -math.inf
    a["ub"][:20] = math.inf
    create(lp, a)


@pytest.mark.parametrize("on_device", [False, True])
def test_A_AT_mismatch(lp, on_device):
    a = arrays(lp)
    a["Ax"][40] *= 2.0   # CSR(A) no longer the transpose of CSR(A^T)
    expect(lp, a, E_CSR, "different matrices", layouts=("A", "AT"), on_device=on_device)
    a = arrays(lp)
    # same values, one entry moved to another (valid, still sorted) column of its row
    i = next(r for r in range(lp.m) if a["Ap"][r + 1] - a["Ap"][r] >= 1 and
             a["Aj"][a["Ap"][r + 1] - 1] < lp.n - 1)
    q = a["Ap"][i + 1] - 1
    a["Aj"][q] = lp.n - 1 if a["Aj"][q] < lp.n - 1 else a["Aj"][q]
    expect(lp, a, E_CSR, "different matrices", layouts=("A", "AT"), on_device=on_device)


def test_bad_dimensions(lp):
    a = arrays(lp)
    with pytest.raises(cpd.CpdError) as ei:
        cpd.Problem(0, lp.n, AT=(a["ATp"], a["ATj"], a["ATx"]), b=a["b"][:0], c=a["c"])
    assert ei.value.code == E_DIM


def test_device_tensor_type_checks(lp):
    """The binding refuses device tensors it would otherwise reinterpret."""
    a = arrays(lp)
    dev = lambda v, dt=None: torch.as_tensor(np.ascontiguousarray(v)).cuda() if dt is None else \
        torch.as_tensor(np.ascontiguousarray(v)).to(dt).cuda()  # noqa: E731
    AT = (dev(a["ATp"]), dev(a["ATj"]), dev(a["ATx"]))
    vec = {k: dev(a[k]) for k in ("b", "c", "lb", "ub")}
    with pytest.raises(ValueError, match="dtype"):
        cpd.Problem(lp.m, lp.n, AT=(AT[0].to(torch.int64), AT[1], AT[2]), **vec)
    with pytest.raises(ValueError, match="dtype"):
        cpd.Problem(lp.m, lp.n, AT=AT, **{**vec, "c": vec["c"].float()})
    with pytest.raises(ValueError, match="contiguous"):
        cpd.Problem(lp.m, lp.n, AT=AT, **{**vec, "b": torch.stack([vec["b"], vec["b"]], 1)[:, 0]})
    P = cpd.Problem(lp.m, lp.n, AT=AT, **vec)
    S = cpd.Solver(P)
    with pytest.raises(ValueError, match="dtype"):
        S.set_iterate(x=torch.zeros(lp.n, dtype=torch.float32, device="cuda"))


def test_scale_and_senses_refused_while_solver_alive(lp):
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P)
    with pytest.raises(cpd.CpdError) as ei:
        P.scale()
    assert ei.value.code == E_STATE
    with pytest.raises(cpd.CpdError) as ei:
        P.set_senses(np.zeros(lp.m, np.int8))
    assert ei.value.code == E_STATE
    S.close()
    P.scale()                                  # allowed once the solver is gone
    P.set_senses(np.zeros(lp.m, np.int8))
    S2 = cpd.Solver(P, max_iters=10)
    S2.solve()

