"""The library's device-memory cache (csrc/devmem.cu, cpd_memcache_* in include/cpd.h).

A destroyed problem's buffers are kept for reuse; a re-created problem must produce
bit-identical iterates (the reused memory holds stale data from the previous problem,
so anything that read a buffer before writing it would show here), and release must
hand every idle byte back.
"""
import numpy as np
import pytest

import lpgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_13894_b200 as cpd  # noqa: E402


def _run(lp, **kw):
    P = cpd.Problem.from_lp(lp)
    S = cpd.Solver(P, max_iters=400, **kw)
    r = S.solve()
    x, y = S.get_iterate()
    S.close()
    P.close()
    return r, x, y


@pytest.mark.parametrize("name", ["c2-s", "c5-s"])
def test_reuse_is_bit_identical(name):
    lp = lpgen.config(name)
    cpd.memcache_release(0)
    assert cpd.memcache_info(0) == 0
    r0, x0, y0 = _run(lp)
    held = cpd.memcache_info(0)
    assert held > 0   # the destroyed problem's and solver's buffers are cached
    # a different problem in between scribbles over reused buffers
    _run(lpgen.config("c3-s"))
    r1, x1, y1 = _run(lp)
    assert r1["iterations"] == r0["iterations"] and r1["pobj"] == r0["pobj"]
    assert np.array_equal(x0, x1) and np.array_equal(y0, y1)
    cpd.memcache_release(0)
    assert cpd.memcache_info(0) == 0


def test_cache_bad_device():
    with pytest.raises(cpd.CpdError):
        cpd.memcache_info(10 ** 6)
    with pytest.raises(cpd.CpdError):
        cpd.memcache_release(-1)
