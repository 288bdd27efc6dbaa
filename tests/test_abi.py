"""The C-ABI library loads and exports every symbol include/cpd.h declares
(`-m "not gpu"`: no compute calls need a GPU here; without one they fail loudly)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2511_13894_b200 as cpd
from paper_2511_13894_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cpd.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cpd_[a-z_]+)\s*\(", src)))


def test_header_matches_binding_list():
    assert declared() == sorted(cpd.DECLARED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    path = _build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cpd_[a-z_]+)$", out, flags=re.M))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    L = cpd.lib()
    for s in declared():
        assert getattr(L, s) is not None


def test_built_for_sm100a():
    path = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_defaults_and_version():
    p = cpd.cpd_params_default()
    assert (p.eps_rel, p.eps_abs, p.check_every, p.step_scale, p.power_iters, p.restart) == \
        (1e-4, 1e-6, 64, 0.9, 128, 1)
    assert (p.beta_suff, p.beta_nec, p.beta_art, p.theta) == (0.2, 0.8, 0.36, 0.5)
    cp = cpd.cpd_corner_params_default()
    assert (cp.eps_abs, cp.obj_scale, cp.min_iters, cp.candidate_floor) == (1e-6, 1.0, 100, 100000)
    assert cpd.lib().cpd_version() == 1


def test_null_arguments_are_errors_not_crashes():
    L = cpd.lib()
    assert L.cpd_solve(None, None) == -1            # CPD_E_ARG
    assert b"NULL" in L.cpd_last_error()
    assert L.cpd_problem_destroy(None) == 0
    assert L.cpd_step(None, 1) == -1


def test_dimension_errors():
    L = cpd.lib()
    h = C.c_void_p()
    z = np.zeros(4)
    rc = L.cpd_problem_create(0, 1, 0, None, None, None, None, None, None, z.ctypes.data, z.ctypes.data,
                              None, None, 0, 0, C.byref(h))
    assert rc == -2   # CPD_E_DIM


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="GPU present")
def test_no_gpu_fails_loudly():
    """No CPU fallback: without a CUDA device the compute path reports CPD_E_CUDA."""
    import lpgen
    lp = lpgen.config("c1")
    with pytest.raises(cpd.CpdError) as e:
        cpd.Problem.from_lp(lp)
    assert e.value.code == -6


def test_corner_decide_host_only(golden):
    """cpd_corner_decide (host only, reading D-4) on the hand cases, without a GPU."""
    import oracle
    for c in golden("corner_examples.json")["decide"]["cases"]:
        assert cpd.corner_decide(c, c["m"]) == oracle.corner_decide(c, c["m"]) == (c["primal"], c["dual"])
    with pytest.raises(cpd.CpdError):
        cpd._check(cpd.lib().cpd_corner_decide(None, 1, None, None))


def test_params_defaults_halpern_fields():
    """cpd_params carries the NEXT-1 fields with their documented defaults (struct layout
    shared with include/cpd.h)."""
    p = cpd.cpd_params_default()
    assert (p.method, p.reflection, p.pid, p.kp, p.ki, p.kd) == (0, 1.0, 0, 0.99, 0.01, 0.0)
    assert (p.check_every, p.restart, p.use_graph) == (64, 1, 1)
