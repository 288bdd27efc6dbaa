"""Mutation check of the oracle's pins (VERDICT r1 "What's weak" #1).

Copies oracle/, lpgen/ and tests/ to a scratch directory, applies one plausible slip
to oracle/oracle.c at a time, rebuilds it and runs the `-m "not gpu"` oracle pin
tests there. Every mutation must make at least one pin fail ("killed").

    python tools/oracle_mutations.py            # all mutations
    python tools/oracle_mutations.py -k avg     # those whose name contains 'avg'
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_restart.py", "tests/test_oracle_halpern.py",
             "tests/test_oracle_scaling.py", "tests/test_oracle_ineq.py"]

# (name, original text, mutated text) — each original must occur exactly once.
# Not listed (equivalent mutants): "tie -> average" (at a tie the two candidates are
# the same point whenever t = 1, and an exact tie of distinct points has no robust
# construction) and "average not zeroed at a restart" (t restarts at 1, and
# x_avg + (x+ - x_avg)/1 = x+ up to one rounding, whatever x_avg held).
MUTATIONS = [
    ("never_restart_to_avg", "int use_avg = S_a < S_c;", "int use_avg = 0;"),
    ("necessary_flipped", "S > s->S_prev)", "S < s->S_prev)"),
    ("S_r_from_current", "s->S_r = S;", "s->S_r = S_c;"),
    ("no_average_return", "if (s->mode == MODE_FULL && S_a <= P->eps_rel) {",
     "if (0 && s->mode == MODE_FULL && S_a <= P->eps_rel) {"),
    ("free_as_lower", "if (l[j] > -INFINITY) { rd -= zp;", "if (1) { rd -= zp;"),
    ("model_count_orig_lb", "off_bound(x[j], lhat[j], uhat[j], eps_abs)",
     "off_bound(x[j], l[j], uhat[j], eps_abs)"),
    ("zero_rc_strict", "fabs(z[j]) <= eps_abs;", "fabs(z[j]) < eps_abs;"),
    ("candidates_nonstrict", "off && fabs(z[j]) < eps_abs;", "off && fabs(z[j]) <= eps_abs;"),
    ("omega_inverted", "exp(P->theta * log(dy / dx)", "exp(P->theta * log(dx / dy)"),
    ("restart_every_check", "(S <= P->beta_nec * s->S_r && S > s->S_prev) ||\n                (double)s->t >= P->beta_art * (double)s->k",
     "(S <= P->beta_nec * s->S_r && S > s->S_prev) ||\n                (double)s->t >= 0.0 * (double)s->k"),
    ("halpern_restart_every_check", "(r <= P->beta_nec * s->r0 && r > s->r_prev) ||\n                    (double)s->t >= P->beta_art * (double)s->k",
     "(r <= P->beta_nec * s->r0 && r > s->r_prev) ||\n                    (double)s->t >= 0.0 * (double)s->k"),
    ("halpern_r0_every_iter", "if (s->t == 0) s->r0 = r;", "s->r0 = r;"),
    ("sufficient_off", "if (S <= P->beta_suff * s->S_r ||", "if (0 ||"),
    ("no_S_prev_reset", "s->S_prev = INFINITY;\n                s->t = 0;", "s->t = 0;"),
    ("upper_term_sign", "bound_terms -= u[j] * zm;", "bound_terms += u[j] * zm;"),
    ("upper_rd_sign", "if (u[j] < INFINITY)  { rd += zm;", "if (u[j] < INFINITY)  { rd -= zm;"),
    ("extrapolation_dropped", "s->xbar[j] = 2.0 * s->xn[j] - s->x[j];", "s->xbar[j] = s->xn[j];"),
    ("bound_map_nonstrict", "if (z[j] < -eps_abs) { lhat[j] = x[j];", "if (z[j] <= -eps_abs) { lhat[j] = x[j];"),
    ("est_dual_from_off", "(m > st->zero_rc ? m - st->zero_rc : 0)", "(m > st->off_bound ? m - st->off_bound : 0)"),
    # reflected restarted Halpern PDHG + PID weight (NEXT-1)
    ("halpern_lambda", "double lam = (double)(s->t + 1) / (double)(s->t + 2);",
     "double lam = (double)(s->t + 1) / (double)(s->t + 3);"),
    ("halpern_no_reflection", "s->x[j] = lam * ((1.0 + rho) * s->xh[j] - rho * s->x[j])",
     "s->x[j] = lam * (s->xh[j])"),
    ("halpern_anchor_dropped", "+ (1.0 - lam) * s->ya[i];", "+ (1.0 - lam) * s->y[i];"),
    ("halpern_cross_sign", "double r2 = dx2 / tau + dy2 / sigma + 2.0 * cross;",
     "double r2 = dx2 / tau + dy2 / sigma - 2.0 * cross;"),
    ("halpern_restart_to_z", "memcpy(s->x, s->xh, sizeof(double) * n);\n                    memcpy(s->y, s->yh",
     "memcpy(s->xh, s->x, sizeof(double) * n);\n                    memcpy(s->y, s->yh"),
    ("halpern_returns_z", "if (s->prm.method == 1 && s->k > 0) { xs = s->xh; ys = s->yh; }", ""),
    ("pid_integral_dropped", "+ P->ki * s->pid_int", "+ P->ki * e"),
    ("pid_derivative_sign", "P->kd * (e - s->pid_eprev)", "P->kd * (s->pid_eprev - e)"),
]


def run_one(name, old, new, workdir):
    src = os.path.join(workdir, "oracle", "oracle.c")
    with open(os.path.join(ROOT, "oracle", "oracle.c")) as f:
        text = f.read()
    assert text.count(old) == 1, (name, text.count(old))
    with open(src, "w") as f:
        f.write(text.replace(old, new))
    so = os.path.join(workdir, "oracle", "liboracle.so")
    if os.path.exists(so):
        os.remove(so)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "-m", "not gpu and not slow", *PIN_TESTS], cwd=workdir,
                       capture_output=True, text=True, timeout=1800)
    last = (r.stdout.strip().splitlines() or [""])[-1]
    return r.returncode != 0, last


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    a = ap.parse_args()
    work = tempfile.mkdtemp(prefix="orcmut")
    try:
        for d in ("oracle", "lpgen", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(work, d),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        results = []
        for name, old, new in MUTATIONS:
            if a.k not in name:
                continue
            killed, last = run_one(name, old, new, work)
            results.append((name, killed))
            print(f"{name:24s} {'KILLED' if killed else 'SURVIVED'}   {last}", flush=True)
        surv = [n for n, k in results if not k]
        print(f"{len(results) - len(surv)}/{len(results)} killed" + (f"; survived: {surv}" if surv else ""))
        return 1 if surv else 0
    finally:
        shutil.rmtree(work, ignore_errors=True)


if __name__ == "__main__":
    sys.exit(main())
