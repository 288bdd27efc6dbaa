"""Wall-clock phases of one end-to-end step (bench.py e2e): problem creation from pinned
host arrays, solver creation, phase 1, corner push, D2H of x, y, z, teardown.
CPD_TIMING=1 adds the library's creation-phase lines on stderr."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2511_13894_b200 as cpd  # noqa: E402


def main():
    lp = lpgen.config(sys.argv[1] if len(sys.argv) > 1 else "c5")
    pin = {}
    for k, a in (("ATp", lp.ATp), ("ATj", lp.ATj), ("ATx", lp.ATx), ("b", lp.b), ("c", lp.c), ("lb", lp.lb),
                 ("ub", lp.ub)):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        pin[k] = t.numpy()
    xo = torch.empty(lp.n, dtype=torch.float64, pin_memory=True).numpy()
    yo = torch.empty(lp.m, dtype=torch.float64, pin_memory=True).numpy()
    zo = torch.empty(lp.n, dtype=torch.float64, pin_memory=True).numpy()
    for rep in range(int(os.environ.get('REPS', '3'))):
        T = [time.perf_counter()]
        P = cpd.Problem(lp.m, lp.n, AT=(pin["ATp"], pin["ATj"], pin["ATx"]), b=pin["b"], c=pin["c"], lb=pin["lb"],
                        ub=pin["ub"])
        torch.cuda.synchronize(); T.append(time.perf_counter())
        S = cpd.Solver(P, max_iters=1024)
        torch.cuda.synchronize(); T.append(time.perf_counter())
        S.solve()
        T.append(time.perf_counter())
        S.corner_push(max_iters=1024, candidate_floor=100_000)
        T.append(time.perf_counter())
        cpd._check(cpd.lib().cpd_get_iterate(S.h, xo.ctypes.data, yo.ctypes.data, zo.ctypes.data, cpd.HOST))
        T.append(time.perf_counter())
        S.close()
        T.append(time.perf_counter())
        P.close()
        torch.cuda.synchronize(); T.append(time.perf_counter())
        names = ("create", "solver", "solve", "corner", "d2h", "solver close", "problem close")
        print(f"rep {rep}: " + " | ".join(f"{n} {1e3 * (T[i + 1] - T[i]):.0f} ms" for i, n in enumerate(names)),
              f" | cached {cpd.memcache_info(0) / 2**30:.1f} GiB", flush=True)


if __name__ == "__main__":
    main()
