"""Short run of the hot path for ncu captures: `iters` lockstep iterations (eager
launches, restart check every iteration so every K1/K2 launch does work)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import lpgen  # noqa: E402
import paper_2511_13894_b200 as cpd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--check-every", type=int, default=1)
    ap.add_argument("--graph", type=int, default=0)
    a = ap.parse_args()
    t = time.time()
    lp = lpgen.config(a.config)
    print(f"gen {time.time() - t:.1f}s", flush=True)
    P = cpd.Problem.from_lp(lp)
    print(P.info(), flush=True)
    S = cpd.Solver(P, step_size=1e-3, check_every=a.check_every, use_graph=a.graph)
    S.step(a.iters)
    x, y = S.get_iterate()
    print("done", float(abs(x).sum()), flush=True)


if __name__ == "__main__":
    main()
