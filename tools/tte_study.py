"""Time to eps_rel = 1e-4 of the method variants on one config (one B200):
R-PDHG, R-PDHG + diagonal scaling, Halpern + PID (+ scaling).
python tools/tte_study.py --config c5 --cap 200000 --variants plain,scaled,halpern,halpern_scaled"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import paper_2511_13894_b200 as cpd  # noqa: E402

VARIANTS = {"plain": (False, {}), "scaled": (True, {}), "halpern": (False, dict(method=1, pid=1)),
            "halpern_scaled": (True, dict(method=1, pid=1)), "halpern_nopid_scaled": (True, dict(method=1, pid=0))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--cap", type=int, default=200000)
    ap.add_argument("--time-limit", type=float, default=600.0)
    ap.add_argument("--variants", default="plain,scaled,halpern,halpern_scaled")
    ap.add_argument("--corner", type=int, default=1)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    t = time.time()
    lp = lpgen.config(a.config)
    print(f"gen {time.time() - t:.1f}s", flush=True)
    res = {}
    for v in a.variants.split(","):
        scale, kw = VARIANTS[v]
        P = cpd.Problem.from_lp(lp)
        if scale:
            P.scale(10, 1)
        S = cpd.Solver(P, max_iters=a.cap, time_limit_s=a.time_limit, **kw)
        r = S.solve()
        e = {"status": cpd.STATUS[r["status"]], "iterations": r["iterations"], "seconds": r["wall_s"],
             "it_per_s": r["iterations"] / max(r["wall_s"], 1e-9), "score": r["score"], "pobj": r["pobj"],
             "restarts": r["restarts"]}
        if r["status"] == 0 and a.corner:
            rc, b, af = S.corner_push(max_iters=a.cap, time_limit_s=a.time_limit)
            e.update(corner_status=cpd.STATUS[rc["status"]], corner_iterations=rc["iterations"],
                     corner_seconds=rc["wall_s"], off_bound_before=b["off_bound"], off_bound_after=af["off_bound"])
        res[v] = e
        print(v, json.dumps(e), flush=True)
        S.close()
        P.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"config": a.config, "m": lp.m, "n": lp.n, "nnz": lp.nnz, "results": res}, f, indent=1)


if __name__ == "__main__":
    main()
