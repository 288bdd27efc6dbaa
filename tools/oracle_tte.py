"""Time to eps_rel = 1e-4 of the CPU oracle (single thread, as it stands) on the configs
it finishes within minutes; writes a JSON record with the host it ran on.
python tools/oracle_tte.py --configs c1,c2,c3 --out profiles/r02_oracle_tte.json"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lpgen  # noqa: E402
import oracle  # noqa: E402


def host():
    model = None
    with open("/proc/cpuinfo") as f:
        for ln in f:
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    return {"nproc": os.cpu_count(), "model": model}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3")
    ap.add_argument("--methods", default="rpdhg,halpern")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = {"host": host(), "threads": 1, "results": {}}
    for nm in a.configs.split(","):
        lp = lpgen.config(nm)
        olp = oracle.OracleLP(lp)
        for meth in a.methods.split(","):
            kw = dict(method=1, pid=1) if meth == "halpern" else {}
            t0 = time.perf_counter()
            x, y, r = oracle.solve(olp, oracle.default_params(**kw))
            dt = time.perf_counter() - t0
            res["results"][f"{nm}:{meth}"] = {"status": oracle.STATUS[r["status"]], "iterations": r["iterations"],
                                              "seconds": dt, "ms_per_iter": 1e3 * dt / max(r["iterations"], 1),
                                              "pobj": r["pobj"]}
            print(nm, meth, json.dumps(res["results"][f"{nm}:{meth}"]), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
