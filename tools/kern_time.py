"""Per-kernel device time of the hot loop (CUDA events on the solver's stream,
profile=1) for one or more builds of libcpd — tuning experiments.

python tools/kern_time.py --config c5 --libs paper_2511_13894_b200/libcpd.so,/tmp/libcpd_x.so
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import lpgen  # noqa: E402
import paper_2511_13894_b200 as cpd  # noqa: E402
from paper_2511_13894_b200 import _build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--libs", default=_build.LIB)
    ap.add_argument("--iters", type=int, default=256)
    ap.add_argument("--corner", type=int, default=0)
    ap.add_argument("--method", type=int, default=0, help="0 R-PDHG, 1 reflected restarted Halpern")
    ap.add_argument("--noprof", action="store_true", help="no per-kernel events: wall it/s only")
    ap.add_argument("--env", default="", help="';'-separated variants of K=V,K=V env settings per run")
    a = ap.parse_args()
    t = time.time()
    lp = lpgen.config(a.config)
    print(f"gen {time.time() - t:.1f}s", flush=True)
    runs = [(p, e) for p in a.libs.split(",") for e in (a.env.split(";") if a.env else [""])]
    for path, env in runs:
        for kv in filter(None, env.split(",")):
            k, v = kv.split("=")
            os.environ[k] = v
        _build.LIB = path
        cpd._lib = None
        P = cpd.Problem.from_lp(lp)
        S = cpd.Solver(P, step_size=1e-3, profile=0 if a.noprof else 1, max_iters=a.iters, method=a.method)
        S.step(64)
        S.kernel_times(reset=True)
        t0 = time.time()
        S.step(a.iters)
        wall = time.time() - t0
        kt = S.kernel_times()
        line = [f"{os.path.basename(path)} [{env}]: {a.iters / wall:.1f} it/s wall"]
        for k, (ms, n) in kt.items():
            if n:
                b = S.kernel_bytes(k)
                line.append(f"{k} {ms / n:.3f} ms ({b / (ms / n) / 1e6:.0f} GB/s)")
        if a.corner:
            x, y = S.get_iterate()
            S.set_iterate(x, y)
            S.corner_push(max_iters=64, min_iters=10 ** 9)
            S.kernel_times(reset=True)
            S.set_iterate(x, y)
            S.corner_push(max_iters=a.iters, min_iters=10 ** 9)
            for k, (ms, n) in S.kernel_times().items():
                if n and "corner" in k:
                    b = S.kernel_bytes(k)
                    line.append(f"{k} {ms / n:.3f} ms ({b / (ms / n) / 1e6:.0f} GB/s)")
        print(" | ".join(line), flush=True)
        S.close()
        P.close()


if __name__ == "__main__":
    main()
