import os, sys
os.environ.update({"CPD_HEAVY_MIN": "4096", "CPD_SLAB_COLS": "8192", "CPD_WARP": "1", "CPD_SHORT": "1"})
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"]
import lpgen, paper_2511_13894_b200 as cpd
lp = lpgen.config("c5-s")
for h in sys.argv[1:]:
    os.environ["CPD_HOTD"] = h
    P = cpd.Problem.from_lp(lp)
    print(h, P.plan_info(), flush=True)
    S = cpd.Solver(P, restart=1)
    try:
        S.step(1); S.step(100); print("ok", flush=True)
    except Exception as e:
        print("ERR", e, flush=True)
