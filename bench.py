#!/usr/bin/env python
"""bench.py — PDHG iterations/s and achieved HBM GB/s (fp64) of the R-PDHG +
corner-push hot path (BASELINE.json metric) on B200.

One STEP = one pass of the whole hot path over the
workload: reset the iterate to 0, cpd_solve (power iteration for the step size,
norms, phase-1 R-PDHG with restart checks, capped at --iters1 iterations or
eps_rel = 1e-4), cpd_corner_push (Algorithm 1 setup, steering iterations with the
P:391-395 stop capped at --iters2, statistics before/after).  `value` = PDHG
iterations (both phases) per second of device time over K timed steps, inputs
resident in HBM.  `e2e` = the same metric through the public C-ABI with the LP in
pinned HOST memory: every step creates the problem from host arrays (H2D,
device validation and transpose), solves, corner-pushes and reads x, y, z back.

Workload: BASELINE.json config 5 (largest synthetic LP: m=4e6, n=2e7, nnz=2.4e8,
Zipf(1.2) rows; fits one B200), seeded, generated on the host (lpgen).  The
oracle (CPU, single thread) is timed on a bounded sample for `cpu_baseline`, and
is the `--impl reference` arm (this tier has no reference implementation).

Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under torchrun.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line: everything else any library prints on file
# descriptor 1 (NCCL's version banner, ...) is sent to stderr, and the JSON line is
# written to the saved original stdout
_JSON_FD = os.dup(1)
os.dup2(2, 1)


def emit(res):
    os.write(_JSON_FD, (json.dumps(res) + "\n").encode())

METRIC = "PDHG iterations/sec and achieved HBM GB/s (fp64) at 1/2/4/8 B200; time to eps=1e-4"
UNIT = "iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--iters1", type=int, default=1024, help="phase-1 iteration cap per step")
    ap.add_argument("--iters2", type=int, default=1024, help="corner-phase iteration cap per step")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tte", default="c2,c3,c4,c5", help="configs for the time-to-eps side measurement ('' = off)")
    ap.add_argument("--ref-iters", type=int, default=0, help="oracle iterations per reference step (0: auto)")
    ap.add_argument("--partition", type=int, default=-1,
                    help="multi-GPU partition: 0 row-block, 1 col-block, -1 auto (shard the long side)")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the distributed (split) path even with one rank (checks the N>1 code path)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- helpers
def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(config, kernel):
    """dram read+write bytes per launch of `kernel` from the committed ncu summary
    (tools/ncu_traffic.py), or (None, why) when the summary was captured on other
    library sources than the ones benchmarked (its source_hash differs)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        from paper_2511_13894_b200 import _build
        have, want = d[config].get("source_hash"), _build.source_hash()
        if have != want:
            return None, f"stale: ncu summary of sources {have}, benchmarked sources {want}"
        if kernel not in d[config] and kernel == "dual_step_A:corner":
            kernel = "dual_step_A"   # the dual step is the same pass in both phases
        return d[config][kernel]["dram_bytes_per_launch"], f"ncu --set full capture of sources {want}"
    except Exception as e:
        return None, f"unavailable ({type(e).__name__})"


def dist_init(n):
    if n <= 1 and int(os.environ.get("WORLD_SIZE", "1")) <= 1:
        return 0, 1, 0
    import torch.distributed as dist
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    dist.init_process_group(backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_step(S, iters1, iters2):
    """One pass of the hot path on a resident problem. Returns PDHG iterations done."""
    S.set_iterate(None, None)
    r1 = S.solve()
    r2, before, after = S.corner_push(max_iters=iters2, candidate_floor=100_000)
    return r1["iterations"] + r2["iterations"], r1, r2, before, after


# ----------------------------------------------------------------- reference arm
def reference_arm(args, lp, rank, world):
    """The oracle (single-threaded C, fp64) timed on a bounded sample of the same
    workload: each step runs `it` phase-1 iterations from x = 0, y = 0 (termination
    tests on, exactly as the oracle stands; eta from its power iteration is computed
    once, untimed, since it is per-problem setup)."""
    import oracle
    if rank != 0:
        return None
    olp = oracle.OracleLP(lp)
    eta = 0.9 / oracle.power_sigma(olp, 8, 7) if lp.nnz > 5e7 else 0.9 / oracle.power_sigma(olp)
    it = args.ref_iters or (3 if lp.nnz > 5e7 else 200)
    times, iters = [], 0
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = oracle.Run(olp, oracle.default_params(step_size=eta, max_iters=it))
        r.run(it)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            iters += r.k
    total = sum(times)
    v = iters / total
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {**workload_config(args, lp, world),
                                         "parallelism": f"CPU oracle, single thread (rank 0 of {world})"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{it} phase-1 iterations from x=0,y=0 per step on {lp.name} (full size)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def workload_config(args, lp, world, part=None):
    return {"workload": f"{lp.name}: BASELINE.json config 5 (m={lp.m}, n={lp.n}, nnz={lp.nnz}, Zipf(1.2) rows)"
            if lp.name == "c5" else f"{lp.name} (m={lp.m}, n={lp.n}, nnz={lp.nnz})",
            "m": lp.m, "n": lp.n, "nnz": lp.nnz, "seed": lp.meta.get("seed"),
            "step": f"set_iterate(0) + cpd_solve(max_iters={args.iters1}, eps_rel=1e-4) + "
                    f"cpd_corner_push(max_iters={args.iters2})",
            "l2": "inputs larger than L2 (matrix 5.9 GB vs 126 MB L2)" if lp.nnz > 1e7 else "no flush",
            "parallelism": (f"{part} x{world}" if part else "1 GPU")}


def host_cpu():
    """nproc and the CPU model name of the host the oracle runs on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


# oracle iterations timed per config for its ms/iteration (bounded: ~10-15 s in all)
_ORC_SAMPLE = {"c1": 2000, "c2": 100, "c3": 4, "c4": 6, "c5": 2}


def cpu_baseline(lp, tte=("c1", "c2")):
    """The oracle as it stands (single-threaded C, fp64) on this host: ms per phase-1
    iteration (termination tests on, from x = 0) on C1-C5, and its time to eps_rel =
    1e-4 from x = 0 (power iteration for eta included) on the configs it finishes in
    seconds.  `value` = its it/s on the benchmarked workload (lp)."""
    import lpgen
    import oracle
    per = {}
    main_v, main_sample = None, None
    for nm, it in _ORC_SAMPLE.items():
        L = lp if nm == lp.name else lpgen.config(nm)
        olp = oracle.OracleLP(L)
        eta = 0.9 / oracle.power_sigma(olp, 4, 7)
        t0 = time.perf_counter()
        r = oracle.Run(olp, oracle.default_params(step_size=eta, max_iters=it))
        r.run(it)
        dt = time.perf_counter() - t0
        per[nm] = {"ms_per_iter": 1e3 * dt / max(r.k, 1), "iterations": r.k, "seconds": dt}
        if nm == lp.name:
            main_v = r.k / dt
            main_sample = (f"{r.k} phase-1 R-PDHG iterations (termination tests on) from x=0 on {lp.name} "
                           f"full size, {dt:.1f} s, single thread")
        del olp
    tt = {}
    for nm in tte:
        L = lpgen.config(nm)
        olp = oracle.OracleLP(L)
        t0 = time.perf_counter()
        x, y, r = oracle.solve(olp, oracle.default_params())
        tt[nm] = {"status": oracle.STATUS[r["status"]], "iterations": r["iterations"],
                  "seconds": time.perf_counter() - t0}
    return {"value": main_v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": main_sample,
            "host": host_cpu(), "ms_per_iter": per, "time_to_eps": tt,
            "note": "oracle time to eps on C3 (3,266 its at ~0.16 s) / C4 / C5 exceeds the bench's minutes: "
                    "see profiles/r02_oracle_tte.json"}


# phase-1 iteration cap of the time-to-eps runs; C5 runs only its fastest variant
# (Halpern + PID + diagonal scaling, ~61k iterations, ~2 min on one B200) under a time
# limit, reported as "not reached after N iterations" with its score if it stops short
_TTE_CAP = {"c5": 200000}
_TTE_TLIM = {"c5": 300.0}
_TTE_VARIANTS = {"": (False, {}), ":scaled": (True, {}), ":halpern": (False, dict(method=1, pid=1)),
                 ":halpern_scaled": (True, dict(method=1, pid=1))}
_TTE_ONLY = {"c5": (":halpern_scaled",)}


def time_to_eps(names, device, lp_cache=None):
    """Wall time from cpd_solve entry to return at eps_rel = 1e-4 (problem resident),
    plain R-PDHG and with the diagonal preconditioning (cpd_problem_scale, NEXT-1),
    then Algorithm 1 from the phase-1 point with the P:391-395 stop: the Fig. 4 analogue
    (steering / phase-1 iteration ratio) and the Fig. 1 analogue (off-bound
    count before / after and its trajectory every 64 iterations)."""
    import lpgen
    import paper_2511_13894_b200 as cpd
    out = {}
    for nm in names:
        lp = (lp_cache or {}).get(nm) or lpgen.config(nm)
        cap = _TTE_CAP.get(nm, 200000)
        for tag in _TTE_ONLY.get(nm, tuple(_TTE_VARIANTS)):
            scale, kw = _TTE_VARIANTS[tag]
            P = cpd.Problem.from_lp(lp, device=device)
            if scale:
                P.scale(10, 1)
            S = cpd.Solver(P, max_iters=cap, time_limit_s=_TTE_TLIM.get(nm, 0.0), **kw)
            if nm not in _TTE_CAP:
                S.solve()   # warm-up (graph capture)
                S.set_iterate(None, None)
            r = S.solve()
            e = {"status": cpd.STATUS[r["status"]], "iterations": r["iterations"],
                 "seconds": r["wall_s"], "it_per_s": r["iterations"] / r["wall_s"],
                 "pobj": r["pobj"], "score": r["score"],
                 "method": "Halpern+PID" if kw else "R-PDHG", "scaled": scale}
            if r["status"] != 0:
                e["note"] = f"eps_rel=1e-4 not reached after {r['iterations']} iterations (score {r['score']:.3g})"
            elif nm in _TTE_CAP:
                pass   # (C5: phase 1 only, the corner phase would double the minutes)
            else:
                rc, before, after = S.corner_push(max_iters=200000)   # Algorithm 1 from the phase-1 point
                k, off, _ = S.trajectory()
                e.update({"corner_status": cpd.STATUS[rc["status"]], "corner_iterations": rc["iterations"],
                          "corner_seconds": rc["wall_s"],
                          "corner_over_phase1": rc["iterations"] / max(r["iterations"], 1),
                          "off_bound_before": before["off_bound"], "off_bound_after": after["off_bound"],
                          "off_bound_model_after": after["off_bound_model"], "m": lp.m,
                          "fix_lb": before["fix_lb"], "fix_ub": before["fix_ub"],
                          "candidates": before["candidates"], "is_candidate": before["is_candidate"],
                          "trajectory_off_bound": [int(v) for v in off[:: max(1, len(off) // 16)]]})
            out[nm + tag] = e
            S.close()
            P.close()
    return out


def self_launch(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: start N ranks with torchrun on this
    node (127.0.0.1) and exit with its status; rank 0's JSON line goes to our stdout."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, stdout=_JSON_FD)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank, world, local = dist_init(args.gpus)
    import lpgen
    lp = lpgen.config(args.config)
    if args.impl == "reference":
        res = reference_arm(args, lp, rank, world)
        if rank == 0:
            emit(res)
        return
    import torch
    import paper_2511_13894_b200 as cpd
    dev = local
    torch.cuda.set_device(dev)
    uid = None
    dist_path = world > 1 or args.force_dist
    if world > 1:
        import torch.distributed as dist
        obj = [cpd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    elif dist_path:
        uid = cpd.nccl_unique_id()
    # resident problem (a0: validation + transpose + plans happen here, untimed)
    if dist_path:
        P = cpd.Problem.create_dist(lp, rank, world, uid, partition=args.partition, device=dev)
    else:
        P = cpd.Problem.from_lp(lp, device=dev)
    S = cpd.Solver(P, max_iters=args.iters1, profile=1)
    P_info = P.dist_info()
    plan = P.plan_info()
    for _ in range(args.warmup):
        run_step(S, args.iters1, args.iters2)
    S.kernel_times(reset=True)
    c0 = S.counters()["launches"]
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    last = None
    with ClockSampler(dev) as clk:
        ev0.record()
        for _ in range(args.steps):
            n_it, r1, r2, before, after = run_step(S, args.iters1, args.iters2)
            iters += n_it
            last = (r1, r2, before, after)
        ev1.record()
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    launches = S.counters()["launches"] - c0
    value = iters / (ms / 1e3)
    kt = S.kernel_times()
    # dominant kernel (largest share of device time in the timed region)
    dom = max((k for k in kt if kt[k][1] > 0), key=lambda k: kt[k][0])
    dom_ms = kt[dom][0] / kt[dom][1]
    dom_bytes = S.kernel_bytes(dom)
    peak, peak_kind = measured_peak()
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    # model bytes per PDHG iteration (K1 + K2) -> whole-path GB/s
    b_it1 = S.kernel_bytes("primal_step_AT") + S.kernel_bytes("dual_step_A")
    b_it2 = S.kernel_bytes("primal_step_AT:corner") + S.kernel_bytes("dual_step_A:corner")
    r1, r2, before, after = last
    it1, it2 = r1["iterations"], r2["iterations"]
    hbm_gbs = value * (it1 * b_it1 + it2 * b_it2) / max(it1 + it2, 1) / 1e9
    kernel_share = {k: round(v[0] / ms, 4) for k, v in kt.items() if v[1] > 0}
    traffic, traffic_src = ncu_traffic(args.config, dom)
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded lpgen, BASELINE.json config recipe)",
        "config": workload_config(args, lp, world,
                                  {0: "row-block", 1: "col-block"}.get(P_info["partition"]) if dist_path else None),
        "hbm_gbs_model": hbm_gbs,
        "iterations_per_step": {"phase1": it1, "corner": it2},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": dom, "kernel_ms": dom_ms, "algorithmic_bytes_per_launch": dom_bytes,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                     "whole_path_gbs": hbm_gbs, "whole_path_frac": hbm_gbs / peak,
                     "whole_path_frac_of_8tbs": hbm_gbs / 8000.0,
                     "pair": pair_roofline(S, kt, peak)},
        "kernel_time_share": kernel_share,
        "plan": {k: int(plan[k]) for k in ("warp", "heavy_rows", "long_pieces", "hot_rows", "fused_rows", "fused_nnz")},
        "gpu_launches": launches,
        "corner_stats": {"before": before, "after": after},
    }
    with_e2e = not args.no_e2e
    S.close()
    P.close()
    if with_e2e:
        res["e2e"] = e2e_measure(args, lp, dev, rank, world, dist_path)
    clk_s = clk.summary()
    res["clocks"] = clk_s
    if dist_path:
        res["partition"] = {0: "row-block", 1: "col-block"}[P_info["partition"]]
    if args.tte and world == 1:
        try:
            res["time_to_eps"] = time_to_eps([x for x in args.tte.split(",") if x], dev, {lp.name: lp})
        except Exception as e:  # pragma: no cover
            res["time_to_eps"] = {"error": str(e)}
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        res["cpu_baseline"] = cpu_baseline(lp)
    if rank == 0:
        emit(res)


def pair_roofline(S, kt, peak):
    """Primal + dual step as one unit (K1 + K2 of one PDHG iteration, phase 1): hot-row
    fusion moves part of the A x+ product into K1's stream, so the pair's algorithmic bytes
    over its summed CUDA-event time is the figure that no work shifting between the two
    kernels can move."""
    ks = ("primal_step_AT", "dual_step_A")
    if not all(k in kt and kt[k][1] > 0 for k in ks):
        return None
    ms = sum(kt[k][0] / kt[k][1] for k in ks)
    b = sum(S.kernel_bytes(k) for k in ks)
    return {"kernels": list(ks), "ms": ms, "algorithmic_bytes": b, "achieved": b / (ms / 1e3) / 1e9,
            "frac": b / (ms / 1e3) / 1e9 / peak}


def e2e_measure(args, lp, dev, rank=0, world=1, dist_path=False):
    """Public API with HOST buffers: H2D of the LP from pinned memory, problem
    creation (device validation + transpose), solve + corner push, D2H of x, y, z.
    N > 1: every rank creates its block from the same host arrays (collective)."""
    import torch
    import paper_2511_13894_b200 as cpd
    pin = {}
    for k, a in (("ATp", lp.ATp), ("ATj", lp.ATj), ("ATx", lp.ATx), ("b", lp.b), ("c", lp.c),
                 ("lb", lp.lb), ("ub", lp.ub)):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        pin[k] = t.numpy()
    h2d = sum(a.nbytes for a in pin.values())
    xo = torch.empty(lp.n, dtype=torch.float64, pin_memory=True).numpy()
    yo = torch.empty(lp.m, dtype=torch.float64, pin_memory=True).numpy()
    zo = torch.empty(lp.n, dtype=torch.float64, pin_memory=True).numpy()
    d2h = xo.nbytes + yo.nbytes + zo.nbytes
    steps = args.e2e_steps or max(1, min(args.steps, 2))

    if world > 1:
        import torch.distributed as dist

    def one():
        if dist_path:
            obj = [cpd.nccl_unique_id() if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0)
            import types
            hl = types.SimpleNamespace(m=lp.m, n=lp.n, ATp=pin["ATp"], ATj=pin["ATj"], ATx=pin["ATx"], b=pin["b"],
                                       c=pin["c"], lb=pin["lb"], ub=pin["ub"])
            P = cpd.Problem.create_dist(hl, rank, world, obj[0], partition=args.partition, device=dev)
        else:
            P = cpd.Problem(lp.m, lp.n, AT=(pin["ATp"], pin["ATj"], pin["ATx"]), b=pin["b"], c=pin["c"],
                            lb=pin["lb"], ub=pin["ub"], device=dev)
        S = cpd.Solver(P, max_iters=args.iters1)
        r1 = S.solve()
        r2, _, _ = S.corner_push(max_iters=args.iters2, candidate_floor=100_000)
        import ctypes as C
        cpd._check(cpd.lib().cpd_get_iterate(S.h, xo.ctypes.data, yo.ctypes.data, zo.ctypes.data, cpd.HOST))
        S.close()
        P.close()
        return r1["iterations"] + r2["iterations"]

    one()   # warm-up
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    iters = sum(one() for _ in range(steps))
    ev1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world)
    return {"value": iters / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps, "ms_per_step": ms / steps}


if __name__ == "__main__":
    main()
