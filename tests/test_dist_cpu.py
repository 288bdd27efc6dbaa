"""Multi-GPU host logic on CPU (world_size 2, gloo) — `-m "not gpu"`.

The library's partition (cpd_partition) and layout (cpd_dist_layout, the same
host function cpd_problem_create_dist uses) decide which block of A each rank keeps
and which slice of the exchanged vector it owns.  Here
two gloo processes take those blocks and run the distributed R-PDHG iteration's
algebra with the exchanges the CUDA path makes (reduce-scatter of the partial
product, all-gather of the updated slice, allreduce of scalars) in numpy, and the
result must equal the oracle's single-process iterates.  gloo has no
reduce-scatter, so it is expressed as allreduce + own slice (same sums).
"""
import math
import os

import numpy as np
import pytest

import lpgen
import oracle
import paper_2511_13894_b200 as cpd

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

WORLD = 2
ITERS = 60


def _dense_blocks(lp):
    A = lp.dense_A()
    return A


def _worker(rank, world, port, name, part, eta, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lp = lpgen.config(name)
        m, n = lp.m, lp.n
        bnd = cpd.partition(m, n, lp.ATp, lp.ATj, world, part)
        # every rank computes the same partition
        allb = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, torch.as_tensor(bnd))
        assert all(np.array_equal(b.numpy(), bnd) for b in allb)
        A = lp.dense_A()
        l, u = lp.lb, lp.ub

        def allreduce(v):
            t = torch.as_tensor(np.atleast_1d(np.asarray(v, dtype=np.float64))).clone()
            dist.all_reduce(t)
            return t.numpy()

        def reduce_scatter(full, L):   # gloo: allreduce, then the owned slice
            pad = np.zeros(world * L)
            pad[:full.size] = full
            tot = allreduce(pad)
            return tot[rank * L:(rank + 1) * L]

        def all_gather(sl, L, N):
            t = torch.zeros(L, dtype=torch.float64)
            t[:sl.size] = torch.as_tensor(sl)
            out = [torch.zeros(L, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(out, t)
            return torch.cat(out).numpy()[:N]

        # the library's own layout arithmetic (cpd_dist_layout = what create_dist uses)
        lay = [cpd.dist_layout(m, n, lp.ATp, lp.ATj, world, part, qq) for qq in range(world)]
        me = lay[rank]
        assert me["partition"] == part and me["split"] == (1 if part == 0 else 0)
        b0, b1 = me["block_begin"], me["block_end"]
        assert (b0, b1) == (int(bnd[rank]), int(bnd[rank + 1]))
        L = me["L"]
        if part == 1:   # col-block: columns [b0, b1); m-side slices
            s0 = me["gofs_m"]
            s1 = s0 + me["own_len_m"]
            assert me["own_len_n"] == b1 - b0 and me["gofs_n"] == b0 and me["poff_m"] == s0 and me["poff_n"] == 0
            assert me["local_rows_AT"] == b1 - b0
            Ap = A[:, b0:b1]
            nb2 = allreduce(np.dot(lp.b[s0:s1], lp.b[s0:s1]))[0]
            nc2 = allreduce(np.dot(lp.c[b0:b1], lp.c[b0:b1]))[0]
            om = math.sqrt(nc2) / math.sqrt(nb2)
            tau, sig = eta / om, eta * om
            x = np.zeros(b1 - b0)
            y = np.zeros(m)            # replica
            ys = np.zeros(s1 - s0)     # owned slice
            for _ in range(ITERS):
                xp = np.minimum(np.maximum(x - tau * (lp.c[b0:b1] - Ap.T @ y), l[b0:b1]), u[b0:b1])
                axb = reduce_scatter(Ap @ (2 * xp - x), L)[:s1 - s0]   # A(2x+ - x), summed over ranks
                ys = ys + sig * (lp.b[s0:s1] - axb)
                y = all_gather(ys, L, m)
                x = xp
            Lc = max(d["own_len_n"] for d in lay)
            xf = all_gather(np.pad(x, (0, Lc - x.size)), Lc, None)
            xfull = np.concatenate([xf[qq * Lc:qq * Lc + lay[qq]["own_len_n"]] for qq in range(world)])
            yfull = y
        else:           # row-block: rows [b0, b1); n-side slices
            s0 = me["gofs_n"]
            s1 = s0 + me["own_len_n"]
            assert me["own_len_m"] == b1 - b0 and me["gofs_m"] == b0 and me["poff_n"] == s0 and me["poff_m"] == 0
            assert me["local_rows_AT"] == n
            Ap = A[b0:b1, :]
            nb2 = allreduce(np.dot(lp.b[b0:b1], lp.b[b0:b1]))[0]
            nc2 = allreduce(np.dot(lp.c[s0:s1], lp.c[s0:s1]))[0]
            om = math.sqrt(nc2) / math.sqrt(nb2)
            tau, sig = eta / om, eta * om
            xs = np.zeros(s1 - s0)    # owned slice
            x = np.zeros(n)           # replica
            y = np.zeros(b1 - b0)
            for _ in range(ITERS):
                g = reduce_scatter(Ap.T @ y, L)[:s1 - s0]
                xsp = np.minimum(np.maximum(xs - tau * (lp.c[s0:s1] - g), l[s0:s1]), u[s0:s1])
                xp = all_gather(xsp, L, n)
                y = y + sig * (lp.b[b0:b1] - Ap @ (2 * xp - x))
                x, xs = xp, xsp
            xfull = x
            Lr = max(d["own_len_m"] for d in lay)
            yf = all_gather(np.pad(y, (0, Lr - y.size)), Lr, None)
            yfull = np.concatenate([yf[qq * Lr:qq * Lr + lay[qq]["own_len_m"]] for qq in range(world)])
        # the slices of the split side tile it exactly, in rank order
        side = "n" if part == 0 else "m"
        ends = [(d[f"gofs_{side}"], d[f"gofs_{side}"] + d[f"own_len_{side}"]) for d in lay]
        assert ends[0][0] == 0 and ends[-1][1] == (n if part == 0 else m)
        assert all(ends[i][1] == ends[i + 1][0] for i in range(world - 1))
        if rank == 0:
            q.put((xfull, yfull))
    finally:
        dist.destroy_process_group()


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("part", [0, 1])
@pytest.mark.parametrize("name", ["c1", "c2-s"])
def test_sharded_iteration_matches_oracle(name, part):
    """Two gloo ranks, each with the block and owned slice cpd_dist_layout assigns,
    reproduce the oracle's single-process iterates (1e-9)."""
    lp = lpgen.config(name)
    olp = oracle.OracleLP(lp)
    eta = 0.9 / oracle.power_sigma(olp)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, name, part, eta, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    xg, yg = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    R = oracle.Run(olp, oracle.default_params(step_size=eta, restart=0), mode=oracle.MODE_NONE)
    R.run(ITERS)
    xo, yo = R.get()
    assert np.linalg.norm(xg - xo) <= 1e-9 * np.linalg.norm(xo)
    assert np.linalg.norm(yg - yo) <= 1e-9 * np.linalg.norm(yo)


@pytest.mark.parametrize("part", [0, 1])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_blocks(world, part):
    """Contiguous, non-empty, covering, and nnz-balanced to within one row's weight."""
    lp = lpgen.config("c5-s")
    bnd = cpd.partition(lp.m, lp.n, lp.ATp, lp.ATj, world, part)
    R = lp.n if part == 1 else lp.m
    assert bnd[0] == 0 and bnd[-1] == R and np.all(np.diff(bnd) >= 1)
    if part == 1:
        w = np.diff(lp.ATp.astype(np.int64)) + 1
    else:
        w = np.bincount(lp.ATj, minlength=lp.m) + 1
    pre = np.concatenate([[0], np.cumsum(w)])
    loads = pre[bnd[1:]] - pre[bnd[:-1]]
    assert loads.max() <= pre[-1] / world + w.max() + 1


@pytest.mark.parametrize("part", [0, 1, -1])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_dist_layout_tiles(world, part):
    """Every rank's owned slices / blocks tile both sides exactly (no gap, no overlap),
    slices are ceil(rows / world) long except at the end, offsets match the blocks."""
    lp = lpgen.config("c5-s")
    lay = [cpd.dist_layout(lp.m, lp.n, lp.ATp, lp.ATj, world, part, r) for r in range(world)]
    pt = lay[0]["partition"]
    assert pt == (part if part >= 0 else (1 if lp.n >= lp.m else 0))
    for side, N in (("m", lp.m), ("n", lp.n)):
        o = 0
        for d in lay:
            assert d[f"gofs_{side}"] == o
            o += d[f"own_len_{side}"]
        assert o == N
    split = lay[0]["split"]
    sp = "n" if split == 1 else "m"
    N = lp.n if split == 1 else lp.m
    assert all(d["L"] == -(-N // world) for d in lay)
    assert all(d[f"own_len_{sp}"] == max(0, min(d["L"], N - r * d["L"])) for r, d in enumerate(lay))
    assert all(d[f"poff_{sp}"] == d[f"gofs_{sp}"] for d in lay)
    bnd = cpd.partition(lp.m, lp.n, lp.ATp, lp.ATj, world, pt)
    assert [d["block_begin"] for d in lay] == list(bnd[:-1])


def test_partition_rejects_too_many_ranks():
    lp = lpgen.config("c1")
    with pytest.raises(cpd.CpdError):
        cpd.partition(lp.m, lp.n, lp.ATp, lp.ATj, lp.m + 1, 0)
