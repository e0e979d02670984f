"""Multi-GPU decomposition of one large swarm (BASELINE config 4), CPU only.

sf_plan_frame_sharded splits the groups of one swarm over ranks: each rank
owns groups [r*G/n, (r+1)*G/n), draws by GLOBAL row index, updates its groups'
bests locally, and the ranks exchange one population-best candidate per
iteration (all-gather), reduced in group order with the reference's strict
'<' (runner.hpp:88-91).  This test restates exactly that decomposition in
numpy on world_size-2 gloo processes (the all-gather is the real collective)
and checks that it reproduces the UNSHARDED oracle plan_frame bit for bit.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle_lib import (EVOLVED_PATH_HYPERS, RNG_PHILOX, WorldBuf, oracle, oracle_plan_frame,
                        planner_cfg, ptr, rect, u32p)

G, N, D, CAP, TW, DELTA = 8, 6, 6, 12, 4, 25.0


def make_world():
    return WorldBuf(100.0, 100.0, (50.0, 5.0), (50.0, 95.0),
                    [rect(20, 30, 45, 55), rect(55, 40, 80, 60), rect(35, 65, 60, 80), rect(10, 70, 25, 90)])


def u(o, seed, idx):
    return (o.or_philox_word(seed, int(idx)) >> 11) * 2.0 ** -53


def shard_plan(rank, nranks, seed, gather):
    """One rank's share of plan_frame, draws and updates as the device does."""
    o = oracle()
    w = make_world()
    hyp = EVOLVED_PATH_HYPERS
    R = G * N
    g0, g1 = rank * G // nranks, (rank + 1) * G // nranks
    rows = np.arange(g0 * N, g1 * N)
    lo = np.zeros(D)
    hi = np.array([w.head[0] if d < D // 2 else w.head[1] for d in range(D)])
    x = np.zeros((len(rows), D))
    v = np.zeros((len(rows), D))
    for i, r in enumerate(rows):            # swarm.hpp:94-132, global draw indices
        g = r // N
        for d in range(D):
            x[i, d] = lo[d] + u(o, seed, r * D + d) * (hi[d] - lo[d])
            vmax = hyp[g, 5] * (hi[d] - lo[d])
            v[i, d] = -vmax + u(o, seed, R * D + r * D + d) * (vmax - (-vmax))
    pbx, pbf = x.copy(), np.full(len(rows), np.inf)
    gbx, gbf = np.zeros((G, D)), np.full(G, np.inf)
    tbx, tbf, tbq = np.zeros(D), np.inf, 0
    pbq = np.zeros(len(rows), dtype=np.int64)
    gbq = np.zeros(G, dtype=np.int64)
    window = []
    cfg = planner_cfg(tw=TW, delta=DELTA, G=G, N=N, D=D, max_iters=CAP)
    for k in range(1, CAP + 1):
        f = np.zeros(len(rows))
        q = np.zeros(len(rows), dtype=np.uint32)
        o.or_eval_path_rows(ptr(np.ascontiguousarray(x)), len(rows), D, C.byref(w.struct()), 30.0, 4.0,
                            ptr(f), ptr(q, u32p))
        better = f < pbf                       # runner.hpp:73-80
        pbf[better], pbq[better] = f[better], q[better]
        pbx[better] = x[better]
        for g in range(g0, g1):                # runner.hpp:81-87, local groups
            sl = slice((g - g0) * N, (g - g0 + 1) * N)
            i = int(np.argmin(pbf[sl]))        # first index of the minimum
            if pbf[sl][i] < gbf[g]:
                gbf[g], gbq[g] = pbf[sl][i], pbq[sl][i]
                gbx[g] = pbx[sl][i]
        lg = g0 + int(np.argmin(gbf[g0:g1]))   # this rank's candidate
        cands = gather((float(gbf[lg]), int(gbq[lg]), lg, gbx[lg].tolist()))
        for cf, cq, cg, cx in sorted(cands, key=lambda c: c[2]):   # group order, strict '<'
            if cf < tbf:
                tbf, tbq, tbx = cf, cq, np.array(cx)
        window.append(tbf)                     # planner.hpp:179-187
        window = window[-TW:]
        a = np.array(window)
        if o.or_should_truncate(ptr(a), len(a), int(tbq == 0), C.byref(cfg)):
            return tbx, tbf, k, True
        if k == CAP:
            break
        base = 2 * R * D + (k - 1) * 3 * R     # swarm.hpp:59-70, 138-174
        frac = k / CAP
        for i, r in enumerate(rows):
            g = r // N
            h = hyp[g]
            w_ = h[3] - (h[3] - h[4]) * frac
            a1, a2, a3 = (h[j] * u(o, seed, base + j * R + r) for j in range(3))
            for d in range(D):
                vmax = h[5] * (hi[d] - lo[d])
                nv = w_ * v[i, d] + a1 * (pbx[i, d] - x[i, d]) + a2 * (gbx[g, d] - x[i, d]) + a3 * (tbx[d] - x[i, d])
                nv = -vmax if nv < -vmax else (vmax if vmax < nv else nv)
                v[i, d] = nv
                xn = x[i, d] + nv
                x[i, d] = lo[d] if xn < lo[d] else (hi[d] if hi[d] < xn else xn)
    return tbx, tbf, CAP, False


def _worker(rank, nranks, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)

    def gather(obj):
        out = [None] * nranks
        dist.all_gather_object(out, obj)
        return out

    res = shard_plan(rank, nranks, seed, gather)
    q.put((rank, res[0].tolist(), res[1], res[2], res[3]))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("seed", [11, 12345])
def test_group_sharded_plan_equals_unsharded_oracle(seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    st, rec, best, _, _ = oracle_plan_frame(make_world(), None, EVOLVED_PATH_HYPERS,
                                            planner_cfg(tw=TW, delta=DELTA, G=G, N=N, D=D, max_iters=CAP),
                                            seed, RNG_PHILOX)
    assert st == 0
    for rank, tbx, tbf, k, trunc in results:   # both ranks hold the identical record
        assert tbx == best.tolist() and tbf == rec.fitness
        assert k == rec.iterations and trunc == bool(rec.truncated)


def test_single_rank_restatement_equals_oracle():
    st, rec, best, _, _ = oracle_plan_frame(make_world(), None, EVOLVED_PATH_HYPERS,
                                            planner_cfg(tw=TW, delta=DELTA, G=G, N=N, D=D, max_iters=CAP),
                                            7, RNG_PHILOX)
    tbx, tbf, k, trunc = shard_plan(0, 1, 7, lambda c: [c])
    assert tbx.tolist() == best.tolist() and tbf == rec.fitness and k == rec.iterations
