"""Generate tests/golden/*.json from the REFERENCE (oracle/_ref, compiled
unmodified from /root/reference/proj/include by oracle/Makefile).

Run in the build container (the only place /root/reference exists):
    make -C oracle all && python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/) and, through it, the CUDA engine.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import (DEFAULT_GROUP_HYPERS, EVOLVED_PATH_HYPERS, PlanRecord, WorldBuf,  # noqa: E402
                        generate_world, planner_cfg, ptr, rect, ref, ref_plan_frame, u32p, szp)


def main():
    mt, ph = ref("mt"), ref("philox")
    assert mt is not None and ph is not None, "build oracle/_ref first (make -C oracle ref)"
    out = {}
    # ---- rng.hpp
    rng = {}
    for kind, lib in (("mt", mt), ("philox", ph)):
        rng[kind] = {}
        for seed in (0, 1, 42, 987654321, 2**63 + 12345):
            a = np.zeros(8)
            lib.ref_uniform_stream(C.c_uint64(seed), 8, ptr(a))
            rng[kind][str(seed)] = a.tolist()
    rng["derive_seed"] = [[r, t, mt.ref_derive_seed(r, t.encode())] for r in (0, 1, 3, 99)
                          for t in ("world", "plan", "outer", "lfv")]
    rng["derive_seed_idx"] = [[r, t, i, mt.ref_derive_seed_idx(r, t.encode(), i)]
                              for r in (1, 3) for t in ("plan", "lfv") for i in (0, 1, 7, 99)]
    out["rng"] = rng
    # ---- geometry.hpp
    corpus = [((0, 0), (1, 1), (0, 1), (1, 0)), ((0, 0), (1, 0), (0, 1), (1, 1)),
              ((0, 0), (2, 0), (1, 0), (3, 0)), ((0, 0), (1, 0), (2, 0), (3, 0)),
              ((0, 0), (1, 0), (1, 0), (2, 5)), ((0, 0), (3, 0), (1, 0), (2, 0)),
              ((0, 0), (4, 0), (2, 0), (2, 3)), ((0, 0), (4, 4), (2, 2), (2, 2)),
              ((0, 0), (4, 4), (5, 5), (5, 5)), ((0, 0), (0, 0), (0, 0), (0, 0)),
              ((0, 0), (0, 4), (0, 4), (0, 8)), ((0, 0), (4, 0), (4, 0), (8, 0)),
              ((0, 0), (2, 2), (2, 2), (4, 0)), ((0, 0), (1, 1), (2, 2), (3, 3)),
              ((0, 0), (10, 0), (5, -3), (5, 3)), ((0, 0), (10, 10), (0, 1), (10, 11))]
    g = np.random.default_rng(8008)
    for _ in range(300):
        r = [3, 12, 60][_ % 3]
        corpus.append(tuple(tuple(int(v) for v in g.integers(-r, r + 1, 2)) for _ in range(4)))
    seg = []
    for a1, a2, b1, b2 in corpus:
        arr = [np.array(p, dtype=np.float64) for p in (a1, a2, b1, b2)]
        seg.append([list(a1), list(a2), list(b1), list(b2),
                    int(mt.ref_segments_intersect(*(ptr(x) for x in arr)))])
    out["segments"] = seg
    square = np.array([0, 0, 4, 0, 4, 4, 0, 4], dtype=np.float64)
    concave = np.array([0, 0, 6, 0, 6, 6, 3, 3, 0, 6], dtype=np.float64)
    inside = []
    for poly, n, pts in ((square, 4, [(2, 2), (5, 2), (2, 0), (0, 0), (4, 2)]),
                         (concave, 5, [(1, 1), (3, 5), (3, 3), (5, 1)])):
        for p in pts:
            pa = np.array(p, dtype=np.float64)
            inside.append([poly.tolist(), list(p), int(mt.ref_point_strictly_inside(ptr(pa), ptr(poly), n))])
    out["inside"] = inside
    # random integer-grid worlds: Q, fitness, length (test_geometry.cpp:209-229)
    worlds = []
    for trial in range(60):
        obs = []
        for _ in range(1 + trial % 4):
            x0, y0 = g.integers(0, 34, 2)
            obs.append(rect(float(x0), float(y0), float(x0 + 1 + g.integers(0, 6)), float(y0 + 1 + g.integers(0, 6))))
        start, target = g.integers(0, 41, 2).astype(float), g.integers(0, 41, 2).astype(float)
        w = WorldBuf(40.0, 40.0, start, target, obs)
        D = 2 * (1 + trial % 3)
        xs = g.integers(0, 41, (8, D)).astype(np.float64)
        f, q, l = np.zeros(8), np.zeros(8, dtype=np.uint32), np.zeros(8)
        mt.ref_eval_path_rows(C.byref(w.struct()), ptr(xs), 8, D, 30.0, 4.0, ptr(f), ptr(q, u32p), ptr(l))
        worlds.append(dict(start=start.tolist(), target=target.tolist(), obstacles=[list(map(list, o)) for o in obs],
                           D=D, xs=xs.tolist(), fitness=f.tolist(), q=q.tolist(), length=l.tolist()))
    out["grid_worlds"] = worlds
    # paper-scene random paths (real-valued)
    pw = generate_world("mt", mt.ref_derive_seed(3, b"world"))
    xs = g.uniform(0, 366, (64, 16))
    f, q, l = np.zeros(64), np.zeros(64, dtype=np.uint32), np.zeros(64)
    mt.ref_eval_path_rows(C.byref(pw.struct()), ptr(xs), 64, 16, 30.0, 4.0, ptr(f), ptr(q, u32p), ptr(l))
    out["paper_paths"] = dict(head=pw.head.tolist(), offsets=pw.offsets.tolist(), verts=pw.verts.tolist(),
                              vel=pw.vel.tolist(), xs=xs.tolist(), fitness=f.tolist(), q=q.tolist(),
                              length=l.tolist())
    # ---- benchmarks.hpp
    bench = []
    for kind in (1, 2, 3, 4):
        for D in (1, 3, 8, 30):
            xs = g.uniform(-600, 600, (4, D))
            xs[0] = 0.5
            f = np.zeros(4)
            assert mt.ref_bench_eval(kind, ptr(xs), 4, D, ptr(f)) == 0
            bench.append(dict(kind=kind, D=D, xs=xs.tolist(), f=f.tolist()))
    out["bench"] = bench
    # ---- simenv.hpp: worlds and 20 steps (both streams)
    sim = {}
    for kind in ("mt", "philox"):
        lib = mt if kind == "mt" else ph
        w = generate_world(kind, lib.ref_derive_seed(3, b"world"))
        steps = []
        for _ in range(20):
            lib.ref_step_world(ptr(w.head), w.n, ptr(w.offsets, u32p), ptr(w.verts), ptr(w.vel), 1.0)
        steps = dict(head=w.head.tolist(), verts=w.verts.tolist(), vel=w.vel.tolist())
        w0 = generate_world(kind, lib.ref_derive_seed(3, b"world"))
        sim[kind] = dict(world=dict(head=w0.head.tolist(), verts=w0.verts.tolist(), vel=w0.vel.tolist(),
                                    offsets=w0.offsets.tolist()), after20=steps)
    out["simenv"] = sim
    # ---- planner.hpp: the first 6 frames of the acceptance scenario (seed 3)
    plan = {}
    for kind in ("mt", "philox"):
        lib = mt if kind == "mt" else ph
        w = generate_world(kind, lib.ref_derive_seed(3, b"world"))
        cfg = planner_cfg(max_iters=30, window_carryover=1)
        prev, win, frames = None, [], []
        for f in range(6):
            seed = lib.ref_derive_seed_idx(3, b"plan", f)
            st, rec, best, win, _ = ref_plan_frame(kind, w, prev, EVOLVED_PATH_HYPERS, cfg, seed, win)
            assert st == 0
            frames.append(dict(seed=seed, fitness=rec.fitness, length=rec.length, q=rec.intersections,
                               iterations=rec.iterations, truncated=rec.truncated, best=best.tolist(),
                               window=win.tolist()))
            prev = best
            lib.ref_step_world(ptr(w.head), w.n, ptr(w.offsets, u32p), ptr(w.verts), ptr(w.vel), 1.0)
        plan[kind] = frames
    out["plan_frames"] = plan
    # published-scenario statistics (proj/test_output.txt:25-27), mt stream
    recs = (PlanRecord * 100)()
    assert mt.ref_run_scenario(3, 0, 100, C.byref(planner_cfg(max_iters=30, window_carryover=1)), recs, None) == 0
    its = [recs[i].iterations for i in range(100)]
    out["scenario_seed3"] = dict(mean_iterations=float(np.mean(its)), iterations=its,
                                 truncated=sum(recs[i].truncated for i in range(100)),
                                 colliding_truncations=sum(1 for i in range(100) if recs[i].truncated and recs[i].intersections),
                                 mean_length=float(np.mean([recs[i].length for i in range(100)])))
    # ---- runner.hpp: run_dtpso on BF1..BF4 (philox stream)
    runs = []
    for kind in (1, 2, 3, 4):
        trace, fp, ff = np.zeros(60), np.zeros(30), C.c_double(0)
        bad = (C.c_size_t * 3)()
        assert ph.ref_run_dtpso(kind, None, 30, 30.0, 4.0, ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS)), 8, 10, 60,
                                42, ptr(trace), ptr(fp), C.byref(ff), bad) == 0
        runs.append(dict(kind=kind, G=8, N=10, T=60, seed=42, trace=trace.tolist(), final_point=fp.tolist(),
                         final_fitness=ff.value))
    out["run_dtpso_philox"] = runs
    # ---- hsef.hpp: unflatten repair + a small evolution (philox)
    raw = np.array([9.0, -3.0, 0.1, 2.0, -0.5, 7.0, 1.0, 1.0, 1.0, 0.2, 0.7, 0.5, 1.0, 1.0, 1.0, 0.02, 0.8, 0.5])
    h = np.zeros(18)
    mt.ref_unflatten(ptr(raw), 3, ptr(h))
    lo, hi = np.full(6, -600.0), np.full(6, 600.0)
    bt, rt, bh = np.zeros(3), np.zeros(3), np.zeros(24)
    assert ph.ref_evolve(1, None, 6, 30.0, 4.0, 4, 5, 20, 2, 3, 3, 99,
                         ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS[:2])), ptr(bt), ptr(rt), ptr(bh)) == 0
    out["hsef"] = dict(raw=raw.tolist(), unflatten=h.tolist(),
                       evolve=dict(kind=1, D=6, inner=[4, 5, 20], outer=[2, 3, 3], seed=99,
                                   best_trace=bt.tolist(), round_trace=rt.tolist(), best=bh.tolist()))
    with open(os.path.join(HERE, "reference_vectors.json"), "w") as f:
        json.dump(out, f)
    print("wrote", os.path.join(HERE, "reference_vectors.json"))


if __name__ == "__main__":
    main()
