"""Parity of the CUDA engine against the CPU oracle (and the reference harness).

Everything here runs through the C ABI (libsepso_cuda.so) on a real GPU.  The
checker is oracle/liboracle.so (C restatement, pinned to the reference in
tests/test_oracle_cpu.py).  Bars (north star / SURVEY.md section 8):
  * FP64 engine: bit-exact on identical inputs, whole frames included.
  * FP32 engine: Q, argmin indices and truncation decisions exact on identical
    (FP32-representable) inputs; fitness/positions within REL = 1e-5 of the
    span-scaled value.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2308_10169_b200 as pe
from oracle_lib import (EVOLVED_PATH_HYPERS, DEFAULT_GROUP_HYPERS, PROB_PATH, RNG_PHILOX, ptr,
                        oracle, oracle_plan_frame, oracle_run_dtpso, planner_cfg, float_world,
                        world_from_engine, u32p, rect)

pytestmark = pytest.mark.gpu
REL = 1e-5   # FP32 tolerance stated by the north star


def rnd_hypers(rng, G):
    h = np.zeros((G, 6))
    h[:, 0:3] = rng.uniform(0, 2.5, (G, 3))
    h[:, 4] = rng.uniform(0.05, 0.5, G)
    h[:, 3] = h[:, 4] + rng.uniform(0, 0.4, G)
    h[:, 5] = rng.uniform(0.05, 1.0, G)
    return h


def paper_world(root=3):
    o = oracle()
    return pe.generate_world(pe.ScenarioConfig(), o.or_derive_seed(root, b"world"))


def oracle_eval(world, xs, D, alpha=30.0, beta=4.0):
    o = oracle()
    wb = world_from_engine(world)
    rows = xs.size // D
    f = np.zeros(rows)
    q = np.zeros(rows, dtype=np.uint32)
    o.or_eval_path_rows(ptr(np.ascontiguousarray(xs, dtype=np.float64)), rows, D,
                        C.byref(wb.struct()), alpha, beta, ptr(f), ptr(q, u32p))
    return f, q


# ------------------------------------------------------------------- stages
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("warm", [False, True])
def test_init_swarm_draws(prec, warm, eng32, eng64):
    eng = eng64 if prec == "fp64" else eng32
    rng = np.random.default_rng(1)
    G, N, D = 3, 7, 6
    hyp = rnd_hypers(rng, G)
    lo = rng.uniform(-5, 0, D)
    hi = lo + rng.uniform(1, 10, D)
    prev = (lo + hi) / 2 if warm else None
    x, v = eng.init_swarm(hyp, lo, hi, G, N, D, 777, prev=prev, warm=3, pi_radius=0.7)
    xo, vo = np.zeros(G * N * D), np.zeros(G * N * D)
    st = oracle().or_init_swarm_seed(ptr(hyp), ptr(lo), ptr(hi), G, N, D, 777, RNG_PHILOX,
                                     ptr(prev), 3 if warm else 0, 0.7, ptr(xo), ptr(vo))
    assert st == 0
    if prec == "fp64":
        assert np.array_equal(x, xo) and np.array_equal(v, vo)
    else:
        span = np.tile(hi - lo, G * N)
        assert np.all(np.abs(x - xo) <= REL * span)
        assert np.all(np.abs(v - vo) <= REL * span)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_step_matches_oracle(prec, eng32, eng64):
    eng = eng64 if prec == "fp64" else eng32
    rng = np.random.default_rng(2)
    for trial in range(6):
        G, N, D = rng.integers(1, 5), rng.integers(1, 9), rng.integers(1, 13)
        hyp = rnd_hypers(rng, G)
        lo = rng.uniform(-50, 0, D)
        hi = lo + rng.uniform(1, 100, D)
        E = G * N * D
        f32 = (lambda a: a.astype(np.float32).astype(np.float64)) if prec == "fp32" else (lambda a: a)
        x = f32(rng.uniform(np.tile(lo, G * N), np.tile(hi, G * N)))
        v = f32(rng.uniform(-1, 1, E) * np.tile(hi - lo, G * N) * 0.3)
        pbx = f32(rng.uniform(np.tile(lo, G * N), np.tile(hi, G * N)))
        gbx = f32(rng.uniform(np.tile(lo, G), np.tile(hi, G)))
        tbx = f32(rng.uniform(lo, hi))
        lo, hi = f32(lo), f32(hi)
        k, T = int(rng.integers(1, 30)), 30
        first = int(rng.integers(0, 1000))
        xg, vg = eng.step(hyp, lo, hi, G, N, D, x, v, pbx, gbx, tbx, 99, first, k, T)
        xo, vo = x.copy(), v.copy()
        oracle().or_step_seed(ptr(hyp), ptr(lo), ptr(hi), G, N, D, ptr(xo), ptr(vo), ptr(pbx),
                              ptr(gbx), ptr(tbx), 99, RNG_PHILOX, first, k, T)
        if prec == "fp64":
            assert np.array_equal(xg, xo) and np.array_equal(vg, vo)
        else:
            span = np.tile(hi - lo, G * N)
            assert np.all(np.abs(xg - xo) <= REL * span), trial
            assert np.all(np.abs(vg - vo) <= REL * span), trial


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_path_fitness_paper_scene(prec, eng32, eng64):
    eng = eng64 if prec == "fp64" else eng32
    rng = np.random.default_rng(3)
    for root in range(4):
        w = paper_world(root)
        if prec == "fp32":
            w = float_world(w)
        D = 16
        xs = rng.uniform(0, 366, (500, D))
        if prec == "fp32":
            xs = xs.astype(np.float32).astype(np.float64)
        f, q = eng.eval_path_rows(w, xs, D)
        fo, qo = oracle_eval(w, xs, D)
        assert np.array_equal(q, qo)
        if prec == "fp64":
            assert np.array_equal(f, fo)
        else:
            assert np.all(np.abs(f - fo) <= REL * np.maximum(1.0, np.abs(fo)))


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_path_q_integer_grid_adversarial(prec, eng32, eng64):
    """Touching / collinear / degenerate layouts (test_geometry.cpp:209-229,
    acceptance.cpp:412-434): Q equals the oracle on integer-grid worlds."""
    eng = eng64 if prec == "fp64" else eng32
    rng = np.random.default_rng(4)
    for trial in range(120):
        n_obs = 1 + trial % 4
        obs = []
        for _ in range(n_obs):
            x0, y0 = rng.integers(0, 34, 2)
            obs.append(rect(x0, y0, x0 + 1 + rng.integers(0, 6), y0 + 1 + rng.integers(0, 6)))
        w = pe.PolygonWorld(40, 40, rng.integers(0, 41, 2), rng.integers(0, 41, 2), obs)
        D = 2 * (1 + trial % 3)
        xs = rng.integers(0, 41, (64, D)).astype(np.float64)
        f, q = eng.eval_path_rows(w, xs, D)
        fo, qo = oracle_eval(w, xs, D)
        assert np.array_equal(q, qo), trial
        if prec == "fp64":
            assert np.array_equal(f, fo)
        else:
            assert np.all(np.abs(f - fo) <= REL * np.maximum(1.0, np.abs(fo)))


def test_fixture_q4(eng32, eng64):
    """test_geometry.cpp:158-171 / acceptance.cpp:436-446: Q = 4, fitness = len + 7680."""
    w = pe.PolygonWorld(10, 10, (0, 3), (0, 6), [rect(2, 2, 6, 6)])
    for eng in (eng32, eng64):
        f, q = eng.eval_path_rows(w, np.array([8.0, 0.0, 3.0, 5.0]), 4)
        assert q[0] == 4
        length = np.hypot(8, 0) + np.hypot(8, 2) + np.hypot(0, 1)
        assert abs(f[0] - (length + 7680.0)) <= 1e-9 * f[0] + (0 if eng is eng64 else 1e-3)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_update_bests_ties(prec, eng32, eng64):
    eng = eng64 if prec == "fp64" else eng32
    rng = np.random.default_rng(5)
    for trial in range(10):
        G, N, D = int(rng.integers(1, 5)), int(rng.integers(1, 40)), int(rng.integers(1, 6))
        R = G * N
        vals = np.array([1.0, 2.0, 3.0, 5.0])
        x = rng.integers(0, 9, R * D).astype(np.float64)
        pbx = rng.integers(0, 9, R * D).astype(np.float64)
        pbf = rng.choice(np.append(vals, np.inf), R)
        gbx = rng.integers(0, 9, G * D).astype(np.float64)
        gbf = rng.choice(np.append(vals, np.inf), G)
        tbx = rng.integers(0, 9, D).astype(np.float64)
        tbf = float(rng.choice(np.append(vals, np.inf)))
        fit = rng.choice(vals, R)      # many ties: incumbent must win
        got = eng.update_bests(G, N, D, x, pbx, pbf, gbx, gbf, tbx, tbf, fit)
        ref = [pbx.copy(), pbf.copy(), gbx.copy(), gbf.copy(), tbx.copy()]
        t = C.c_double(tbf)
        oracle().or_update_bests_arrays(G, N, D, ptr(x), ptr(ref[0]), ptr(ref[1]), ptr(ref[2]),
                                        ptr(ref[3]), ptr(ref[4]), C.byref(t), ptr(fit))
        for a, b in zip(got[:5], ref):
            assert np.array_equal(a, b), trial
        assert got[5] == t.value


# --------------------------------------------------------------- whole runs
def test_plan_frame_fp64_bit_exact_scenario(eng64):
    """Ten frames of the paper scenario (root seed 3, cap 30, carryover):
    FP64 engine == oracle on every record field, best path and window."""
    o = oracle()
    root = 3
    w = paper_world(root)
    cfg = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    ocfg = planner_cfg(max_iters=30, window_carryover=1)
    prev, win_g, win_o = None, [], []
    for f in range(10):
        seed = o.or_derive_seed_idx(root, b"plan", f)
        rec = eng64.plan_frame(w, prev, EVOLVED_PATH_HYPERS, cfg, seed, win_g)
        st, ro, bo, win_o, _ = oracle_plan_frame(world_from_engine(w), None if prev is None else pe.encode_path(prev),
                                                 EVOLVED_PATH_HYPERS, ocfg, seed, RNG_PHILOX, win_o)
        assert st == 0
        best = pe.encode_path(rec.best_path)
        assert rec.iterations == ro.iterations and rec.truncated == bool(ro.truncated), f
        assert rec.intersections == ro.intersections
        assert np.array_equal(best, bo), f
        assert rec.fitness == ro.fitness and rec.length == ro.length
        assert np.array_equal(np.array(win_g), win_o)
        prev = rec.best_path
        w = pe.step_world(w, 1.0)


def test_plan_frame_fp32_first_frame_tracks_oracle(eng32):
    """FP32 trajectories drift from FP64 chaotically; the first frame from a
    cold start must still reach a comparable, collision-free plan."""
    o = oracle()
    w = float_world(paper_world(3))
    cfg = pe.PlannerConfig(max_iters_per_frame=30)
    seed = o.or_derive_seed_idx(3, b"plan", 0)
    rec = eng32.plan_frame(w, None, EVOLVED_PATH_HYPERS, cfg, seed)
    st, ro, bo, _, _ = oracle_plan_frame(world_from_engine(w), None, EVOLVED_PATH_HYPERS,
                                         planner_cfg(max_iters=30), seed, RNG_PHILOX)
    assert rec.collision_free == bool(ro.collision_free)
    assert abs(rec.length - ro.length) <= 0.05 * ro.length
    # the record is self-consistent: fitness = length + alpha * Q^beta
    assert abs(rec.fitness - (rec.length + 30.0 * rec.intersections ** 4)) <= REL * rec.fitness
    f, q = oracle_eval(w, pe.encode_path(rec.best_path).astype(np.float64), 16)
    assert q[0] == rec.intersections


@pytest.mark.parametrize("kind", ["BF1", "BF2", "BF3", "BF4"])
def test_run_dtpso_fp64(kind, eng64):
    """Whole runs bit-exact (BF3 / BF4 through the glibc cos restatement)."""
    k = pe.engine.PROBLEMS[kind]
    for seed in (42, 7):
        r = eng64.run_dtpso(kind, DEFAULT_GROUP_HYPERS, 8, 10, 200, seed, dim=30)
        st, tr, fp, ff, _ = oracle_run_dtpso(k, DEFAULT_GROUP_HYPERS, 8, 10, 200, seed, D=30,
                                             lo=np.full(30, -600.0), hi=np.full(30, 600.0))
        assert st == 0
        assert np.array_equal(r["trace"], tr) and np.array_equal(r["final_point"], fp)


def test_batched_equals_single(eng64):
    o = oracle()
    worlds = [paper_world(r) for r in range(5)]
    cfg = pe.PlannerConfig(max_iters_per_frame=20)
    seeds = [o.or_derive_seed_idx(r, b"plan", 0) for r in range(5)]
    recs, best, stat = eng64.plan_frames_batched(worlds, None, None, EVOLVED_PATH_HYPERS, cfg, seeds)
    for i in range(5):
        r1 = eng64.plan_frame(worlds[i], None, EVOLVED_PATH_HYPERS, cfg, seeds[i])
        assert stat[i] == 0
        assert r1.fitness == recs[i].fitness and r1.iterations == recs[i].iterations
        assert np.array_equal(pe.encode_path(r1.best_path), best[i])


def test_lfv_batch_matches_oracle(eng64):
    o = oracle()
    rng = np.random.default_rng(6)
    cands = rng.uniform(-0.5, 3.0, (6, 48))
    seeds = [o.or_derive_seed_idx(11, b"lfv", i) for i in range(6)]
    got = eng64.lfv_batch("BF1", cands, seeds, 8, 10, 60, dim=30)
    lo, hi = np.full(30, -600.0), np.full(30, 600.0)
    for i in range(6):
        ref = o.or_lfv_flat(ptr(np.ascontiguousarray(cands[i])), 8, 1, None, 30, ptr(lo), ptr(hi),
                            30.0, 4.0, 8, 10, 60, seeds[i], RNG_PHILOX)
        assert got[i] == ref


def test_evolve_small_matches_oracle(eng64):
    o = oracle()
    r = eng64.evolve("BF1", (4, 5, 20), (2, 3, 3), 99, DEFAULT_GROUP_HYPERS[:2], dim=6)
    bt, rt, bh = np.zeros(3), np.zeros(3), np.zeros(24)
    lo, hi = np.full(6, -600.0), np.full(6, 600.0)
    st = o.or_evolve_flat(1, None, 6, ptr(lo), ptr(hi), 30.0, 4.0, 4, 5, 20, 2, 3, 3, 99,
                          ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS[:2])), RNG_PHILOX,
                          ptr(bt), ptr(rt), ptr(bh))
    assert st == 0
    assert np.array_equal(r["best_lfv_trace"], bt) and np.array_equal(r["evolution_lfv_trace"], rt)
    assert np.array_equal(r["best"].reshape(-1), bh)


def test_nonfinite_fitness_raises(eng64, eng32):
    """runner.hpp:56-61: first non-finite row names (g, n, k)."""
    for eng in (eng64, eng32):
        with pytest.raises(pe.NonFiniteFitnessError) as ei:
            eng.run_dtpso("BF1", DEFAULT_GROUP_HYPERS[:2], 2, 3, 5, 1, dim=4,
                          lo=np.full(4, -1e200), hi=np.full(4, 1e200))
        assert (ei.value.group, ei.value.index_in_group, ei.value.iteration) == (0, 0, 1)


def test_invalid_arguments_raise(eng32):
    w = paper_world(3)
    with pytest.raises(ValueError):
        eng32.plan_frame(w, None, EVOLVED_PATH_HYPERS, pe.PlannerConfig(tw=1), 1)
    with pytest.raises(ValueError):
        eng32.plan_frame(w, None, EVOLVED_PATH_HYPERS[:3], pe.PlannerConfig(), 1)
    with pytest.raises(ValueError):
        eng32.run_dtpso("BF1", DEFAULT_GROUP_HYPERS, 8, 10, 0, 1)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_general_polygons_q(prec, eng32, eng64):
    """Non-rectangular, concave and sliver polygons (the FP32 filtered paths:
    vertex-cross early exit, containment) agree with the oracle on Q."""
    eng = eng64 if prec == "fp64" else eng32
    rng = np.random.default_rng(9)
    for trial in range(40):
        polys = []
        for _ in range(int(rng.integers(1, 9))):
            cx, cy = rng.uniform(20, 180, 2)
            n = int(rng.integers(3, 9))
            ang = np.sort(rng.uniform(0, 2 * np.pi, n))
            rad = rng.uniform(3, 25, n) * (rng.uniform(0.2, 1.0, n) if trial % 2 else 1.0)
            poly = np.stack([cx + rad * np.cos(ang), cy + rad * np.sin(ang)], 1)
            if trial % 5 == 0:          # a near-degenerate sliver edge
                poly = np.vstack([poly, poly[-1] + 1e-4])
            polys.append(np.clip(poly, 0, 200))
        w = pe.PolygonWorld(200, 200, rng.uniform(0, 200, 2), rng.uniform(0, 200, 2), polys)
        if prec == "fp32":
            w = float_world(w)
        D = 2 * int(rng.integers(1, 9))
        xs = rng.uniform(0, 200, (256, D))
        if prec == "fp32":
            xs = xs.astype(np.float32).astype(np.float64)
        f, q = eng.eval_path_rows(w, xs, D)
        fo, qo = oracle_eval(w, xs, D)
        assert np.array_equal(q, qo), trial
