"""The reference's own mt19937_64 stream on the device: with SF_FP64 the engine
reproduces the UNMODIFIED reference (golden vectors generated from
oracle/_ref/libsfref_mt.so, and the C restatement) bit for bit."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2308_10169_b200 as pe
from oracle_lib import (DEFAULT_GROUP_HYPERS, EVOLVED_PATH_HYPERS, RNG_MT, oracle, oracle_plan_frame,
                        oracle_run_dtpso, planner_cfg, ptr, world_from_engine)

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))


def test_init_and_step_draw_the_reference_stream(eng64mt):
    o = oracle()
    rng = np.random.default_rng(3)
    G, N, D = 3, 50, 7          # 2*R*D = 2100 words: crosses several 312-word blocks
    h = np.array([[1.5, 1.2, 0.8, 0.7, 0.3, 0.4]] * G)
    lo, hi = rng.uniform(-5, 0, D), rng.uniform(1, 5, D)
    x, v = eng64mt.init_swarm(h, lo, hi, G, N, D, 4242)
    xo, vo = np.zeros(G * N * D), np.zeros(G * N * D)
    assert o.or_init_swarm_seed(ptr(h), ptr(lo), ptr(hi), G, N, D, 4242, RNG_MT, None, 0, 0.0, ptr(xo), ptr(vo)) == 0
    assert np.array_equal(x, xo) and np.array_equal(v, vo)
    pbx, gbx, tbx = xo[::-1].copy(), rng.uniform(lo, hi, (G, D)).reshape(-1), rng.uniform(lo, hi)
    first = 2 * G * N * D + 5 * 3 * G * N          # stream position of step 6
    xg, vg = eng64mt.step(h, lo, hi, G, N, D, xo, vo, pbx, gbx, tbx, 4242, first, 6, 20)
    xs, vs = xo.copy(), vo.copy()
    o.or_step_seed(ptr(h), ptr(lo), ptr(hi), G, N, D, ptr(xs), ptr(vs), ptr(pbx), ptr(gbx), ptr(tbx), 4242, RNG_MT,
                   first, 6, 20)
    assert np.array_equal(xg, xs) and np.array_equal(vg, vs)


def test_fp64_frames_equal_the_unmodified_reference(eng64mt):
    """The first six frames of the acceptance scenario (root seed 3, cap 30,
    carryover), golden vectors produced by the reference itself."""
    o = oracle()
    w = pe.generate_world(pe.ScenarioConfig(), o.or_derive_seed(3, b"world"), "mt19937")
    cfg = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    prev, win = None, []
    for f, fr in enumerate(GOLD["plan_frames"]["mt"]):
        rec = eng64mt.plan_frame(w, prev, EVOLVED_PATH_HYPERS, cfg, fr["seed"], win)
        assert (rec.iterations, rec.truncated, rec.intersections) == (fr["iterations"], bool(fr["truncated"]), fr["q"])
        assert rec.fitness == fr["fitness"] and rec.length == fr["length"]
        assert pe.encode_path(rec.best_path).tolist() == fr["best"] and win == fr["window"]
        prev = rec.best_path
        w = pe.step_world(w, 1.0)


def test_fp64_scenario_100_frames_equals_reference_iterations(eng64mt):
    """run_scenario (simenv.hpp:239-276) through the C ABI, the whole published
    scenario: per-frame iteration counts equal the reference's (16.21 mean,
    91 truncated -- proj/test_output.txt:25-27)."""
    recs = eng64mt.run_scenario(pe.ScenarioConfig(root_seed=3), "sepso", 100,
                                pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True))
    s = GOLD["scenario_seed3"]
    assert [r.iterations for r in recs] == s["iterations"]
    assert sum(r.truncated for r in recs) == s["truncated"]
    assert abs(np.mean([r.length for r in recs]) - s["mean_length"]) < 1e-9


def test_fp32_scenario_statistics_match_reference(eng32mt):
    recs = eng32mt.run_scenario(pe.ScenarioConfig(root_seed=3), "sepso", 100,
                                pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True))
    s = GOLD["scenario_seed3"]
    assert abs(np.mean([r.iterations for r in recs]) - s["mean_iterations"]) < 1.5
    assert abs(np.mean([r.length for r in recs]) - s["mean_length"]) < 0.02 * s["mean_length"]
    assert sum(r.collision_free for r in recs) >= 90


def test_staged_mt_equals_fused_mt(eng64mt):
    o = oracle()
    w = pe.generate_world(pe.ScenarioConfig(), o.or_derive_seed(5, b"world"), "mt19937")
    cfg = pe.PlannerConfig(max_iters_per_frame=12)
    a = eng64mt.plan_frame(w, None, EVOLVED_PATH_HYPERS, cfg, 321)
    b = eng64mt.plan_frame_sharded(w, None, EVOLVED_PATH_HYPERS, cfg, 321)
    assert a.fitness == b.fitness and a.iterations == b.iterations and np.array_equal(a.best_path, b.best_path)


def test_run_dtpso_mt_equals_reference(eng64mt):
    for run_seed in (42, 7):
        r = eng64mt.run_dtpso("BF1", DEFAULT_GROUP_HYPERS, 8, 10, 100, run_seed, dim=30)
        st, tr, fp, ff, _ = oracle_run_dtpso(1, DEFAULT_GROUP_HYPERS, 8, 10, 100, run_seed, D=30,
                                             lo=np.full(30, -600.0), hi=np.full(30, 600.0), rng=RNG_MT)
        assert st == 0 and np.array_equal(r["trace"], tr) and np.array_equal(r["final_point"], fp)


def test_evolve_mt_equals_reference(eng64mt):
    o = oracle()
    r = eng64mt.evolve("BF1", (4, 5, 20), (2, 3, 3), 99, DEFAULT_GROUP_HYPERS[:2], dim=6)
    bt, rt, bh = np.zeros(3), np.zeros(3), np.zeros(24)
    lo, hi = np.full(6, -600.0), np.full(6, 600.0)
    assert o.or_evolve_flat(1, None, 6, ptr(lo), ptr(hi), 30.0, 4.0, 4, 5, 20, 2, 3, 3, 99,
                            ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS[:2])), RNG_MT, ptr(bt), ptr(rt),
                            ptr(bh)) == 0
    assert np.array_equal(r["best_lfv_trace"], bt) and np.array_equal(r["best"].reshape(-1), bh)


@pytest.mark.parametrize("G,N", [(40, 3), (33, 2)])
def test_run_dtpso_many_groups_equals_oracle(eng64mt, G, N):
    """More groups than lanes of a warp (the best update loops over groups)."""
    rng = np.random.default_rng(G)
    hyp = np.column_stack([rng.uniform(0.5, 2.5, (G, 3)), rng.uniform(0.6, 1.0, G), rng.uniform(0.1, 0.5, G),
                           rng.uniform(0.05, 0.5, G)])
    r = eng64mt.run_dtpso("BF3", hyp, G, N, 25, 5, dim=8)
    st, tr, fp, ff, _ = oracle_run_dtpso(3, hyp, G, N, 25, 5, D=8, lo=np.full(8, -600.0), hi=np.full(8, 600.0),
                                         rng=RNG_MT)
    assert st == 0 and np.allclose(r["trace"], tr, rtol=1e-12, atol=0) and np.allclose(r["final_point"], fp,
                                                                                       rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("per_group", [2048, 8192])
def test_parallel_stream_fill_equals_sequential(eng64mt, per_group):
    """Long init fills run as parallel segments from jumped generator states
    (mt_jump.cpp, stage_mt_fill_parallel): the same words and the same
    generator state afterwards (the step draws continue from it)."""
    o = oracle()
    w = pe.generate_world(pe.ScenarioConfig(), o.or_derive_seed(7, b"world"), "mt19937")
    cfg = pe.PlannerConfig(max_iters_per_frame=4, per_group=per_group, auto_truncate=False)
    os.environ["SEPSO_SEQ_FILL"] = "1"
    try:
        a = eng64mt.plan_frame_sharded(w, None, EVOLVED_PATH_HYPERS, cfg, 99)
    finally:
        del os.environ["SEPSO_SEQ_FILL"]
    b = eng64mt.plan_frame_sharded(w, None, EVOLVED_PATH_HYPERS, cfg, 99)
    assert a.iterations == b.iterations == 4
    assert a.fitness == b.fitness and np.array_equal(a.best_path, b.best_path)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_wide_parallel_fill_and_staged_bests_equal_sequential(prec, eng32mt, eng64mt):
    """A staged benchmark swarm whose init fill takes 128 jumped segments (2^27
    words: seven jump levels, exponent-list jumps): trace and final point
    equal the same run with the sequential fill.  (The staged bookkeeping --
    pbest copies deferred to the step -- is pinned against the reference by
    test_gpu_workloads' scale-harness test.)"""
    eng = eng32mt if prec == "fp32" else eng64mt
    G, N, D, T = 8, 8192, 1024, 3                 # 2 * 65,536 * 1,024 = 2^27 init words
    os.environ["SEPSO_SEQ_FILL"] = "1"
    try:
        a = eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, G, N, T, 21, dim=D)
    finally:
        del os.environ["SEPSO_SEQ_FILL"]
    b = eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, G, N, T, 21, dim=D)
    assert np.array_equal(a["trace"], b["trace"]) and np.array_equal(a["final_point"], b["final_point"])
    assert np.all(np.diff(b["trace"]) <= 0)       # tbest never worsens
