"""Parity of every workload bench.py reports, in the precision it reports it.

Checkers: the UNMODIFIED reference (oracle/_ref/libsfref_mt.so, the reference's
own mt19937_64 stream) for FP64 bit-exactness and for the FP32 statistics;
numpy for Ackley (an extension the reference does not have).
  * config 1 -- BenchmarkProblem::evaluate_rows (benchmarks.hpp:45-88) row by
    row; whole run_dtpso traces (runner.hpp:97-129) on BF1-BF4; FP32 trial
    statistics of the benchmarked 8 x 10 x 1400 runs.
  * config 3 -- lfv_fitness / evolve (hsef.hpp:108-171) on the PATH problem
    with the inner budget the reference's CLI uses (8 x 170 x 30,
    proj/tools/swarmforge.cpp:270-278).
  * run_scenario variants (simenv.hpp:188-234): sepso-noat, sepso-nopi,
    dtpso, dppso, pso (G = 1, N = 1360) frame by frame.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2308_10169_b200 as pe
from oracle_lib import (DEFAULT_GROUP_HYPERS, EVOLVED_PATH_HYPERS, PROB_PATH, PlanRecord, oracle,
                        planner_cfg, ptr, ref, world_from_engine)

pytestmark = pytest.mark.gpu
REL = 1e-5   # FP32 tolerance stated by the north star
BF = {"BF1": 1, "BF2": 2, "BF3": 3, "BF4": 4}


def _ref():
    r = ref("mt")
    if r is None:
        pytest.skip("oracle/_ref/libsfref_mt.so not built")
    return r


def ref_bench(kind, xs, D):
    out = np.zeros(xs.shape[0])
    assert _ref().ref_bench_eval(kind, ptr(np.ascontiguousarray(xs)), xs.shape[0], D, ptr(out)) == 0
    return out


def ref_dtpso(kind, G, N, T, seed, D=30):
    trace, fp, ff = np.zeros(T), np.zeros(D), C.c_double(0)
    bad = (C.c_size_t * 3)()
    st = _ref().ref_run_dtpso(kind, None, D, 30.0, 4.0, ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS[:G])),
                              G, N, T, seed, ptr(trace), ptr(fp), C.byref(ff), bad)
    assert st == 0
    return trace, fp, ff.value


def bench_rows(rng, n, D):
    """Rows over the benchmark box [-600, 600] plus near-optimum and integer rows
    (cos arguments at exact multiples of pi/2 after the 2*pi product)."""
    xs = rng.uniform(-600, 600, (n, D))
    xs[: n // 4] = rng.uniform(-5.12, 5.12, (n // 4, D))
    xs[n // 4: n // 3] = rng.integers(-600, 601, (n // 3 - n // 4, D))
    xs[-1] = 0.0
    return xs


# ------------------------------------------------------------ config 1 rows
@pytest.mark.parametrize("name", ["BF1", "BF2", "BF3", "BF4"])
def test_eval_bench_rows_fp64_bit_exact(name, eng64mt):
    """sf_eval_bench_rows == the reference's evaluate_rows bit for bit (BF3/BF4
    through the glibc cos restatement, cos_glibc.cuh)."""
    rng = np.random.default_rng(11)
    for D in (30, 7, 1):
        xs = bench_rows(rng, 4000, D)
        got = eng64mt.eval_bench_rows(name, xs, D)
        assert np.array_equal(got, ref_bench(BF[name], xs, D)), D


@pytest.mark.parametrize("name", ["BF1", "BF2", "BF3", "BF4"])
def test_eval_bench_rows_fp32(name, eng32mt):
    """FP32 engine on FP32-representable rows: within REL of the reference's
    FP64 value (relative to max(1, |f|) and to the sum of |terms|, the scale
    the FP32 rounding errors are relative to)."""
    rng = np.random.default_rng(12)
    D = 30
    xs = bench_rows(rng, 4000, D).astype(np.float32).astype(np.float64)
    got = eng32mt.eval_bench_rows(name, xs, D)
    want = ref_bench(BF[name], xs, D)
    scale = {"BF1": np.sum(xs * xs, 1),
             "BF2": np.sum(100 * (xs[:, 1:] - xs[:, :-1] ** 2) ** 2 + (1 - xs[:, :-1]) ** 2, 1),
             "BF3": np.sum(xs * xs + 20.0, 1),
             "BF4": 1.0 + np.sum(xs * xs, 1) / 4000 + 1.0}[name]
    assert np.all(np.abs(got - want) <= REL * np.maximum(1.0, scale))


def ackley_np(xs):
    D = xs.shape[1]
    s1 = np.sum(xs * xs, 1)
    s2 = np.sum(np.cos(2 * np.pi * xs), 1)
    return -20.0 * np.exp(-0.2 * np.sqrt(s1 / D)) - np.exp(s2 / D) + 20.0 + np.e


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_ackley_formula(prec, eng64mt, eng32mt):
    """Ackley (BASELINE config 1; not in the reference): the standard formula
    -20 exp(-0.2 sqrt(sum x^2 / D)) - exp(sum cos(2 pi x) / D) + 20 + e."""
    eng = eng64mt if prec == "fp64" else eng32mt
    rng = np.random.default_rng(13)
    xs = bench_rows(rng, 2000, 30)
    if prec == "fp32":
        xs = xs.astype(np.float32).astype(np.float64)
    got = eng.eval_bench_rows("ACKLEY", xs, 30)
    want = ackley_np(xs)
    tol = 1e-12 if prec == "fp64" else 2e-5
    assert np.all(np.abs(got - want) <= tol * np.maximum(1.0, np.abs(want)))
    assert abs(got[-1]) <= (1e-12 if prec == "fp64" else 1e-5)       # the minimum f(0) = 0


# ----------------------------------------------------------- config 1 runs
@pytest.mark.parametrize("name", ["BF1", "BF2", "BF3", "BF4"])
def test_run_dtpso_fp64_full_trace_equals_reference(name, eng64mt):
    """Whole run_dtpso runs, benchmark seeds (acceptance.cpp:175): every trace
    entry and the final point equal the unmodified reference's."""
    o = oracle()
    for t in range(2):
        seed = o.or_derive_seed_idx(3003, f"bench-{name}".encode(), t)
        r = eng64mt.run_dtpso(name, DEFAULT_GROUP_HYPERS, 8, 10, 1400, seed, dim=30)
        tr, fp, ff = ref_dtpso(BF[name], 8, 10, 1400, seed)
        assert np.array_equal(r["trace"], tr), (name, t, int(np.argmax(r["trace"] != tr)))
        assert np.array_equal(r["final_point"], fp) and r["final_fitness"] == ff


def test_run_dtpso_batched_fp64_equals_reference(eng64mt):
    """The batched launch the config-1 bench times: per-trial results equal the
    reference's run_dtpso on each seed."""
    o = oracle()
    seeds = [o.or_derive_seed_idx(3003, b"bench-BF3", t) for t in range(6)]
    traces, fps, ffs, stat = eng64mt.run_dtpso_batched("BF3", DEFAULT_GROUP_HYPERS, 8, 10, 400, seeds)
    for i, s in enumerate(seeds):
        tr, fp, ff = ref_dtpso(3, 8, 10, 400, s)
        assert stat[i] == 0
        assert np.array_equal(traces[i], tr) and np.array_equal(fps[i], fp) and ffs[i] == ff


@pytest.mark.parametrize("name", ["BF3", "BF4"])
def test_config1_fp32_trial_statistics(name, eng32mt):
    """The FP32 engine's trials (the config-1 bench line) against the reference's
    FP64 trials on the same 64 seeds: FP32 trajectories fork chaotically, so the
    final-fitness distributions are compared (median within 25 %, two-sided
    Mann-Whitney U p > 0.01)."""
    from concurrent.futures import ThreadPoolExecutor
    from scipy.stats import mannwhitneyu
    o = oracle()
    seeds = [o.or_derive_seed_idx(3003, f"bench-{name}".encode(), t) for t in range(64)]
    _, _, f32, stat = eng32mt.run_dtpso_batched(name, DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds)
    assert np.all(stat == 0)
    with ThreadPoolExecutor(8) as ex:
        f64 = np.array(list(ex.map(lambda s: ref_dtpso(BF[name], 8, 10, 1400, s)[2], seeds)))
    m32, m64 = np.median(f32), np.median(f64)
    assert abs(m32 - m64) <= 0.25 * m64, (m32, m64)
    assert mannwhitneyu(f32, f64).pvalue > 0.01
    assert np.all(f32 >= 0.0)


# ------------------------------------------------------- config 3 (path HSEF)
def path_world():
    o = oracle()
    return pe.generate_world(pe.ScenarioConfig(root_seed=41), o.or_derive_seed(41, b"world"), "mt19937")


def ref_lfv_path(cand, world, seed, iG=8, iN=170, iT=30):
    wb = world_from_engine(world)
    return _ref().ref_lfv_fitness(ptr(np.ascontiguousarray(cand)), 8, PROB_PATH, C.byref(wb.struct()), 16,
                                  30.0, 4.0, iG, iN, iT, seed)


def test_lfv_batch_path_fp64_equals_reference(eng64mt):
    """sf_lfv_batch on the path problem with the CLI's inner budget 8 x 170 x 30:
    each candidate's LFV equals the unmodified reference's lfv_fitness."""
    o = oracle()
    w = path_world()
    rng = np.random.default_rng(14)
    cands = rng.uniform(0.0, 2.6, (6, 48))
    cands[0] = pe.EVOLVED_PATH_HYPERS.reshape(-1)
    seeds = [o.or_derive_seed_idx(o.or_derive_seed(41, b"lfv"), b"lfv", i) for i in range(6)]
    got = eng64mt.lfv_batch("path", cands, seeds, 8, 170, 30, dim=16, world=w)
    for i in range(6):
        assert got[i] == ref_lfv_path(cands[i], w, seeds[i]), i


def test_evolve_path_fp64_equals_reference(eng64mt):
    """evolve (hsef.hpp:125-171) on the path problem: outer (2, 3) for 2
    evolutions, inner 8 x 170 x 30 -- traces and best hypers equal the
    reference's bit for bit."""
    w = path_world()
    r = eng64mt.evolve("path", (8, 170, 30), (2, 3, 2), 41, DEFAULT_GROUP_HYPERS[:2], dim=16, world=w)
    wb = world_from_engine(w)
    bt, rt, bh = np.zeros(2), np.zeros(2), np.zeros(48)
    st = _ref().ref_evolve(PROB_PATH, C.byref(wb.struct()), 16, 30.0, 4.0, 8, 170, 30, 2, 3, 2, 41,
                           ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS[:2])), ptr(bt), ptr(rt), ptr(bh))
    assert st == 0
    assert np.array_equal(r["best_lfv_trace"], bt) and np.array_equal(r["evolution_lfv_trace"], rt)
    assert np.array_equal(r["best"].reshape(-1), bh)


def test_lfv_batch_path_fp32_statistics(eng32mt, eng64mt):
    """FP32 inner runs (the config-3 bench line) against the FP64 ones on the
    same 40 candidates: the LFVs (best path fitness after 30 iterations) agree
    in distribution -- median within 3 %, two-sided Mann-Whitney U p > 0.01."""
    from scipy.stats import mannwhitneyu
    o = oracle()
    w = path_world()
    rng = np.random.default_rng(15)
    cands = np.tile(pe.EVOLVED_PATH_HYPERS.reshape(-1), (40, 1)) * rng.uniform(0.8, 1.2, (40, 48))
    seeds = [o.or_derive_seed_idx(77, b"lfv", i) for i in range(40)]
    l32 = eng32mt.lfv_batch("path", cands, seeds, 8, 170, 30, dim=16, world=w)
    l64 = eng64mt.lfv_batch("path", cands, seeds, 8, 170, 30, dim=16, world=w)
    assert np.all(np.isfinite(l32))
    assert abs(np.median(l32) - np.median(l64)) <= 0.03 * np.median(l64)
    assert mannwhitneyu(l32, l64).pvalue > 0.01


# --------------------------------------------------- run_scenario variants
@pytest.mark.parametrize("variant", ["sepso", "sepso-noat", "sepso-nopi", "dtpso", "dppso", "pso"])
def test_run_scenario_variant_fp64_equals_reference(variant, eng64mt):
    """sf_run_scenario(variant) == the unmodified reference's run_scenario on
    every frame record (simenv.hpp:188-276).  `pso` is one group of 1,360
    particles spread over the whole cluster."""
    frames = 8
    base = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    recs = eng64mt.run_scenario(pe.ScenarioConfig(root_seed=5), variant, frames, base)
    ro = (PlanRecord * frames)()
    cfg = planner_cfg(max_iters=30, window_carryover=1)
    assert _ref().ref_run_scenario(5, pe.engine.VARIANTS.index(variant), frames, C.byref(cfg), ro, None) == 0
    for f in range(frames):
        got, want = recs[f], ro[f]
        assert (got.iterations, got.intersections, got.truncated, got.collision_free) == \
            (want.iterations, want.intersections, bool(want.truncated), bool(want.collision_free)), (variant, f)
        assert got.fitness == want.fitness and got.length == want.length, (variant, f)


# ------------------------------------------- FP32 records on the FP64 world
def test_fp32_record_is_the_reference_evaluation_of_its_path(eng32mt):
    """The FP32 engine plans on the FP32-rounded world, but its PlanRecord is
    the reference's own evaluation of the returned path on the caller's FP64
    world: Q with the reference's predicates, length with its hypot, fitness
    = length + 30 Q^4 (geometry.hpp:196-241) -- bit for bit."""
    o = oracle()
    planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    recs = eng32mt.run_scenario(pe.ScenarioConfig(root_seed=9), "sepso", 12, planner)
    w = pe.generate_world(pe.ScenarioConfig(root_seed=9), o.or_derive_seed(9, b"world"), "mt19937")
    for f, r in enumerate(recs):
        best = pe.encode_path(r.best_path).astype(np.float64)
        wb = world_from_engine(w)
        fit, q, ln = np.zeros(1), np.zeros(1, dtype=np.uint32), np.zeros(1)
        from oracle_lib import u32p
        _ref().ref_eval_path_rows(C.byref(wb.struct()), ptr(best), 1, 16, 30.0, 4.0, ptr(fit), ptr(q, u32p), ptr(ln))
        assert r.intersections == q[0] and r.collision_free == (q[0] == 0), f
        assert r.length == ln[0] and r.fitness == fit[0], f
        w = pe.step_world(w, 1.0)
    # scene batches (device-resident frames, world stepped in the same launch) agree
    sb = pe.SceneBatch(eng32mt, [pe.ScenarioConfig(root_seed=9)], planner, pe.EVOLVED_PATH_HYPERS, 12)
    sb.run(12)
    rb, _ = sb.records(0, 12)
    sb.close()
    assert [(r.fitness, r.intersections) for r in rb] == [(r.fitness, r.intersections) for r in recs]


# --------------------------------------- the `scale` harness (8(f) 4)
@pytest.mark.parametrize("shape", [(8, 64, 32, 12), (8, 2048, 64, 4), (8, 4096, 32, 10)])
def test_engine_equals_per_particle_oracle(shape, eng64mt):
    """proj/tools/swarmforge.cpp:202-255 compares the batched run_dtpso with the
    per-particle run_dppso_reference (runner.hpp:135-239); the FP64 engine --
    fused cluster for the small shape, the HBM-staged path for the large one --
    equals the per-particle oracle's trace and final point bit for bit."""
    G, N, D, T = shape
    r = eng64mt.run_dtpso("BF3", DEFAULT_GROUP_HYPERS, G, N, T, 1, dim=D)
    tr, fp, ff, wall = np.zeros(T), np.zeros(D), C.c_double(0), C.c_double(0)
    assert _ref().ref_run_dppso_reference(3, None, D, 30.0, 4.0, ptr(np.ascontiguousarray(DEFAULT_GROUP_HYPERS)),
                                          G, N, T, 1, ptr(tr), ptr(fp), C.byref(ff), C.byref(wall)) == 0
    assert np.array_equal(r["trace"], tr) and np.array_equal(r["final_point"], fp) and r["final_fitness"] == ff.value
