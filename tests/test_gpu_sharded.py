"""The HBM-resident (staged) large-swarm path on the GPU: sf_plan_frame_sharded
== the fused planner == the oracle in FP64, incl. a wide world (lanes-over-
obstacles kernel) and an attached 1-rank NCCL communicator."""
import numpy as np
import pytest

import paper_2308_10169_b200 as pe
from oracle_lib import (EVOLVED_PATH_HYPERS, RNG_PHILOX, float_world, oracle, oracle_plan_frame,
                        planner_cfg, world_from_engine)

pytestmark = pytest.mark.gpu


def paper_world(root=3):
    return pe.generate_world(pe.ScenarioConfig(), oracle().or_derive_seed(root, b"world"))


def wide_world(seed=5, n_dyn=48, n_static=16, size=1000.0):
    sc = pe.ScenarioConfig(map_size=size, dynamic_obstacles=n_dyn, static_obstacles=n_static)
    return pe.generate_world(sc, seed)


def test_sharded_single_gpu_equals_fused_and_oracle(eng64):
    o = oracle()
    w = paper_world()
    cfg = pe.PlannerConfig(max_iters_per_frame=20, window_carryover=True)
    prev, win_a, win_b = None, [], []
    for f in range(3):
        seed = o.or_derive_seed_idx(3, b"plan", f)
        a = eng64.plan_frame(w, prev, EVOLVED_PATH_HYPERS, cfg, seed, win_a)
        b = eng64.plan_frame_sharded(w, prev, EVOLVED_PATH_HYPERS, cfg, seed, win_b)
        assert (a.iterations, a.truncated, a.intersections) == (b.iterations, b.truncated, b.intersections)
        assert a.fitness == b.fitness and a.length == b.length
        assert np.array_equal(a.best_path, b.best_path) and win_a == win_b
        prev = a.best_path
        w = pe.step_world(w, 1.0)


def test_sharded_wide_world_fp64_equals_oracle(eng64):
    """64 obstacles -> the lanes-over-obstacles evaluation kernel."""
    w = wide_world()
    cfg = pe.PlannerConfig(groups=8, per_group=40, dim=12, max_iters_per_frame=15, tw=5)
    rec = eng64.plan_frame_sharded(w, None, EVOLVED_PATH_HYPERS, cfg, 77)
    st, ro, best, _, _ = oracle_plan_frame(world_from_engine(w), None, EVOLVED_PATH_HYPERS,
                                           planner_cfg(G=8, N=40, D=12, max_iters=15, tw=5), 77, RNG_PHILOX)
    assert st == 0
    assert (rec.iterations, rec.truncated, rec.intersections) == (ro.iterations, bool(ro.truncated), ro.intersections)
    assert rec.fitness == ro.fitness and np.array_equal(pe.encode_path(rec.best_path), best)


def test_wide_world_fitness_q_fp32(eng32):
    """Per-row Q of the wide kernel (FP32, float-rounded world) == oracle."""
    w = float_world(wide_world(seed=9))
    rng = np.random.default_rng(1)
    xs = rng.uniform(0, 1000, (300, 16)).astype(np.float32).astype(np.float64)
    f, q = eng32.eval_path_rows(w, xs, 16)
    import ctypes as C
    from oracle_lib import ptr, u32p
    wb = world_from_engine(w)
    fo, qo = np.zeros(300), np.zeros(300, dtype=np.uint32)
    oracle().or_eval_path_rows(ptr(xs), 300, 16, C.byref(wb.struct()), 30.0, 4.0, ptr(fo), ptr(qo, u32p))
    assert np.array_equal(q, qo)
    assert np.all(np.abs(f - fo) <= 1e-5 * np.maximum(1.0, fo))


def test_sharded_with_one_rank_nccl_comm():
    e = pe.Engine(0, "fp64")
    try:
        e.init_comm(pe.Engine.comm_unique_id(), 1, 0)
        w = paper_world(4)
        cfg = pe.PlannerConfig(max_iters_per_frame=10)
        a = e.plan_frame_sharded(w, None, EVOLVED_PATH_HYPERS, cfg, 99)
        b = e.plan_frame(w, None, EVOLVED_PATH_HYPERS, cfg, 99)
        assert a.fitness == b.fitness and np.array_equal(a.best_path, b.best_path)
    finally:
        e.close()


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_config4_size_fitness_equals_oracle(prec, eng32, eng64):
    """BASELINE config 4 at full size: 1,024 obstacles (768 dynamic + 256 static
    on a 4,140.8 cm map), D = 128 (64 waypoints, 65 segments x 4,096 edges per
    row).  A sample of 48 rows -- random, and random walks near the straight
    start-target line, where the overlaps concentrate -- through the wide
    evaluation kernel: Q exact in both precisions, fitness bit-exact in FP64
    and within 1e-5 (relative) in FP32 (on the FP32-rounded world)."""
    eng = eng64 if prec == "fp64" else eng32
    sc = pe.ScenarioConfig(map_size=366.0 * np.sqrt(128.0), dynamic_obstacles=768, static_obstacles=256)
    w = pe.generate_world(sc, 1)
    if prec == "fp32":
        w = float_world(w)
    rng = np.random.default_rng(4)
    size = w.width
    xs = rng.uniform(0.0, size, (24, 128))
    t = np.linspace(0.0, 1.0, 66)[1:-1]
    line = np.concatenate([w.start[0] + t * (w.target[0] - w.start[0]), w.start[1] + t * (w.target[1] - w.start[1])])
    walks = np.clip(line[None, :] + rng.normal(0.0, 60.0, (24, 128)), 0.0, size)
    xs = np.vstack([xs, walks])
    if prec == "fp32":
        xs = xs.astype(np.float32).astype(np.float64)
    f, q = eng.eval_path_rows(w, xs, 128)
    import ctypes as C
    from oracle_lib import ptr, u32p
    wb = world_from_engine(w)
    n = len(xs)
    fo, qo = np.zeros(n), np.zeros(n, dtype=np.uint32)
    oracle().or_eval_path_rows(ptr(np.ascontiguousarray(xs)), n, 128, C.byref(wb.struct()), 30.0, 4.0, ptr(fo),
                               ptr(qo, u32p))
    assert np.array_equal(q, qo)
    assert qo[:24].min() > 0 and qo.max() > 50          # dense worlds: many crossings per row
    if prec == "fp64":
        assert np.array_equal(f, fo)
    else:
        assert np.all(np.abs(f - fo) <= 1e-5 * np.maximum(1.0, fo))
