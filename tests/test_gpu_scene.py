"""Device-resident scenarios (sf_scene_batch_*): every frame is one fused
planning launch that also advances the world record on the device
(simenv.hpp:155-184), with derive_seed(root, "plan", f) computed on the device.
The FP64 engine with the reference's mt19937_64 stream must reproduce the
UNMODIFIED reference scenario (golden vectors) and the host-driven
run_scenario (simenv.hpp:239-276) frame by frame."""
import json
import os

import numpy as np
import pytest

import paper_2308_10169_b200 as pe

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))
PLANNER = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)


def test_scene_batch_fp64_equals_reference_scenario(eng64mt):
    sb = pe.SceneBatch(eng64mt, [pe.ScenarioConfig(root_seed=3)], PLANNER, pe.EVOLVED_PATH_HYPERS, 100)
    sb.run(100)
    recs, _ = sb.records(0, 100)
    sb.close()
    s = GOLD["scenario_seed3"]
    assert [r.iterations for r in recs] == s["iterations"]
    assert sum(r.truncated for r in recs) == s["truncated"]
    assert abs(np.mean([r.length for r in recs]) - s["mean_length"]) < 1e-9


def test_scene_batch_equals_host_run_scenario(eng64mt):
    roots = [3, 17, 40]
    frames = 12
    sb = pe.SceneBatch(eng64mt, [pe.ScenarioConfig(root_seed=r) for r in roots], PLANNER,
                       pe.EVOLVED_PATH_HYPERS, frames)
    sb.run(5)
    sb.run(frames - 5)                      # frames in two calls: state carries over
    recs, best = sb.records(0, frames, with_best=True)
    sb.close()
    for i, root in enumerate(roots):
        host = eng64mt.run_scenario(pe.ScenarioConfig(root_seed=root), "sepso", frames, PLANNER)
        for f in range(frames):
            d, h = recs[f * len(roots) + i], host[f]
            assert (d.iterations, d.truncated, d.intersections) == (h.iterations, h.truncated, h.intersections)
            assert d.fitness == h.fitness and d.length == h.length
            assert np.array_equal(best[f, i], pe.encode_path(h.best_path) if np.ndim(h.best_path) == 2
                                  else np.asarray(h.best_path))


def test_scene_batch_fp32_statistics(eng32mt):
    sb = pe.SceneBatch(eng32mt, [pe.ScenarioConfig(root_seed=3)], PLANNER, pe.EVOLVED_PATH_HYPERS, 100)
    sb.run(100)
    recs, _ = sb.records(0, 100)
    sb.close()
    s = GOLD["scenario_seed3"]
    assert abs(np.mean([r.iterations for r in recs]) - s["mean_iterations"]) < 1.5
    assert abs(np.mean([r.length for r in recs]) - s["mean_length"]) < 0.02 * s["mean_length"]
    assert sum(r.collision_free for r in recs) >= 90


def test_scene_batch_philox_equals_host_run_scenario(eng64):
    """The same device-resident loop with the Philox stream (the harness build's)."""
    frames = 8
    sb = pe.SceneBatch(eng64, [pe.ScenarioConfig(root_seed=5)], PLANNER, pe.EVOLVED_PATH_HYPERS, frames)
    sb.run(frames)
    recs, _ = sb.records(0, frames)
    sb.close()
    host = eng64.run_scenario(pe.ScenarioConfig(root_seed=5), "sepso", frames, PLANNER)
    for d, h in zip(recs, host):
        assert (d.iterations, d.truncated, d.intersections) == (h.iterations, h.truncated, h.intersections)
        assert d.fitness == h.fitness and d.length == h.length


@pytest.mark.parametrize("eng_name", ["eng32mt", "eng64mt"])
def test_config5_size_batch_equals_single_scenes(eng_name, request):
    """BASELINE config 5 per GPU: 1,024 scenes in one batch (the throughput
    launch shape: ~680 rows per CTA, compacted pair tests) give, scene by
    scene, exactly the records and best paths of the same scenes run alone
    (the latency shape: 16 CTAs, in-place pair tests) -- in FP32 as in FP64."""
    eng = request.getfixturevalue(eng_name)
    n, frames = 1024, 3
    sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(n)], PLANNER, pe.EVOLVED_PATH_HYPERS,
                       frames)
    sb.run(frames)
    recs, best = sb.records(0, frames, with_best=True)
    sb.close()
    for s in (0, 1, 511, 1023):
        one = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s)], PLANNER, pe.EVOLVED_PATH_HYPERS, frames)
        one.run(frames)
        r1, b1 = one.records(0, frames, with_best=True)
        one.close()
        for f in range(frames):
            d, h = recs[f * n + s], r1[f]
            assert (d.iterations, d.truncated, d.intersections) == (h.iterations, h.truncated, h.intersections)
            assert d.fitness == h.fitness and d.length == h.length
            assert np.array_equal(best[f, s], b1[f, 0])
