"""The next frame's init walk ahead of time (csrc/prewalk.cu): run_scenario
and scene batches read frame f+1's init words, walked on a spare SM while
frame f planned, instead of walking them in the planning kernel.  The
results must be bit-identical to walking in the kernel (SEPSO_PREWALK=0),
and to the kernel's fallback when the announced walk never arrives
(SEPSO_PREWALK_TEST=late: the kernel waits ~2 ms, then walks itself).  Batches
of more than 8 scenes take the bulk walk (one launch for every scene,
ordered before the frame by an event).  The FP64 reference parity of the
paths is pinned in test_gpu_scene.py."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(**env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "prewalk_worker.py")], env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_prewalk_equals_in_kernel_walk_and_fallback():
    ahead = _run(SEPSO_PREWALK="1")
    inkernel = _run(SEPSO_PREWALK="0")
    late = _run(SEPSO_PREWALK="1", SEPSO_PREWALK_TEST="late")
    for key in ("fp32", "fp64", "batch", "bulk"):
        assert ahead[key] == inkernel[key], key
        assert late[key] == inkernel[key], key


def test_hinted_plan_frame_loop_equals_run_scenario():
    """A caller's own frame loop with sf_ctx_hint_next_seed (the drop-in
    run_scenario of simenv.hpp does this) plans the same frames as
    sf_run_scenario, bit for bit, in both precisions."""
    import numpy as np
    import paper_2308_10169_b200 as pe
    planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    scen = pe.ScenarioConfig(root_seed=7)
    frames = 6
    for prec in ("fp32", "fp64"):
        eng = pe.Engine(0, prec, "mt19937")
        try:
            ref = eng.run_scenario(scen, "sepso", frames, planner)
            w = pe.generate_world(scen, pe.derive_seed(scen.root_seed, "world"))
            prev, window = None, []
            for f in range(frames):
                eng.hint_next_seed(pe.derive_seed(scen.root_seed, "plan", f + 1) if f + 1 < frames else None)
                r = eng.plan_frame(w, prev, pe.EVOLVED_PATH_HYPERS, planner,
                                   pe.derive_seed(scen.root_seed, "plan", f), window)
                h = ref[f]
                assert (r.iterations, r.truncated, r.intersections) == (h.iterations, h.truncated, h.intersections)
                assert r.fitness == h.fitness and r.length == h.length
                assert np.array_equal(np.asarray(r.best_path), np.asarray(h.best_path))
                prev = r.best_path
                w = pe.step_world(w, scen.dt)
        finally:
            eng.close()
