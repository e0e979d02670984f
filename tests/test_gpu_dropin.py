"""The C++ drop-in (include/swarmforge/*.hpp) on the GPU: a reference user's
program (examples/plan_route.cpp, examples/minimize_rastrigin.cpp) compiled
against the headers + libsepso_cuda.so gives the engine's results -- and, in
FP64 mode, the reference's (Philox harness) results frame for frame."""
import os
import subprocess

import numpy as np
import pytest

import paper_2308_10169_b200 as pe
from oracle_lib import (EVOLVED_PATH_HYPERS, RNG_MT, RNG_PHILOX, generate_world, oracle, oracle_plan_frame,
                        planner_cfg, ptr, u32p)

pytestmark = pytest.mark.gpu
LIB = os.path.dirname(pe.LIB_PATH)


def run(binary, *args, precision="fp32"):
    env = dict(os.environ, SEPSO_PRECISION=precision)
    out = subprocess.run([os.path.join(LIB, binary), *map(str, args)], capture_output=True, text=True,
                         env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    return out.stdout


def parse_frames(text):
    rows = []
    for line in text.splitlines():
        parts = line.split()
        if parts and parts[0].isdigit():
            rows.append((int(parts[1]), int(parts[2]), int(parts[3]), float(parts[4]), float(parts[5])))
    return rows


def test_plan_route_matches_python_engine(eng32mt):
    rows = parse_frames(run("plan_route", 12, 3))
    recs = eng32mt.run_scenario(pe.ScenarioConfig(root_seed=3), "sepso", 12,
                              pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True))
    assert [(r.iterations, int(r.truncated), r.intersections, r.fitness, r.length) for r in recs] == rows


def test_plan_route_fp64_equals_reference_harness():
    """FP64 drop-in (default mt19937 stream) == the UNMODIFIED reference's frames."""
    rows = parse_frames(run("plan_route", 8, 3, precision="fp64"))
    o = oracle()
    w = generate_world("oracle", o.or_derive_seed(3, b"world"), RNG_MT)
    cfg = planner_cfg(max_iters=30, window_carryover=1)
    prev, win = None, []
    for f, (it, tr, q, fit, length) in enumerate(rows):
        st, rec, best, win, _ = oracle_plan_frame(w, prev, EVOLVED_PATH_HYPERS, cfg,
                                                  o.or_derive_seed_idx(3, b"plan", f), RNG_MT, win)
        assert (rec.iterations, rec.truncated, rec.intersections) == (it, tr, q)
        assert rec.fitness == fit and rec.length == length
        prev = best
        o.or_step_world(ptr(w.head), w.n, ptr(w.offsets, u32p), ptr(w.verts), ptr(w.vel), 1.0)


def test_minimize_rastrigin_matches_python_engine(eng32mt):
    text = run("minimize_rastrigin")
    final = float(text.splitlines()[0].split()[3])
    r = eng32mt.run_dtpso("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, 42, dim=30)
    assert final == r["final_fitness"]
    assert "evolve best" in text
