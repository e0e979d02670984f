"""32 scenario seeds (SURVEY.md 8(d), config 2 statistical parity): the FP64
engine with the reference's mt19937_64 stream reproduces the UNMODIFIED
reference frame by frame on every seed; the FP32 production engine matches its
mean path cost and collision-free fraction statistically.  Reference numbers:
tests/golden/scenario_32seeds.json (make_golden_seeds.py, oracle/_ref)."""
import json
import os

import numpy as np
import pytest

import paper_2308_10169_b200 as pe

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scenario_32seeds.json")))
FRAMES = GOLD["frames"]
SEEDS = list(range(1, 33))
PLANNER = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)


def run_batch(eng):
    sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in SEEDS], PLANNER, pe.EVOLVED_PATH_HYPERS,
                       FRAMES)
    sb.run(FRAMES)
    recs, _ = sb.records(0, FRAMES)
    sb.close()
    n = len(SEEDS)
    return {s: [recs[f * n + i] for f in range(FRAMES)] for i, s in enumerate(SEEDS)}


def test_fp64_32_seeds_equal_reference(eng64mt):
    got = run_batch(eng64mt)
    for s in SEEDS:
        g = GOLD["seeds"][str(s)]
        assert [r.iterations for r in got[s]] == g["iterations"], s
        assert [int(r.truncated) for r in got[s]] == g["truncated"], s
        assert [int(r.intersections == 0) for r in got[s]] == g["collision_free"], s
        assert [r.length for r in got[s]] == g["length"], s


def test_fp32_32_seeds_statistics(eng32mt):
    got = run_batch(eng32mt)
    ref_len = np.mean([np.mean(GOLD["seeds"][str(s)]["length"]) for s in SEEDS])
    ref_free = np.mean([np.mean(GOLD["seeds"][str(s)]["collision_free"]) for s in SEEDS])
    ref_it = np.mean([np.mean(GOLD["seeds"][str(s)]["iterations"]) for s in SEEDS])
    gl = np.mean([np.mean([r.length for r in got[s]]) for s in SEEDS])
    gf = np.mean([np.mean([r.intersections == 0 for r in got[s]]) for s in SEEDS])
    gi = np.mean([np.mean([r.iterations for r in got[s]]) for s in SEEDS])
    assert abs(gl - ref_len) < 0.03 * ref_len, (gl, ref_len)
    assert abs(gf - ref_free) < 0.06, (gf, ref_free)
    assert abs(gi - ref_it) < 1.5, (gi, ref_it)
