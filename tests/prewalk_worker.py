"""Records of one FP32 and one FP64 run_scenario and one FP32 scene batch, as
JSON on stdout (tests/test_gpu_prewalk.py runs this under different
SEPSO_PREWALK settings: the walk ahead of time, none, or announced but late)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2308_10169_b200 as pe

PLANNER = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
out = {}
for prec in ("fp32", "fp64"):
    eng = pe.Engine(0, prec, "mt19937")
    recs = eng.run_scenario(pe.ScenarioConfig(root_seed=5), "sepso", 8, PLANNER)
    out[prec] = [[r.fitness, r.length, r.iterations, r.truncated, r.intersections,
                  np.asarray(r.best_path, dtype=np.float64).ravel().tolist()] for r in recs]
    if prec == "fp32":
        sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=5)], PLANNER, pe.EVOLVED_PATH_HYPERS, 8)
        sb.run(3)
        sb.run(5)
        rb, best = sb.records(0, 8, with_best=True)
        sb.close()
        out["batch"] = [[r.fitness, r.length, r.iterations, r.truncated, r.intersections] for r in rb] + \
                       [np.asarray(best, dtype=np.float64).ravel().tolist()]
        # more than 8 scenes: the bulk walk (one launch for every scene, event-ordered)
        sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=20 + i) for i in range(12)], PLANNER,
                           pe.EVOLVED_PATH_HYPERS, 4)
        sb.run(4)
        rb, best = sb.records(0, 4, with_best=True)
        sb.close()
        out["bulk"] = [[r.fitness, r.length, r.iterations, r.truncated, r.intersections] for r in rb] + \
                      [np.asarray(best, dtype=np.float64).ravel().tolist()]
    eng.close()
print(json.dumps(out))
