"""Golden statistics over 32 scenario seeds (SURVEY.md 8(d), config 2:
"Statistical parity: root_seed in 1..32, compare mean path length and
collision_free_fraction"), produced by the UNMODIFIED reference compiled under
oracle/_ref (mt19937_64 stream).  Run here (CPU); the fixture travels."""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import PlanRecord, planner_cfg, ref  # noqa: E402

FRAMES = 20
mt = ref("mt")
out = {"frames": FRAMES, "planner": dict(max_iters=30, window_carryover=1), "seeds": {}}
for seed in range(1, 33):
    recs = (PlanRecord * FRAMES)()
    assert mt.ref_run_scenario(seed, 0, FRAMES, C.byref(planner_cfg(max_iters=30, window_carryover=1)), recs,
                               None) == 0
    r = [recs[i] for i in range(FRAMES)]
    out["seeds"][str(seed)] = dict(iterations=[x.iterations for x in r], length=[x.length for x in r],
                                   collision_free=[int(x.intersections == 0) for x in r],
                                   truncated=[int(x.truncated) for x in r])
with open(os.path.join(HERE, "scenario_32seeds.json"), "w") as f:
    json.dump(out, f)
lens = [np.mean(v["length"]) for v in out["seeds"].values()]
print("mean length", np.mean(lens), "collision-free", np.mean([np.mean(v["collision_free"]) for v in out["seeds"].values()]))
