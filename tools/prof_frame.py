"""Short driver for ncu: a few device-resident frames of the paper scene
(config 2) and one batched frame (config 5 slice)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe

mode = sys.argv[1] if len(sys.argv) > 1 else "scene"
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
if mode == "scene":
    sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=3)], planner, pe.EVOLVED_PATH_HYPERS, 8)
    sb.run(8)
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 296
    sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(n)], planner, pe.EVOLVED_PATH_HYPERS, 3)
    sb.run(3)
recs, _ = sb.records(0, 1)
print("ok", recs[0].iterations)
sb.close()
eng.close()
