"""Smallest fused-kernel frames for compute-sanitizer (memcheck / racecheck /
synccheck): a 2-group scene frame in FP32 and FP64 through the normal launch,
then the same through the resident planner (SEPSO_RESIDENT unset)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
w = pe.generate_world(pe.ScenarioConfig(root_seed=3), pe.derive_seed(3, "world"))
for prec in ("fp32", "fp64"):
    eng = pe.Engine(0, prec)
    cfg = pe.PlannerConfig(groups=4, per_group=24, max_iters_per_frame=4, window_carryover=True)
    win = []
    prev = None
    for f in range(2):
        r = eng.plan_frame(w, prev, pe.EVOLVED_PATH_HYPERS[:4], cfg, 100 + f, win)
        prev = r.best_path
    print(prec, r.iterations, r.fitness, r.intersections)
    eng.close()
