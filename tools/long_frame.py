"""One config-2-shaped frame with a long iteration budget and AT off: a single
fused launch long enough for ncu's per-line stall sampling of the loop."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
w = pe.generate_world(pe.ScenarioConfig(root_seed=3), 12345)
cfg = pe.PlannerConfig(max_iters_per_frame=int(sys.argv[1]) if len(sys.argv) > 1 else 400, auto_truncate=False)
for _ in range(3):
    r = eng.plan_frame(w, None, pe.EVOLVED_PATH_HYPERS, cfg, 777)
print(r.iterations, r.fitness)
