"""Per-iteration cost of the fused planner vs obstacle count (auto-truncation
off, 30 iterations): separates the fixed barrier/sync skeleton from fitness."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe
rng = sys.argv[1] if len(sys.argv) > 1 else "mt19937"
eng = pe.Engine(0, "fp32", rng)
print("rng", rng)
scen = pe.ScenarioConfig(root_seed=3)
w8 = pe.generate_world(scen, 12345)
def rect(x0, y0, x1, y1):
    return [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]
worlds = {"O=0": pe.PolygonWorld(w8.width, w8.height, w8.start, w8.target, []), "O=8 paper": w8}
for cap in (1, 31):
    cfg = pe.PlannerConfig(max_iters_per_frame=cap, auto_truncate=False)
    for name, w in worlds.items():
        eng.plan_frame(w, None, pe.EVOLVED_PATH_HYPERS, cfg, 7)
        eng.enable_timing(True)
        for s in range(20):
            eng.plan_frame(w, None, pe.EVOLVED_PATH_HYPERS, cfg, 100 + s)
        ms, n = eng.kernel_time(); eng.enable_timing(False)
        print(f"cap {cap:2d} {name:10s}: {1e3 * ms / n:7.1f} us/launch")
