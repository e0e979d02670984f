import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
w4 = pe.generate_world(pe.ScenarioConfig(map_size=366.0 * np.sqrt(128.0), dynamic_obstacles=768, static_obstacles=256, root_seed=1), 1)
def frame4(cap, seed):
    cfg4 = pe.PlannerConfig(groups=8, per_group=8192, dim=128, max_iters_per_frame=cap, auto_truncate=False)
    eng.enable_timing(True)
    rec = eng.plan_frame(w4, None, pe.EVOLVED_PATH_HYPERS, cfg4, seed)
    ms_, _ = eng.kernel_time(); eng.enable_timing(False)
    return ms_, rec.fitness
frame4(1, 999)
a, fa = frame4(2, 1000); b, fb = frame4(10, 1000)
print(os.environ.get("SEPSO_LIB", "default"), f"steady {(b - a) / 8:.2f} ms/iter, fitness10 {fb}")
