"""e2e (sf_plan_frame with host buffers) vs kernel-only time per frame."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
scen = pe.ScenarioConfig(root_seed=3)
eng.run_scenario(scen, "sepso", 10, planner)
for flush in (0, 256 * 1024 * 1024):
    eng.set_l2_flush(flush)
    recs = eng.run_scenario(scen, "sepso", 65, planner)
    wall = np.array([r.wall_seconds for r in recs[5:]]) * 1e6
    eng.enable_timing(True)
    recs2 = eng.run_scenario(scen, "sepso", 65, planner)
    ms, n = eng.kernel_time()
    eng.enable_timing(False)
    print(f"flush={flush>0}: e2e per frame {wall.mean():.1f} us (min {wall.min():.1f}); kernel per launch {1e3*ms/n:.1f} us over {n} launches; iters {np.mean([r.iterations for r in recs[5:]]):.2f}")
eng.set_l2_flush(0)
