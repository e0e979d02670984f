"""End-to-end frame time (sf_plan_frame wall, L2 flushed before each frame)
fitted as fixed + per-iteration over a 65-frame scenario (run under
SEPSO_RESIDENT=0/1 to compare the launch path with the resident planner)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
eng.run_scenario(pe.ScenarioConfig(root_seed=3), "sepso", 10, planner)
eng.set_l2_flush(256 * 1024 * 1024)
w, it = [], []
for root in (3, 4, 5):
    recs = eng.run_scenario(pe.ScenarioConfig(root_seed=root), "sepso", 65, planner)
    w += [r.wall_seconds * 1e6 for r in recs[5:]]
    it += [r.iterations for r in recs[5:]]
eng.set_l2_flush(0)
w, it = np.array(w), np.array(it, dtype=float)
(a, b), *_ = np.linalg.lstsq(np.vstack([np.ones_like(it), it]).T, w, rcond=None)
print(f"RESIDENT={os.environ.get('SEPSO_RESIDENT', '1')}: e2e {a:.1f} us + {b:.2f} us/iter over {len(w)} frames "
      f"(mean {w.mean():.1f} us at {it.mean():.2f} iters)")
