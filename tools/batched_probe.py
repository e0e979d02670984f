"""Config 5 shape for ncu: 1,024 paper scenes, frame 0 then warm frames 1-3
(the bench's config5 extra); `-s 1 -c 1` captures the first warm frame."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(1024)], planner, pe.EVOLVED_PATH_HYPERS, 4)
sb.run(4)
recs, _ = sb.records(1, 3)
print("mean iterations", sum(r.iterations for r in recs) / len(recs))
