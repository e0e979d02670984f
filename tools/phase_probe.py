"""Per-phase cycle breakdown of the fused kernel (SEPSO_PHASE_PROF=1)."""
import os, sys
os.environ["SEPSO_PHASE_PROF"] = "1"
os.environ.setdefault("SEPSO_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2308_10169_b200", "lib_prof", "libsepso_cuda.so"))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, sys.argv[1] if len(sys.argv) > 1 else "fp32", sys.argv[2] if len(sys.argv) > 2 else "mt19937")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
for C, T in ((16, int(os.environ.get("PROBE_T", "896"))),):
    eng.set_launch(C, T)
    sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=3)], planner, pe.EVOLVED_PATH_HYPERS, 6)
    sb.run(6)
    sb.records(0, 6)
    sb.close()
