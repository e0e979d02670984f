"""Kernel-internal globaltimer breakdown per frame (SEPSO_PHASE_PROF=1), frames 5..44."""
import os, sys
os.environ["SEPSO_PHASE_PROF"] = "1"
os.environ.setdefault("SEPSO_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2308_10169_b200", "lib_prof", "libsepso_cuda.so"))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=3)], planner, pe.EVOLVED_PATH_HYPERS, 45)
sb.run(45)
sb.records(0, 45)
