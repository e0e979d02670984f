"""Per-phase cycles of the config-5 throughput kernel (PROF build, swarm 0 / CTA 0
of a 1,024-scene batch, warm frames)."""
import os, sys
os.environ["SEPSO_PHASE_PROF"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("SEPSO_LIB", os.path.join(ROOT, "paper_2308_10169_b200", "lib_prof", "libsepso_cuda.so"))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
n = int(os.environ.get("PROBE_SCENES", "1024"))
sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(n)], planner, pe.EVOLVED_PATH_HYPERS, 4)
sb.run(4)
recs, _ = sb.records(1, 3)
print("mean iterations", sum(r.iterations for r in recs) / len(recs))
