"""Phase breakdown of one frame with and without an L2 flush before it (PROF build)."""
import os, sys
os.environ["SEPSO_PHASE_PROF"] = "1"
os.environ.setdefault("SEPSO_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2308_10169_b200", "lib_prof", "libsepso_cuda.so"))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=3)], planner, pe.EVOLVED_PATH_HYPERS, 12)
sb.run(4)
for f in range(4, 12):
    if f % 2 == 0:
        flush.zero_(); torch.cuda.synchronize()
        print("flushed:", file=sys.stderr, flush=True)
    else:
        print("warm:", file=sys.stderr, flush=True)
    sb.run(1)
    eng.synchronize()
