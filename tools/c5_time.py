"""Config-5 A/B: 1,024 paper scenes, warm frames 1-3 (three fused launches)
timed with CUDA events on the launching stream, as bench.py's config5 extra."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
stream = torch.cuda.ExternalStream(eng.stream, device=torch.device('cuda', 0))
best = []
for rep in range(3):
    sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(1024)], planner, pe.EVOLVED_PATH_HYPERS, 4)
    sb.run(1)
    eng.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        sb.run(3)
        e1.record(stream)
    torch.cuda.synchronize()
    best.append(e0.elapsed_time(e1))
    sb.close()
print("config5 warm frames 1-3: %.3f ms  (%.0f plans/s)" % (min(best), 3 * 1024 / (min(best) / 1e3)))
