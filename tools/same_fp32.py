"""Prints a digest of FP32 planning results (scenario records of three root
seeds, a config-5 batch) so two library builds can be compared for identical
output: SEPSO_LIB=... python tools/same_fp32.py."""
import hashlib, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
h = hashlib.sha256()
for root in (3, 4, 5):
    recs = eng.run_scenario(pe.ScenarioConfig(root_seed=root), "sepso", 60,
                            pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True))
    for r in recs:
        h.update(np.array([r.fitness, r.length, r.intersections, r.iterations, r.truncated], dtype=np.float64).tobytes())
        h.update(pe.encode_path(r.best_path).astype(np.float64).tobytes())
sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(256)],
                   pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True), pe.EVOLVED_PATH_HYPERS, 4)
sb.run(4)
recs, best = sb.records(0, 4, with_best=True) if True else None
for r in recs:
    h.update(np.array([r.fitness, r.iterations, r.truncated], dtype=np.float64).tobytes())
print("digest", h.hexdigest()[:16], "mean iters", np.mean([r.iterations for r in recs]))
