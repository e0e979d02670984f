"""BASELINE config 4 on one GPU: 65,536 particles x 64 waypoints x 1,024
obstacles (map 4140.8 cm, 768 dynamic + 256 static), one frame (cap 30)."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 30
eng = pe.Engine(0, "fp32")
sc = pe.ScenarioConfig(map_size=366.0 * np.sqrt(128.0), dynamic_obstacles=768, static_obstacles=256, root_seed=1)
w = pe.generate_world(sc, 1)
cfg = pe.PlannerConfig(groups=8, per_group=8192, dim=128, max_iters_per_frame=cap)
prev = None
for f in range(frames):
    eng.enable_timing(True)
    t0 = time.perf_counter()
    rec = eng.plan_frame_sharded(w, prev, pe.EVOLVED_PATH_HYPERS, cfg, 1000 + f)
    t1 = time.perf_counter()
    ms, n = eng.kernel_time()
    evals = rec.iterations * 65536
    print(json.dumps(dict(frame=f, iterations=rec.iterations, q=rec.intersections, fitness=rec.fitness,
                          wall_ms=1e3 * (t1 - t0), device_ms=ms, evals_per_s=evals / (ms / 1e3),
                          ms_per_iter=ms / rec.iterations)), flush=True)
    prev = rec.best_path
