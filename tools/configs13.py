"""Config 1 (BF1-BF4 trials, batched) and config 3 (HSEF evolutions) timings."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
# config 1: 1,024 trials of G=8 x N=10 x T=1400 on D=30, per benchmark
for name in ("sphere", "rosenbrock", "rastrigin", "griewank"):
    seeds = np.arange(1, 1025, dtype=np.uint64)
    eng.run_dtpso_batched(name, pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds[:64])
    t0 = time.perf_counter()
    tr, fp, ff, st = eng.run_dtpso_batched(name, pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds)
    t1 = time.perf_counter()
    print(f"config1 {name}: {1024 / (t1 - t0):.0f} trials/s, {1024 * 80 * 1400 / (t1 - t0) / 1e9:.2f} G evals/s, median final {np.median(ff):.3g}")
# config 3: HSEF on the frozen frame-0 paper world, inner (8,170,30), outer (8,10,E)
w = pe.generate_world(pe.ScenarioConfig(root_seed=3), 7)
for E in (1, 3):
    t0 = time.perf_counter()
    r = eng.evolve("path", (8, 170, 30), (8, 10, E), 41, world=w, dim=16)
    t1 = time.perf_counter()
    print(f"config3 E={E}: {(t1 - t0) / E * 1e3:.1f} ms per evolution (80 inner swarms x 30 iterations), best lfv {r['best_lfv_trace'][-1]:.3f}")
