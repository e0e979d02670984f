"""Config 3 (HSEF evolve, inner 8x170x30 path swarms, outer 8x10): wall time
per evolution vs the planning kernels' CUDA-event time (host outer PSO and
staging are the difference)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
w = pe.generate_world(pe.ScenarioConfig(root_seed=3), 7)
eng.evolve("path", (8, 170, 30), (8, 10, 1), 41, world=w, dim=16)
for E in (3, 10):
    eng.enable_timing(True)
    t0 = time.perf_counter()
    r = eng.evolve("path", (8, 170, 30), (8, 10, E), 41, world=w, dim=16)
    t1 = time.perf_counter()
    ms, n = eng.kernel_time()
    eng.enable_timing(False)
    print(f"E={E}: wall {(t1 - t0) / E * 1e3:.3f} ms/evolution, kernel {ms / E:.3f} ms/evolution over {n} launches")
