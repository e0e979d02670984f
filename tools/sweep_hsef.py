"""Launch-shape sweep for HSEF evolutions (80 inner paper swarms x 30 iterations)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
w = pe.generate_world(pe.ScenarioConfig(root_seed=3), 7)
eng.evolve("path", (8, 170, 30), (8, 10, 1), 40, world=w, dim=16)
for C, T in [(int(x.split(':')[0]), int(x.split(':')[1])) for x in os.environ.get('SHAPES', '0:0,2:1024,4:512,8:512').split(',')] * 2:
    if True:
        eng.set_launch(C, T)
        try:
            t0 = time.perf_counter()
            eng.evolve("path", (8, 170, 30), (8, 10, 3), 41, world=w, dim=16)
            t1 = time.perf_counter()
            print(f"C={C} T={T}: {(t1 - t0) / 3 * 1e3:.2f} ms per evolution", flush=True)
        except Exception as ex:
            print(f"C={C} T={T}: {ex}")
