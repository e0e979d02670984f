import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2308_10169_b200 as pe
for rng in ("mt19937",):
    eng = pe.Engine(0, "fp32", rng)
    seeds = np.arange(1, 1025, dtype=np.uint64)
    eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds[:64])
    for C, T in ((0, 0), (1, 192), (1, 256), (1, 320), (1, 384), (1, 512), (2, 256), (0, 0)):
        eng.set_launch(C, T)
        eng.enable_timing(True)
        t0 = time.perf_counter()
        eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds)
        t1 = time.perf_counter()
        ms, n = eng.kernel_time(); eng.enable_timing(False)
        print(f"{rng} C={C} T={T}: wall {1e3*(t1-t0):.1f} ms, kernel {ms:.1f} ms")
    eng.close()
