import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32", "mt19937")
seeds = np.arange(1, 1025, dtype=np.uint64)
eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds)
ts = []
for i in range(5):
    eng.enable_timing(True)
    t0 = time.perf_counter()
    tr, fp, ff, st = eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 1400, seeds)
    t1 = time.perf_counter()
    ms, n = eng.kernel_time(); eng.enable_timing(False)
    ts.append((1e3 * (t1 - t0), ms))
print("wall/kernel ms", [f"{a:.1f}/{b:.1f}" for a, b in ts], "checksum", float(np.sum(ff)), float(np.sum(tr[:, -1])))
