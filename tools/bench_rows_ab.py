"""A/B of the benchmark-fitness paths between two library builds (SEPSO_LIB):
sf_eval_bench_rows (staged evaluation kernel) for BF1-BF4 + Ackley at several
D in both precisions, a fused-kernel run_dtpso (config-1 shape) and a staged
run_dtpso (the scale harness shape, T=4) per precision.  Writes every output
to gpurun_out/ab_<tag>.npz; `compare` checks two dumps bit for bit.

    python tools/bench_rows_ab.py dump <tag>
    python tools/bench_rows_ab.py compare <tagA> <tagB>
"""
import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np

if sys.argv[1] == "compare":
    a = np.load(f"gpurun_out/ab_{sys.argv[2]}.npz")
    b = np.load(f"gpurun_out/ab_{sys.argv[3]}.npz")
    bad = 0
    for k in a.files:
        same = a[k].tobytes() == b[k].tobytes()
        bad += not same
        if not same:
            print("DIFF", k, float(np.max(np.abs(a[k] - b[k]))))
    print(f"{len(a.files) - bad}/{len(a.files)} identical")
    sys.exit(1 if bad else 0)

import paper_2308_10169_b200 as pe
out = {}
rng = np.random.default_rng(7)
for prec in ("fp32", "fp64"):
    eng = pe.Engine(0, prec)
    for prob in ("BF1", "BF2", "BF3", "BF4", 5):
        for D in (1, 7, 30, 33, 100, 1000):
            rows = 1000 if D < 1000 else 300
            xs = rng.uniform(-5, 5, size=(rows, D))
            out[f"{prec}_eval_{prob}_{D}"] = eng.eval_bench_rows(prob, xs, D)
    r = eng.run_dtpso("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 200, 11, dim=30)          # fused
    out[f"{prec}_fused_trace"] = r["trace"]
    out[f"{prec}_fused_fp"] = r["final_point"]
    for prob in ("BF1", "BF2", "BF4", 5):                                             # fused, every function
        r = eng.run_dtpso(prob, pe.DEFAULT_GROUP_HYPERS, 8, 10, 150, 13, dim=30)
        out[f"{prec}_fused_{prob}_trace"] = r["trace"]
        out[f"{prec}_fused_{prob}_fp"] = r["final_point"]
    eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, 8, 16384, 2, 1, dim=1000)
    t0 = time.perf_counter()
    r = eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, 8, 16384, 4, 1, dim=1000)       # staged
    print(prec, "staged T=4", f"{1e3 * (time.perf_counter() - t0):.2f} ms")
    out[f"{prec}_staged_trace"] = r["trace"]
    out[f"{prec}_staged_fp"] = r["final_point"]
    r = eng.run_dtpso("BF2", pe.DEFAULT_GROUP_HYPERS, 8, 2048, 3, 5, dim=250)          # staged, Rosenbrock
    out[f"{prec}_staged2_trace"] = r["trace"]
    out[f"{prec}_staged2_fp"] = r["final_point"]
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/ab_{sys.argv[2]}.npz", **out)
print("dumped", len(out))
