"""The bench's `scale` extra (BF1, G=8 N=16384 D=1000 T=10) timed alone:
wall time of run_dtpso through the host API for T=2 and T=10 (fixed cost and
cost per iteration).  Run it under ncu --metrics gpu__time_duration.sum for
the launch list of one T=10 run (SCALE_ONE=1)."""
import os, sys, time
sys.path.insert(0, '/root/repo')
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
G, N, D = 8, 16384, 1000
eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, G, N, 2, 1, dim=D)
if os.environ.get("SCALE_ONE"):
    r = eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, G, N, 10, 1, dim=D)
    print("final", r["final_fitness"])
    sys.exit(0)
for T in (2, 10, 2, 10):
    t0 = time.perf_counter()
    r = eng.run_dtpso("BF1", pe.DEFAULT_GROUP_HYPERS, G, N, T, 1, dim=D)
    print(f"T={T}: {1e3 * (time.perf_counter() - t0):.2f} ms  final {r['final_fitness']:.6g}")
