"""Per-phase cycles of the fused kernel on config 1 (BF3 trials; PROF build)."""
import os, sys
os.environ["SEPSO_PHASE_PROF"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("SEPSO_LIB", os.path.join(ROOT, "paper_2308_10169_b200", "lib_prof", "libsepso_cuda.so"))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32", "mt19937")
seeds = np.arange(1, 1025, dtype=np.uint64)
eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, int(sys.argv[1]) if len(sys.argv) > 1 else 200, seeds)
