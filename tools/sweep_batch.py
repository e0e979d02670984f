"""Launch-shape sweep for the batched scenes (config 5): warm frames 1-3 of
1,024 scenes per launch, device time per frame."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
nb = 1024
CS = [int(x) for x in os.environ.get("SWEEP_C", "0,2,4,8").split(",")]
TS = [int(x) for x in os.environ.get("SWEEP_T", "0,256,512,768,1024").split(",")]
for C in CS:
    for T in TS:
        eng.set_launch(C, T)
        try:
            sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(nb)], planner, pe.EVOLVED_PATH_HYPERS, 4)
            sb.run(1); eng.synchronize()
            eng.enable_timing(True)
            sb.run(3)
            ms, n = eng.kernel_time(); eng.enable_timing(False)
            recs, _ = sb.records(1, 3)
            sb.close()
            print(json.dumps(dict(C=C, T=T, plans_per_s=3 * nb / (ms / 1e3), ms_per_frame=ms / n,
                                  iters=float(np.mean([r.iterations for r in recs])))), flush=True)
        except Exception as ex:
            print(json.dumps(dict(C=C, T=T, error=str(ex))), flush=True)
