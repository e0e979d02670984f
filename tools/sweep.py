"""Launch-shape sweep of the fused planner (cluster size x threads): device
time per frame for one scene (latency) and per batched frame (throughput)."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_10169_b200 as pe

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
eng = pe.Engine(0, prec)
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
cold = pe.PlannerConfig(max_iters_per_frame=30)
res = []
CS = [int(x) for x in os.environ.get('SWEEP_C', '4,8,16').split(',')]
TS = [int(x) for x in os.environ.get('SWEEP_T', '256,512,1024').split(',')]
for C in CS:
    for T in TS:
        eng.set_launch(C, T)
        try:
            # latency: one scenario, 40 frames
            sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=3)], planner, pe.EVOLVED_PATH_HYPERS, 40)
            sb.run(5); eng.synchronize()
            eng.enable_timing(True)
            sb.run(35)
            ms, n = eng.kernel_time(); eng.enable_timing(False)
            recs, _ = sb.records(5, 35)
            it = np.mean([r.iterations for r in recs])
            sb.close()
            # throughput: 1184 cold scenes, 1 frame
            nb = 1184
            sbb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(nb)], cold, pe.EVOLVED_PATH_HYPERS, 2)
            sbb.run(1); eng.synchronize()
            eng.enable_timing(True)
            sbb.run(1)
            msb, nb_ = eng.kernel_time(); eng.enable_timing(False)
            rb, _ = sbb.records(1, 1)
            itb = np.mean([r.iterations for r in rb])
            sbb.close()
            r = dict(C=C, T=T, scene_us_per_frame=1e3 * ms / n, scene_us_per_iter=1e3 * ms / n / it, scene_iters=it,
                     batch_ms=msb, batch_plans_per_s=nb / (msb / 1e3), batch_iters=itb,
                     batch_evals_per_s=nb * itb * 1360 / (msb / 1e3))
        except Exception as ex:
            r = dict(C=C, T=T, error=str(ex))
        print(json.dumps(r), flush=True)
        res.append(r)
