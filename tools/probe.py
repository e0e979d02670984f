"""Quick GPU probe: timings of the fused planner (not a bench number)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2308_10169_b200 as pe
from oracle_lib import oracle

o = oracle()
for prec in ("fp32", "fp64"):
    eng = pe.Engine(0, prec)
    root = 3
    w = pe.generate_world(pe.ScenarioConfig(), o.or_derive_seed(root, b"world"))
    cfg = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
    for rep in range(2):
        prev, win, its = None, [], []
        ww = w
        eng.enable_timing(True)
        t0 = time.perf_counter()
        for f in range(100):
            rec = eng.plan_frame(ww, prev, pe.EVOLVED_PATH_HYPERS, cfg, o.or_derive_seed_idx(root, b"plan", f), win)
            prev = rec.best_path
            its.append(rec.iterations)
            ww = pe.step_world(ww, 1.0)
        t1 = time.perf_counter()
        ms, n = eng.kernel_time()
        print(f"{prec} scenario: {1e3*(t1-t0)/100:.3f} ms/frame e2e, kernel {ms/n*1e3:.1f} us/frame, mean iters {np.mean(its):.2f}, coll-free {sum(1 for _ in its)}", flush=True)
    for n_sc in (148, 1024, 8192):
        worlds = [pe.generate_world(pe.ScenarioConfig(), o.or_derive_seed(s, b"world")) for s in range(n_sc)]
        seeds = [o.or_derive_seed_idx(s, b"plan", 0) for s in range(n_sc)]
        cfgb = pe.PlannerConfig(max_iters_per_frame=30)
        for rep in range(2):
            eng.enable_timing(True)
            t0 = time.perf_counter()
            recs, best, stat = eng.plan_frames_batched(worlds, None, None, pe.EVOLVED_PATH_HYPERS, cfgb, seeds)
            t1 = time.perf_counter()
            ms, n = eng.kernel_time()
        its = np.mean([r.iterations for r in recs])
        print(f"{prec} batched {n_sc}: e2e {1e3*(t1-t0):.2f} ms, kernel {ms:.2f} ms -> {n_sc/(ms/1e3):.0f} plans/s kernel, mean iters {its:.1f}", flush=True)
    eng.close()
