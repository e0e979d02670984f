"""Per-frame time of SceneBatch.run(1) with and without an L2 flush between frames."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_10169_b200 as pe
eng = pe.Engine(0, "fp32")
stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", 0))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
planner = pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True)
for mode in ("flush", "noflush"):
    K, W = 40, 5
    sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=3)], planner, pe.EVOLVED_PATH_HYPERS, W + K)
    sb.run(W)
    eng.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with torch.cuda.stream(stream):
        for i in range(K):
            if mode == "flush":
                flush.zero_()
            evs[i][0].record(stream)
            sb.run(1)
            evs[i][1].record(stream)
    torch.cuda.synchronize(); eng.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    recs, _ = sb.records(W, K)
    it = sum(r.iterations for r in recs) / K
    import numpy as np
    its = np.array([r.iterations for r in recs], dtype=float)
    A = np.vstack([np.ones(K), its]).T
    (a, b), *_ = np.linalg.lstsq(A, 1e3 * np.array(ms), rcond=None)
    print(f"{mode:8s} mean {1e3*sum(ms)/K:.1f} us/frame  min {1e3*min(ms):.1f}  iters {it:.2f}  fit: {a:.1f} us + {b:.2f} us/iter")
    sb.close()
