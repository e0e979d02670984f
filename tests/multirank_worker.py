"""One rank of tests/test_gpu_multirank.py: a gloo process group over
127.0.0.1, the engine on cuda:0 sharded through sf_ctx_set_exchange (host
all-gather -- the ranks share one device, and their kernels never wait on each
other; only the host exchange couples them).  Writes its results to a .npz."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    rank, ws, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    import torch
    import torch.distributed as td
    import paper_2308_10169_b200 as pe
    td.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)

    def allgather(b: bytes) -> bytes:
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(ws)]
        td.all_gather(parts, t)
        return b"".join(p.numpy().tobytes() for p in parts)

    res = {}
    for prec in ("fp64", "fp32"):
        eng = pe.Engine(0, prec, "mt19937")
        eng.set_exchange(ws, rank, allgather)
        w = pe.generate_world(pe.ScenarioConfig(root_seed=7), pe.derive_seed(7, "world"))
        cfg = pe.PlannerConfig(groups=8, per_group=512, dim=16, max_iters_per_frame=14, window_carryover=True)
        win = [300.0 + i for i in range(20)]
        rec = eng.plan_frame_sharded(w, None, pe.EVOLVED_PATH_HYPERS, cfg, 4242, win)
        res[f"{prec}_frame"] = np.array([rec.fitness, rec.length, rec.intersections, rec.iterations, rec.truncated])
        res[f"{prec}_best"] = pe.encode_path(rec.best_path)
        res[f"{prec}_win"] = np.array(win)
        ev = eng.evolve("path", (8, 170, 10), (2, 3, 2), 41, pe.DEFAULT_GROUP_HYPERS[:2], dim=16, world=w)
        res[f"{prec}_evolve"] = np.concatenate([ev["best_lfv_trace"], ev["evolution_lfv_trace"], ev["best"].reshape(-1)])
        eng.set_exchange(1, 0)
        eng.close()
    np.savez(out, **res)
    td.barrier()
    td.destroy_process_group()


if __name__ == "__main__":
    main()
