"""The sharded engine run for real with two ranks: config 4's
group split with the per-iteration tbest-candidate exchange
(sf_plan_frame_sharded, runner.hpp:81-91) and config 3's HSEF candidate split
with the LFV all-gather (sf_evolve, hsef.hpp:151-165).  Two processes, a gloo
process group, the exchange through sf_ctx_set_exchange; both ranks share the
one GPU of the box (their kernels are independent -- only the host exchange
couples them).  Each rank's results must equal the unsharded run bit for bit
(FP64 and FP32: the shards draw the global rows' words and reduce in the
reference's group order)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2308_10169_b200 as pe

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(tmp_path, ws):
    port = _free_port()
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(ws)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "multirank_worker.py"), str(r), str(ws), str(port),
                               outs[r]]) for r in range(ws)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    return [dict(np.load(o)) for o in outs]


@pytest.fixture(scope="module")
def two_ranks(tmp_path_factory):
    return _run_ranks(tmp_path_factory.mktemp("mr"), 2)


def _unsharded(prec):
    eng = pe.Engine(0, prec, "mt19937")
    w = pe.generate_world(pe.ScenarioConfig(root_seed=7), pe.derive_seed(7, "world"))
    cfg = pe.PlannerConfig(groups=8, per_group=512, dim=16, max_iters_per_frame=14, window_carryover=True)
    win = [300.0 + i for i in range(20)]
    rec = eng.plan_frame_sharded(w, None, pe.EVOLVED_PATH_HYPERS, cfg, 4242, win)
    ev = eng.evolve("path", (8, 170, 10), (2, 3, 2), 41, pe.DEFAULT_GROUP_HYPERS[:2], dim=16, world=w)
    eng.close()
    return {"frame": np.array([rec.fitness, rec.length, rec.intersections, rec.iterations, rec.truncated]),
            "best": pe.encode_path(rec.best_path), "win": np.array(win),
            "evolve": np.concatenate([ev["best_lfv_trace"], ev["evolution_lfv_trace"], ev["best"].reshape(-1)])}


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_two_rank_sharded_frame_equals_unsharded(prec, two_ranks):
    ref = _unsharded(prec)
    for r in two_ranks:
        for key in ("frame", "best", "win"):
            assert np.array_equal(r[f"{prec}_{key}"], ref[key]), (prec, key)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_two_rank_sharded_evolve_equals_unsharded(prec, two_ranks):
    ref = _unsharded(prec)
    for r in two_ranks:
        assert np.array_equal(r[f"{prec}_evolve"], ref["evolve"]), prec
