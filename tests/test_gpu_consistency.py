"""Cluster-decision consistency (race detection): the fused
kernel's partial exchange has no closing cluster barrier and relies on every
CTA taking identical decisions (stop, status, new tbest group, changed gbest
slots) at every iteration.  The consistency build (make VARIANT=check
EXTRA=-DSEPSO_CHECK) logs each CTA's decision word per iteration and the host
fails the call when two CTAs of a cluster differ.  compute-sanitizer is not
available on this pool, so this is the race check of record.  The test runs
scenario frames, batched scenes, HSEF and benchmark trials through that build
in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2308_10169_b200", "lib_check", "libsepso_cuda.so")

SCRIPT = r'''
import sys
sys.path.insert(0, sys.argv[1])
import paper_2308_10169_b200 as pe
for prec in ("fp32", "fp64"):
    for rng in ("mt19937", "philox"):
        eng = pe.Engine(0, prec, rng)
        recs = eng.run_scenario(pe.ScenarioConfig(root_seed=3), "sepso", 25,
                                pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True))
        for v in ("dtpso", "pso"):
            eng.run_scenario(pe.ScenarioConfig(root_seed=4), v, 4, pe.PlannerConfig(max_iters_per_frame=30))
        sb = pe.SceneBatch(eng, [pe.ScenarioConfig(root_seed=s) for s in range(64)],
                           pe.PlannerConfig(max_iters_per_frame=30, window_carryover=True), pe.EVOLVED_PATH_HYPERS, 3)
        sb.run(3)
        sb.records(0, 3)
        sb.close()
        w = pe.generate_world(pe.ScenarioConfig(root_seed=3), pe.derive_seed(3, "world"))
        eng.evolve("path", (8, 170, 10), (2, 4, 2), 41, pe.DEFAULT_GROUP_HYPERS[:2], dim=16, world=w)
        eng.run_dtpso_batched("BF3", pe.DEFAULT_GROUP_HYPERS, 8, 10, 200, list(range(1, 65)))
        eng.close()
print("consistent")
'''


def test_cluster_decisions_identical_across_ctas():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2308_10169_b200"), "VARIANT=check",
                        "EXTRA=-DSEPSO_CHECK"], check=True)
    env = dict(os.environ, SEPSO_LIB=LIB)
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "consistent" in out.stdout
    # the check is live: a flipped decision word must fail the call
    env["SEPSO_CHECK_SELFTEST"] = "1"
    bad = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=900)
    assert bad.returncode != 0 and "consistency check" in bad.stderr
