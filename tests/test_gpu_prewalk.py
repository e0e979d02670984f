"""The next frame's init walk ahead of time (csrc/prewalk.cu): run_scenario
and scene batches read frame f+1's init words, walked on a spare SM while
frame f planned, instead of walking them in the planning kernel.  The
results must be bit-identical to walking in the kernel (SEPSO_PREWALK=0),
and to the kernel's fallback when the announced walk never arrives
(SEPSO_PREWALK_TEST=late: the kernel waits ~2 ms, then walks itself).  Batches
of more than 8 scenes take the bulk walk (one launch for every scene,
ordered before the frame by an event).  The FP64 reference parity of the
paths is pinned in test_gpu_scene.py."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(**env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "prewalk_worker.py")], env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_prewalk_equals_in_kernel_walk_and_fallback():
    ahead = _run(SEPSO_PREWALK="1")
    inkernel = _run(SEPSO_PREWALK="0")
    late = _run(SEPSO_PREWALK="1", SEPSO_PREWALK_TEST="late")
    for key in ("fp32", "fp64", "batch", "bulk"):
        assert ahead[key] == inkernel[key], key
        assert late[key] == inkernel[key], key
