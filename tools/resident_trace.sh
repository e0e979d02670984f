#!/bin/bash
# Resident-planner timing split (SEPSO_RESIDENT_TRACE) of tools/e2e_probe.py:
# mean host wait / device staging / device frame over the last 60 frames.
for N in 0; do
  SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_$N.log | tail -1
  grep "host wait" gpurun_out/rt_$N.log | tail -60 | awk '{h+=$4; s+=$9; f+=$12; c++} END {print "host", h/c, "stage", s/c, "frame", f/c}'
done
# least-squares split of the device frame into fixed + per-iteration
python - <<'PY'
import re, numpy as np
rows = [(float(m.group(1)), int(m.group(2))) for m in
        (re.search(r"frame ([0-9.]+) us.*iters (\d+)", l) for l in open("gpurun_out/rt_0.log")) if m]
f, it = np.array([r[0] for r in rows]), np.array([r[1] for r in rows], dtype=float)
(a, b), *_ = np.linalg.lstsq(np.vstack([np.ones_like(it), it]).T, f, rcond=None)
print(f"resident device frame: {a:.1f} us + {b:.2f} us/iter over {len(rows)} frames")
PY
