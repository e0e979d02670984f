#!/bin/bash
# Per-frame split of sf_plan_frame on the resident planner (SEPSO_RESIDENT_TRACE=1):
# host prep / post->seen / after, device stage / frame, and the constants stage
# (cycles) over the L2-flushed frames of tools/e2e_probe.py; then the
# fixed + per-iteration fit of tools/e2e_fit.py.
SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_split.log | tail -1
grep "plan_frame\]" gpurun_out/rt_split.log | tail -60 | awk '{a+=$4; b+=$7; c2+=$10; c++} END {print "host prep", a/c, "post->seen", b/c, "after", c2/c}'
grep "host wait" gpurun_out/rt_split.log | tail -60 | awk '{s+=$9; f+=$12; c++} END {print "device stage", s/c, "frame", f/c}'
grep "prelude cycles: hyp" gpurun_out/rt_split.log | tail -60 | awk '{a+=$5; b+=$7; m+=$9; k+=$11; s+=$13; c++} END {print "constants (cycles): hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
grep "record cycles" gpurun_out/rt_split.log | tail -60 | awk '{a+=$5; b+=$7; c++} END {print "record (cycles): path_length64", a/c, "rest", b/c}'
timeout 120 python tools/e2e_fit.py
