timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_1.log | tail -2
echo noflush; grep "prelude:" gpurun_out/rt_1.log | sed -n 20,70p | awk '{a+=$4; b+=$6; m+=$8; k+=$10; s+=$12; c++} END {print "hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
echo flush; grep "prelude:" gpurun_out/rt_1.log | tail -60 | awk '{a+=$4; b+=$6; m+=$8; k+=$10; s+=$12; c++} END {print "hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
grep "\[resident\] init" gpurun_out/rt_1.log | tail -60 | awk '{i+=$3; p+=$6; o+=$17; c++} END {print "init", i/c, "pre", p/c, "out", o/c}'
grep "host wait" gpurun_out/rt_1.log | tail -60 | awk '{h+=$4; s+=$9; f+=$12; c++} END {print "host", h/c, "stage", s/c, "frame", f/c}'
