SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_1.log | tail -2
echo noflush; grep "prelude:" gpurun_out/rt_1.log | sed -n 20,70p | awk '{a+=$4; b+=$6; m+=$8; k+=$10; s+=$12; c++} END {print "hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
echo flush; grep "prelude:" gpurun_out/rt_1.log | tail -60 | awk '{a+=$4; b+=$6; m+=$8; k+=$10; s+=$12; c++} END {print "hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
