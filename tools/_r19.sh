SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_4.log | tail -1
echo noflush; grep "to-pre-check" gpurun_out/rt_4.log | sed -n 20,70p | awk '{a+=$6; b+=$8; c++} END {print "to-pre-check", a/c, "to-branch", b/c}'
echo flush; grep "to-pre-check" gpurun_out/rt_4.log | tail -60 | awk '{a+=$6; b+=$8; c++} END {print "to-pre-check", a/c, "to-branch", b/c}'
grep "prelude cycles: hyp" gpurun_out/rt_4.log | tail -60 | awk '{a+=$5; b+=$7; m+=$9; k+=$11; s+=$13; c++} END {print "hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
