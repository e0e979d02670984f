SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_3.log | tail -1
echo noflush; grep "prelude cycles" gpurun_out/rt_3.log | sed -n 20,70p | awk '{a+=$5; b+=$7; m+=$9; k+=$11; s+=$13; c++} END {print "hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
echo flush; grep "prelude cycles" gpurun_out/rt_3.log | tail -60 | awk '{a+=$5; b+=$7; m+=$9; k+=$11; s+=$13; c++} END {print "hyp", a/c, "load_world", b/c, "misc", m/c, "consts", k/c, "sync", s/c}'
grep "prelude cycles" gpurun_out/rt_3.log | tail -3
