SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_6.log | tail -1
grep "record cycles" gpurun_out/rt_6.log | tail -60 | awk '{a+=$5; b+=$7; c++} END {print "path_length64", a/c, "rest", b/c}'
grep "record cycles" gpurun_out/rt_6.log | sed -n 20,70p | awk '{a+=$5; b+=$7; c++} END {print "noflush path_length64", a/c, "rest", b/c}'
