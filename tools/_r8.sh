bash tools/resident_trace.sh
grep "\[resident\] init" gpurun_out/rt_0.log | tail -60 | awk '{i+=$3; p+=$6; w+=$8; l+=$11; r+=$14; o+=$17; c++} END {print "init", i/c, "pre", p/c, "wait", w/c, "loop", l/c, "rec", r/c, "out", o/c}'
grep "\[resident\] init" gpurun_out/rt_0.log | tail -3
