bash tools/resident_trace.sh
grep "\[resident\] init" gpurun_out/rt_0.log | tail -60 | awk '{i+=$4; l+=$7; r+=$10; o+=$13; c++} END {print "init", i/c, "loop", l/c, "rec", r/c, "out", o/c}'
timeout 120 python tools/phase_probe.py 2>&1 | sed -n 2,4p | cut -c1-1200
