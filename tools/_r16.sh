timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
bash tools/_r14.sh
grep "\[resident\] init" gpurun_out/rt_3.log | tail -60 | awk '{i+=$3; p+=$6; o+=$17; c++} END {print "init", i/c, "pre", p/c, "out", o/c}'
grep "host wait" gpurun_out/rt_3.log | tail -60 | awk '{h+=$4; s+=$9; f+=$12; c++} END {print "host wait", h/c, "stage", s/c, "frame", f/c}'
timeout 60 python tools/flush_probe.py 2>&1 | tail -2
bash tools/_r12.sh
