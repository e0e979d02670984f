SEPSO_RESIDENT_TRACE=1 timeout 120 python tools/e2e_probe.py 2> gpurun_out/rt_5.log | tail -1
grep "plan_frame\]" gpurun_out/rt_5.log | tail -60 | awk '{a+=$4; b+=$7; c2+=$10; c++} END {print "prep", a/c, "post->seen", b/c, "after", c2/c}'
grep "host wait" gpurun_out/rt_5.log | tail -60 | awk '{h+=$4; s+=$9; f+=$12; c++} END {print "host wait", h/c, "stage", s/c, "frame", f/c}'
