#!/bin/bash
# ncu capture of one single-scene fused launch (config 2, a warm-started frame of the scenario)
python tools/prof_frame.py scene > gpurun_out/plain_scene.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:swarm_kernel -s 3 -c 1 \
    -o gpurun_out/prof_scene python tools/prof_frame.py scene > gpurun_out/ncu_scene.log 2>&1
echo "ncu_scene rc=$?"
