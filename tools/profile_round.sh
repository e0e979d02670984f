#!/bin/bash
# End-of-change profiling pass (run on the GPU box after the plain bench exited 0):
#  1. ncu launch list of a short bench run -> gpurun_out/bench_launches.csv
#  2. ncu --set full of the config-2 latency kernel (one L2-flushed frame),
#     the config-5 throughput kernel, config 4's k_eval_path_wide and k_step.
set -x
O=gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file $O/bench_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:swarm_kernel -s 8 -c 1 -o $O/scene \
    python tools/flush_probe.py > $O/ncu_scene.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:swarm_kernel -s 1 -c 1 -o $O/batched \
    python tools/batched_probe.py > $O/ncu_batched.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_eval_path_wide|k_step" -s 2 -c 2 -o $O/config4 \
    python tools/probe_config4.py > $O/ncu_c4.log 2>&1
ls -la $O
