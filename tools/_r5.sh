timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
for v in 0 1 0 1; do echo "== PREWALK=$v"; SEPSO_PREWALK=$v timeout 120 python tools/e2e_probe.py 2>&1 | tail -2; SEPSO_PREWALK=$v timeout 60 python tools/flush_probe.py 2>&1 | tail -2; done
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log
