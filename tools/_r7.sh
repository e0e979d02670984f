timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
timeout 120 python tools/e2e_probe.py 2>&1 | tail -2
timeout 60 python tools/flush_probe.py 2>&1 | tail -2
bash tools/resident_trace.sh
grep "\[resident\] init" gpurun_out/rt_0.log | tail -60 | awk '{i+=$3; l+=$6; r+=$9; o+=$12; c++} END {print "init", i/c, "loop", l/c, "rec", r/c, "out", o/c}'
timeout 120 python tools/phase_probe.py 2>&1 | sed -n 2,4p | grep -o "init: [^|]*|  *ns: [^|]*"
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('value',d['value'],'e2e',d['e2e']['value'],'ref-cpu',d['cpu_baseline']['value'], 'fp64', d['fp64']['e2e_plans_per_s'], 'c5', d['config5']['plans_per_s'], 'c3', d['config3']['ms_per_evolution'], 'launches', d['gpu_launches'])
PY
