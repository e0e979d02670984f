timeout 300 python bench.py > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('value',d['value'],'e2e',d['e2e']['value'],'ref-cpu',d['cpu_baseline']['value'], 'fp64', d['fp64']['e2e_plans_per_s'], 'c5', d['config5']['plans_per_s'], 'c3', d['config3']['ms_per_evolution'], 'launches', d['gpu_launches'], 'iters', d['e2e']['mean_iterations_per_frame'])
PY
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; tail -c 400 gpurun_out/bench_ref.log
