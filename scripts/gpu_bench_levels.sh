mkdir -p gpurun_out
ADAPT_PROFILE_LEVELS=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_levels.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_levels.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], {k: v for k, v in d['phase_ms_per_step'].items()})
PY
