mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
ADAPT_PROFILE_LEVELS=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_levels_two.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/bench_levels_two.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], {k: v for k, v in d['phase_ms_per_step'].items()})
for i,l in enumerate(d['levels']): print(i, l['rows_hist'], l['rows_part'], l['ms'])
PY
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_plain_two.log 2>&1; echo "plain rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_plain_two.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['level_loop_roofline'])"
