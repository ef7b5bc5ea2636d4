# two-level moves: parity suite, then the per-level bench (both schedules)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
for mode in two one; do
  if [ $mode = one ]; then export ADAPT_ONE_LEVEL=1; fi
  ADAPT_PROFILE_LEVELS=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_levels_$mode.log 2>&1; echo "bench $mode rc=$?"
  python - $mode <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/bench_levels_{sys.argv[1]}.log').read().strip().splitlines()[-1])
print(sys.argv[1], d['ms_per_step'], {k: v for k, v in d['phase_ms_per_step'].items()})
for i,l in enumerate(d['levels']): print(i, l['rows_hist'], l['rows_part'], l['ms'])
PY
done
unset ADAPT_ONE_LEVEL
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_plain.log 2>&1; echo "plain rc=$?"; tail -c 600 gpurun_out/bench_plain.log
