# experiment: stale-level histograms (odd levels from the parent's pieces + route filter)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
ADAPT_STALE_HIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_forest.py tests/test_gpu_fullsize.py -q -x -k "not c5" > gpurun_out/pytest_stale.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_stale.log
for v in 0 1; do
  if [ $v = 1 ]; then export ADAPT_STALE_HIST=1; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_stale$v.log 2>&1; echo "bench rc=$?"
  python - $v <<'PY'
import json,sys
l=[x for x in open('gpurun_out/bench_stale%s.log'%sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
print("stale", sys.argv[1], "ms/step", d["ms_per_step"], "phases", d["phase_ms_per_step"])
for i, lv in enumerate(d["levels"]): print(i, lv["rows_hist"], lv["ms"])
PY
done
