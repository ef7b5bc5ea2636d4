mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
#timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_forest.py tests/test_gpu_kfold.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
for m in 1 3; do
ADAPT_HIST_PLAN=$m timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_plan$m.log 2>&1; echo "bench rc=$?"
python - $m <<'PY'
import json,sys
l=[x for x in open('gpurun_out/bench_plan%s.log'%sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
print("mode", sys.argv[1], "ms/step", d["ms_per_step"], "hist", d["phase_ms_per_step"]["hist"])
print(" ".join("%.3f" % lv["ms"]["hist"] for lv in d["levels"]))
PY
done
