# quick: parity subset + the main C4 step (no side configs)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_forest.py tests/test_gpu_kfold.py -q -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy ${BENCH_EXTRA} > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_quick.log') if x.startswith('{')][-1]; d=json.loads(l)
print("ms/step", d["ms_per_step"], "train/s %.3g" % d["train_samples_per_s"], "phases", d["phase_ms_per_step"])
print("level loop", d["level_loop_roofline"]["ms_per_step"], d["level_loop_roofline"]["frac"])
for i, lv in enumerate(d["levels"]): print(i, lv["ms"])
PY
