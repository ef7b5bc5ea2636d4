mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 > gpurun_out/bp.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['c3_train'], d['level_loop_roofline']['schedule'])"
ADAPT_TWO_LEVEL=1 SAN_TAG=_2lvl bash scripts/gpu_sanitize.sh
