TAG=head python scripts/c3_time.py
TAG=head_hostsegs ADAPT_HOST_SEGS=1 python scripts/c3_time.py
BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
timeout 600 python bench.py --steps 10 --warmup 3 $BA > gpurun_out/bp.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bp.log').read().strip().splitlines()[-1]); print('C4', d['ms_per_step'], d['phase_ms_per_step'])"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
