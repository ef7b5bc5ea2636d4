BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
timeout 1200 python -m pytest tests/test_gpu_dev_segs.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_dev4.log 2>&1; echo "pytest dev4 rc=$?"; tail -3 gpurun_out/pytest_dev4.log
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 $BA > /tmp/b2.log 2>&1; python -c "
import json; d=json.loads([x for x in open('/tmp/b2.log') if x.startswith('{')][-1]); print('plain', d['ms_per_step'])"; done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
