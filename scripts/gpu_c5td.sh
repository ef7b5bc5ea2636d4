for i in 1 2; do timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-records --no-kfold --no-c2 --no-proxy > /tmp/b.log 2>&1; python -c "
import json; d=json.loads([x for x in open('/tmp/b.log') if x.startswith('{')][-1]); c=d['select_c5']; print(d['ms_per_step'], c['trained']['ms_per_batch'], c['trained']['roofline']['frac'], c['complete']['ms_per_batch'], c['complete']['roofline']['frac'])"; done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
