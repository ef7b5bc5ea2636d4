BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
for v in dev host dev host; do
  if [ $v = host ]; then export ADAPT_HOST_HASH=1; else unset ADAPT_HOST_HASH; fi
  timeout 600 python bench.py --steps 10 --warmup 3 $BA > /tmp/b.log 2>&1; python -c "
import json; d=json.loads([x for x in open('/tmp/b.log') if x.startswith('{')][-1]); ph=d['phase_ms_per_step']; print('$v', d['ms_per_step'], ph['ingest'], ph.get('values'))"
done
unset ADAPT_HOST_HASH
python scripts/c3_time.py
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
