BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
for v in new all new all; do
  if [ $v = all ]; then export ADAPT_ZERO_ALL=1; else unset ADAPT_ZERO_ALL; fi
  ADAPT_PROFILE_LEVELS=1 timeout 600 python bench.py --steps 5 --warmup 3 $BA > /tmp/b.log 2>&1; python -c "
import json; d=json.loads([x for x in open('/tmp/b.log') if x.startswith('{')][-1]); ph=d['phase_ms_per_step']; print('$v', d['ms_per_step'], ph['zero'], ph['hist'])"
done
unset ADAPT_ZERO_ALL
timeout 300 python bench.py --steps 10 --warmup 3 $BA > /tmp/b2.log 2>&1; python -c "
import json; d=json.loads([x for x in open('/tmp/b2.log') if x.startswith('{')][-1]); print('plain', d['ms_per_step'])"
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
