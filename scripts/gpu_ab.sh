# A/B of the level-loop schedules: GPU tests, then plain benches per variant
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
if [ -z "$NO_TESTS" ]; then
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
for v in ${VARIANTS:-two one}; do
  env $(echo $v | tr '+' ' ' | sed 's/two//;s/one/ADAPT_ONE_LEVEL=1/;s/nojoint/ADAPT_NO_JOINT=1/') ADAPT_PROFILE_LEVELS=1 timeout 600 python bench.py --steps 3 --warmup 2 $BA > gpurun_out/bl_$v.log 2>&1
  env $(echo $v | tr '+' ' ' | sed 's/two//;s/one/ADAPT_ONE_LEVEL=1/;s/nojoint/ADAPT_NO_JOINT=1/') timeout 300 python bench.py --steps 10 --warmup 3 $BA > gpurun_out/bp_$v.log 2>&1
  python - $v <<'PY'
import json,sys
v=sys.argv[1]
d=json.loads(open(f'gpurun_out/bl_{v}.log').read().strip().splitlines()[-1])
p=json.loads(open(f'gpurun_out/bp_{v}.log').read().strip().splitlines()[-1])
print(v, 'plain', round(p['ms_per_step'],3), 'loop frac', round(p['level_loop_roofline']['frac'],4), 'profiled', round(d['ms_per_step'],3), {k: v for k, v in d['phase_ms_per_step'].items()})
print('  levels', [(i, l['ms']) for i,l in enumerate(d['levels'])])
PY
done
