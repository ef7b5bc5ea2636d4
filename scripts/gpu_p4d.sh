BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
for v in base brload base brload; do
  if [ $v = base ]; then d=.; else d=.variants/$v; fi
  (cd $d && ADAPT_PROFILE_LEVELS=1 timeout 600 python bench.py --steps 5 --warmup 3 $BA > /tmp/bv_$v.log 2>&1; python - $v <<'PY'
import json,sys
d=json.loads([x for x in open('/tmp/bv_%s.log'%sys.argv[1]) if x.startswith('{')][-1])
print(sys.argv[1], "ms/step", round(d["ms_per_step"],3), "partition", d["phase_ms_per_step"]["partition"], [l['ms'].get('partition') for l in d['levels']])
PY
)
done
