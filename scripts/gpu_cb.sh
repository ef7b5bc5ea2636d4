BA="--no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy"
for v in base tq4 base tq4; do
  if [ $v = base ]; then d=.; else d=.variants/$v; fi
  (cd $d && ADAPT_PROFILE_LEVELS=1 timeout 600 python bench.py --steps 5 --warmup 3 $BA > /tmp/bv_$v.log 2>&1; python - $v <<'PY'
import json,sys
d=json.loads([x for x in open('/tmp/bv_%s.log'%sys.argv[1]) if x.startswith('{')][-1])
ph=d["phase_ms_per_step"]
print(sys.argv[1], "ms/step", round(d["ms_per_step"],3), {k: ph[k] for k in ('partition','tag','hist','ingest')})
PY
)
done
timeout 300 python bench.py --steps 10 --warmup 3 $BA > /tmp/b2.log 2>&1; python -c "
import json; d=json.loads([x for x in open('/tmp/b2.log') if x.startswith('{')][-1]); print('plain', d['ms_per_step'])"
