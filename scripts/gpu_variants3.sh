# partition unroll variants (built locally as gpurun_variants_u*.so)
mkdir -p gpurun_out
cp paper_2303_08873_b200/libadapt.so /tmp/libadapt_base.so
for v in base u3 u4; do
  if [ $v = base ]; then cp /tmp/libadapt_base.so paper_2303_08873_b200/libadapt.so; else cp gpurun_variants_$v.so paper_2303_08873_b200/libadapt.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_var_$v.log 2>&1
  python - $v <<'PY'
import json,sys
l=[x for x in open('gpurun_out/bench_var_%s.log'%sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l)
print(sys.argv[1], "ms/step", round(d["ms_per_step"],3), "partition", d["phase_ms_per_step"]["partition"], "hist", d["phase_ms_per_step"]["hist"])
PY
done
cp /tmp/libadapt_base.so paper_2303_08873_b200/libadapt.so
