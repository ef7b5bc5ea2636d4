# A/B of compile-time tuning knobs: rebuild on the box per variant, bench the C4 step
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for v in "" ${VARIANTS}; do
  ADAPT_NVCC_DEFS="$v" python paper_2303_08873_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_var.log 2>&1
  python -c "
import json;l=[x for x in open('gpurun_out/bench_var.log') if x.startswith('{')][-1];d=json.loads(l);p=d['phase_ms_per_step']
print('[$v]', round(d['ms_per_step'],3), {k:p[k] for k in ('ingest','partition','hist','split','select')})"
done
