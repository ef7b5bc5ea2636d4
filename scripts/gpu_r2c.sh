mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python -c "
import json;l=[x for x in open('gpurun_out/bench_default.log') if x.startswith('{')][-1];d=json.loads(l)
print(d['ms_per_step'], d['cpu_baseline'].get('per_config'))"
