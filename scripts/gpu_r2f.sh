mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-c2 > gpurun_out/bench_r2f.log 2>&1; echo "bench rc=$?"
python -c "
import json;l=[x for x in open('gpurun_out/bench_r2f.log') if x.startswith('{')][-1];d=json.loads(l)
p=d['strong_scaling_proxy']
print(d['ms_per_step'], d['phase_ms_per_step'], d['kfold']['ms'], {k:v for k,v in p.items() if k in ('ms_per_step','kernel_ms_per_step','host_idle_share','projected_step_ms_p8','projected_speedup_p8')})"
