mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kfold.py tests/test_gpu_forest.py tests/test_gpu_quantile.py -q -x > gpurun_out/pytest_r2e.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2e.log
bash scripts/gpu_kf_trace.sh 2>&1 | tail -6 | cut -c1-400
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-records --no-c5 --no-c2 > gpurun_out/bench_r2e.log 2>&1; echo "bench rc=$?"
python -c "
import json;l=[x for x in open('gpurun_out/bench_r2e.log') if x.startswith('{')][-1];d=json.loads(l)
p=d['strong_scaling_proxy']
print(d['ms_per_step'], d['kfold']['ms'], {k:v for k,v in p.items() if k in ('ms_per_step','kernel_ms_per_step','host_idle_share','projected_step_ms_p8','projected_speedup_p8')})"
