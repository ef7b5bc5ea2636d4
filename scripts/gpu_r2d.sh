mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nccl_self.py -q -x -k "select_table or nccl or errors" > gpurun_out/pytest_r2d.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2d.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"
python -c "
import json;l=[x for x in open('gpurun_out/bench_e2e.log') if x.startswith('{')][-1];d=json.loads(l)
print(d['ms_per_step'], d['e2e'])"
