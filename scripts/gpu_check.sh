set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"
tail -5 gpurun_out/bench_c3.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 1 > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"
tail -5 gpurun_out/bench_c4.log
