mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_full.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-records > gpurun_out/bench_c5.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_c5.log
