mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x -k "select or c5 or c4_full" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_sel.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-records > gpurun_out/bench_c5.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_c5.log
