mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quantile.py tests/test_gpu_multirank.py tests/test_gpu_kfold.py -q -m gpu -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_q.log
