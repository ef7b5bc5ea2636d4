mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kfold.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -m gpu -x -k "kfold or select or c1" > gpurun_out/pytest_kfold.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_kfold.log
