# round 2: new tests (RS multirank, degenerate general path) + bench with the new sub-objects
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -q -m gpu -x -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_default.log
