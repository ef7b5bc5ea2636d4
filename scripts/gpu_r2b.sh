# host trace at the strong-scaling proxy size + sanitizer + remaining gpu tests
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
ADAPT_TRACE_HOST=1 timeout 300 python bench.py --rows 12500000 --steps 2 --warmup 2 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/trace_proxy.log 2>&1; echo "trace rc=$?"
ADAPT_TRACE_HOST=1 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e --no-records --no-c5 --no-kfold --no-c2 --no-proxy > gpurun_out/trace_full.log 2>&1; echo "trace rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x -k "not fullsize" --deselect tests/test_gpu_parity.py::test_degenerate_cases_general_path > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "degenerate" > gpurun_out/pytest_degen.log 2>&1; echo "degen rc=$?"; tail -3 gpurun_out/pytest_degen.log
SAN_TIMEOUT=900 bash scripts/gpu_sanitize.sh
