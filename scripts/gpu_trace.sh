mkdir -p gpurun_out
bash scripts/gpu_tests.sh
ADAPT_TRACE_HOST=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/trace.log 2>&1; echo trace rc=$?
bash scripts/gpu_bench_levels.sh
