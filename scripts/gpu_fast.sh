mkdir -p gpurun_out
bash scripts/gpu_tests.sh
bash scripts/gpu_bench_levels.sh
