mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_c4.log
