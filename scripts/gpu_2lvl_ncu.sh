mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for spec in hist_kernel:3 hist_kernel:4 partition4_kernel:1 tag_kernel:1; do
  NCU_KERNEL=${spec%%:*} NCU_SKIP=${spec##*:} BENCH_ARGS="--no-c5 --no-kfold --no-c2 --no-proxy" bash scripts/gpu_ncu_one.sh
done
ls gpurun_out
