mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for spec in split_small_kernel:9 split_kernel:11 subtract_kernel:10 winner_kernel:11; do
  NCU_KERNEL=${spec%%:*} NCU_SKIP=${spec##*:} BENCH_ARGS="--no-c5 --no-kfold --no-c2 --no-proxy" bash scripts/gpu_ncu_one.sh
done
