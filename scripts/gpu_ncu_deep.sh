mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for spec in hist_kernel:11 split_kernel:11 hist_kernel:5 winner_kernel:11; do
  NCU_KERNEL=${spec%%:*} NCU_SKIP=${spec##*:} bash scripts/gpu_ncu_one.sh
done
