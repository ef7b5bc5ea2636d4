# round-2 evidence at the two-level schedule: GPU tests, smoke, driver-style
# bench, reference arm, launch list, ncu captures of the step's kernels
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
bash scripts/gpu_tests.sh
bash scripts/gpu_bench_full.sh
for spec in partition4_kernel:1 tag_kernel:1 hist_kernel:3 hist_kernel:4 label_bin:0 select_kernel_c:0 split_kernel:10 partition_kernel:0; do
  NCU_KERNEL=${spec%%:*} NCU_SKIP=${spec##*:} BENCH_ARGS="--no-c5 --no-kfold --no-c2 --no-proxy" bash scripts/gpu_ncu_one.sh
done
NCU_KERNEL=select_kernel_h NCU_SKIP=0 BENCH_ARGS="--no-kfold --no-c2 --no-proxy" bash scripts/gpu_ncu_one.sh
mv gpurun_out/prof_select_kernel_h_0.ncu-rep gpurun_out/prof_select_kernel_h_c5.ncu-rep 2>/dev/null
ls gpurun_out
